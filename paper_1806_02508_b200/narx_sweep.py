"""Host layer of the C4 NARX sweep (lbbsp_narx_sweep_* in include/lbbsp_c.h):
W generalised NARX models (delay d, hidden H) trained / evaluated in one
launch each, histories and parameters resident on the device."""
import ctypes as C

import numpy as np

from . import abi
from ._lib import check, lib

_vp = C.c_void_p


def _L():
    L = lib()
    if not getattr(L, "_sweep_sigs", False):
        L.lbbsp_narxg_param_count.argtypes = [C.c_int, C.c_int]
        L.lbbsp_narxg_init.argtypes = [C.c_uint64, C.c_int, C.c_int, C.POINTER(C.c_float)]
        L.lbbsp_narx_sweep_train.argtypes = [C.c_int] * 4 + [_vp] * 4 + [
            C.POINTER(abi.NarxTrainConfig), C.c_int, _vp, _vp, _vp, _vp]
        L.lbbsp_narx_sweep_train.restype = C.c_int
        L.lbbsp_narx_sweep_scratch_floats.argtypes = [C.c_int] * 4
        L.lbbsp_narx_sweep_scratch_floats.restype = C.c_longlong
        L.lbbsp_narx_sweep_predict.argtypes = [C.c_int] * 4 + [_vp] * 6 + [C.c_double, _vp, _vp]
        L.lbbsp_narx_sweep_predict.restype = C.c_int
        L._sweep_sigs = True
    return L


class NarxSweep:
    def __init__(self, seeds, delay=10, hidden=64):
        import torch
        self.W, self.d, self.h = len(seeds), delay, hidden
        L = _L()
        self.P = L.lbbsp_narxg_param_count(delay, hidden)
        host = np.zeros((self.W, self.P), np.float32)
        for i, s in enumerate(seeds):
            check(L.lbbsp_narxg_init(C.c_uint64(int(s)), delay, hidden,
                                     host[i].ctypes.data_as(C.POINTER(C.c_float))))
        self.params = torch.from_numpy(host).cuda()

    def train(self, v, c, m, cfg=None, fixed_epochs=0, stream=None):
        """v/c/m: float64 arrays [W][L] (host or device tensors)."""
        import torch
        cfg = cfg if cfg is not None else abi.NarxTrainConfig.default(min_history=3)
        tv, tc, tm = (torch.as_tensor(np.ascontiguousarray(x) if isinstance(x, np.ndarray) else x,
                                      dtype=torch.float64).cuda().contiguous() for x in (v, c, m))
        W, Lh = tv.shape
        n_scr = _L().lbbsp_narx_sweep_scratch_floats(W, Lh, self.d, self.h)
        if getattr(self, "_scr", None) is None or self._scr.numel() < n_scr:
            self._scr = torch.empty(n_scr, dtype=torch.float32, device="cuda")
        ep = torch.zeros(W, dtype=torch.int32, device="cuda")
        loss = torch.zeros(W, dtype=torch.float32, device="cuda")
        s = stream if stream is not None else torch.cuda.current_stream().cuda_stream
        check(_L().lbbsp_narx_sweep_train(W, Lh, self.d, self.h, tv.data_ptr(), tc.data_ptr(),
                                          tm.data_ptr(), self.params.data_ptr(), C.byref(cfg),
                                          int(fixed_epochs), ep.data_ptr(), loss.data_ptr(),
                                          self._scr.data_ptr(), s))
        self._last = (tv, tc, tm)
        return ep, loss

    def predict(self, v, c, m, c_now, m_now, floor=1e-3):
        import torch
        tv, tc, tm = (torch.as_tensor(x, dtype=torch.float64).cuda().contiguous() for x in (v, c, m))
        cn = torch.as_tensor(c_now, dtype=torch.float64).cuda().contiguous()
        mn = torch.as_tensor(m_now, dtype=torch.float64).cuda().contiguous()
        out = torch.zeros(self.W, dtype=torch.float64, device="cuda")
        W, Lh = tv.shape
        check(_L().lbbsp_narx_sweep_predict(W, Lh, self.d, self.h, tv.data_ptr(), tc.data_ptr(),
                                            tm.data_ptr(), cn.data_ptr(), mn.data_ptr(),
                                            self.params.data_ptr(), float(floor), out.data_ptr(),
                                            torch.cuda.current_stream().cuda_stream))
        return out

    def host_params(self):
        return self.params.cpu().numpy().astype(np.float64)
