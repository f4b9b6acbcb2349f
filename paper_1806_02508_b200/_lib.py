"""Loader for the in-tree CUDA library liblbbsp_b200.so.

Fails loudly: if the library is missing, every product entry point raises.
There is no CPU fallback on the product path.
"""
import ctypes as C
import os

from . import abi

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LBBSP_LIB_OVERRIDE") or os.path.join(HERE, "liblbbsp_b200.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p

# name -> argtypes ; every function returns int status unless listed in _RESTYPES
SIGNATURES = {
    "lbbsp_version": [],
    "lbbsp_device_count": [],
    "lbbsp_check_status": [C.POINTER(abi.DevStatus)],
    "lbbsp_solve_prop": [_vp, C.c_int, C.c_int, C.c_double, _vp, _vp, _vp],
    "lbbsp_solve_gpu": [_vp, _vp, C.c_int, C.c_int, _vp, _vp, _vp],
    "lbbsp_cpu_allocate": [_dp, C.c_int, C.c_int, _ip],
    "lbbsp_gpu_allocate": [C.POINTER(abi.GpuProfile), _dp, C.c_int, C.c_int, _ip],
    "lbbsp_narx_init": [C.c_uint64, C.POINTER(abi.NarxModel)],
    "lbbsp_ema": [_dp, C.c_int, C.c_double, _dp],
    "lbbsp_narx_predict": [C.POINTER(abi.NarxModel), _dp, _dp, _dp, C.c_double, _dp],
    "lbbsp_glibc_tanh": [_dp, _dp, C.c_longlong],
    "lbbsp_narx_train_online": [C.POINTER(abi.NarxModel), _dp, _dp, _dp, C.c_int,
                                C.POINTER(abi.NarxTrainConfig), C.POINTER(abi.NarxReport), _dp],
    "lbbsp_predictor_create": [C.POINTER(abi.PredictorConfig), C.c_int, C.c_int,
                               C.POINTER(C.c_uint64), C.POINTER(abi.NarxModel), C.POINTER(_vp)],
    "lbbsp_predictor_destroy": [_vp],
    "lbbsp_predictor_observe": [_vp, _vp, _vp, _vp, _vp],
    "lbbsp_predictor_predict": [_vp, _vp, _vp, _vp, _vp],
    "lbbsp_predictor_train_rotation": [_vp, _vp],
    "lbbsp_predictor_train_all": [_vp, _vp],
    "lbbsp_predictor_get_models": [_vp, C.POINTER(abi.NarxModel)],
    "lbbsp_predictor_history_len": [_vp, _ip],
    "lbbsp_sample_stream": [C.c_uint64, C.c_int64, C.c_int, C.c_int, _vp, _vp],
    "lbbsp_lr_data_create": [C.c_uint64, C.c_int, C.c_int, C.c_double, C.POINTER(_vp)],
    "lbbsp_lr_data_upload": [_dp, _dp, C.c_int, C.c_int, C.POINTER(_vp)],
    "lbbsp_lr_data_destroy": [_vp],
    "lbbsp_lr_data_dim": [_vp, _ip, _ip],
    "lbbsp_lr_worker_grads": [_vp, _vp, _vp, _vp, C.c_int, _vp, _vp, _vp],
    "lbbsp_aggregate_apply": [_vp, _vp, C.c_int, C.c_int, C.c_int, C.c_double, _vp, _vp, _vp,
                              _vp, _vp],
    "lbbsp_lr_loss": [_vp, _vp, _vp, _vp],
    "lbbsp_batch_gradient": [_vp, _dp, _ip, C.c_int, _dp],
    "lbbsp_loss": [_vp, _dp, _dp],
    "lbbsp_aggregate": [_dp, _ip, C.c_int, C.c_int, C.c_int, _dp],
    "lbbsp_sim_create": [C.POINTER(abi.SimConfig), C.POINTER(_vp)],
    "lbbsp_sim_destroy": [_vp],
    "lbbsp_sim_run": [_vp, C.c_int, _vp],
    "lbbsp_sim_records": [_vp, C.c_int, _ip, C.POINTER(abi.IterScalars), _ip, _dp, _dp, _dp, _dp,
                          _dp, _dp],
    "lbbsp_sim_status": [_vp, _ip, _ip],
    "lbbsp_sim_launches_per_iteration": [_vp, _ip],
    "lbbsp_benchmark_series": [C.c_uint64, C.c_int, C.c_int] + [C.c_double] * 6 + [_dp] * 3,
    "lbbsp_sim_metrics": [_vp, C.c_int, C.POINTER(abi.Metrics)],
    "lbbsp_sim_record_workers": [_vp, C.c_int, _ip, _ip],
    "lbbsp_sim_summary": [_vp, _dp, C.POINTER(C.c_int64)],
    "lbbsp_compute_metrics": [C.POINTER(abi.RecordsView), C.c_int, C.c_int, C.c_int,
                              C.POINTER(abi.Metrics)],
    "lbbsp_write_records_csv": [C.POINTER(abi.RecordsView), C.c_char_p],
    "lbbsp_write_metrics_json": [C.POINTER(abi.Metrics), C.c_double, C.c_int, C.c_int,
                                 C.c_char_p],
    "lbbsp_trace_parse": [C.c_char_p, C.POINTER(_vp)],
    "lbbsp_trace_create": [C.c_int, C.POINTER(C.c_char_p), _ip, _dp, _dp, _dp, C.POINTER(_vp)],
    "lbbsp_trace_destroy": [_vp],
    "lbbsp_trace_count": [_vp, _ip],
    "lbbsp_trace_info": [_vp, C.c_int, C.POINTER(C.c_char_p), _ip, _dp],
    "lbbsp_trace_points": [_vp, C.c_int, _dp, _dp, _dp],
    "lbbsp_trace_write": [_vp, C.c_char_p],
    "lbbsp_trace_map": [_vp, C.c_int, C.c_uint64, _ip],
    "lbbsp_trace_at": [_vp, C.c_int, C.c_double, _dp, _dp],
    "lbbsp_narx_load_csv": [C.c_char_p, C.POINTER(abi.NarxModel)],
    "lbbsp_narx_save_csv": [C.POINTER(abi.NarxModel), C.c_char_p],
    "lbbsp_scenario_load": [C.c_char_p, C.POINTER(_vp)],
    "lbbsp_scenario_destroy": [_vp],
    "lbbsp_scenario_set_seed": [_vp, C.c_uint64],
    "lbbsp_scenario_get_info": [_vp, C.POINTER(abi.ScenarioInfo)],
    "lbbsp_scenario_sim_cfg": [_vp, C.POINTER(C.POINTER(abi.SimConfig))],
    "lbbsp_predictor_series_rmse": [C.c_int, C.POINTER(abi.PredictorConfig), _dp, _dp, _dp,
                                    C.c_int, C.c_double, C.c_uint64, C.c_int, _dp],
    "lbbsp_cmd_run": [C.c_char_p, C.c_char_p, C.c_int, C.c_uint64],
}

_lib = None


def lib():
    """The loaded product library. Raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                f"g.build()'` (make -C paper_1806_02508_b200/csrc). The B200 path has no CPU "
                f"fallback.")
        L = C.CDLL(LIB_PATH)
        for name, argtypes in SIGNATURES.items():
            fn = getattr(L, name)
            fn.argtypes = argtypes
            fn.restype = C.c_int
        L.lbbsp_last_error.restype = C.c_char_p
        L.lbbsp_last_error.argtypes = []
        _lib = L
    return _lib


def check(code):
    """Raise the reference-typed exception for a non-zero status."""
    if code != 0:
        from .errors import raise_for
        raise_for(code, lib().lbbsp_last_error().decode())
    return code
