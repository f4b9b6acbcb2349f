"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports
every entry point include/lbbsp_c.h declares, and fails loudly (no CPU
fallback) when no device is present."""
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "lbbsp_c.h")


def declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(lbbsp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_entry_points():
    names = declared()
    assert "lbbsp_solve_prop" in names and "lbbsp_mlp_run" in names and len(names) > 40


def test_library_exports_every_declared_symbol():
    from paper_1806_02508_b200._lib import lib
    L = lib()
    missing = [n for n in declared() if not hasattr(L, n)]
    assert not missing, missing


def test_compute_entry_points_fail_loudly_without_device():
    from paper_1806_02508_b200._lib import lib
    from paper_1806_02508_b200 import lbbsp
    from paper_1806_02508_b200.errors import CudaError
    if lib().lbbsp_device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(CudaError, match="no CPU fallback"):
        lbbsp.cpu_allocate([1.0, 2.0], 10)
    with pytest.raises(CudaError):
        lbbsp.Simulation(workers=2, total_budget=8, max_updates=2)


def test_cli_fails_loudly_without_device(tmp_path, capfd):
    """cmd_run parses the scenario on the host, then needs the device driver."""
    from paper_1806_02508_b200._lib import lib
    from paper_1806_02508_b200 import lbbsp
    if lib().lbbsp_device_count() > 0:
        pytest.skip("a device is present")
    cfg = tmp_path / "homo.json"
    cfg.write_text('{"scheme": "bsp", "workers": 2, "total_budget": 8, "max_iterations": 3}')
    assert lbbsp.cmd_run(cfg, tmp_path / "out") == 1
    assert "no CPU fallback" in capfd.readouterr().err


def test_reference_signature_shim_is_built():
    exe = os.path.join(REPO, "tests", "cpp", "test_shim")
    assert os.path.exists(exe), "build() compiles tests/cpp/test_shim against include/lbbsp_b200.hpp"


def test_two_rank_gloo_control_exchange():
    """Multi-GPU control plane on CPU (gloo, world_size 2): every rank
    all-gathers the per-worker speeds and runs the identical deterministic
    solver, so the batch sizes agree without a broadcast."""
    import sys
    code = os.path.join(REPO, "tests", "_gloo_worker.py")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT="29533", PYTHONPATH=REPO)
    procs = [subprocess.Popen([sys.executable, code, str(r), "2"], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE) for r in range(2)]
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e.decode()[-2000:]
    lines = [o.decode().strip().splitlines()[-1] for o, _ in outs]
    assert lines[0] == lines[1]


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_connect_handshake(world):
    """The product's multi-rank control plane (mlp.connect) on CPU ranks over
    gloo: every rank joins rank 0's communicator id, and every rank maps the
    same rank-ordered list of peer handles."""
    import json
    import sys
    code = os.path.join(REPO, "tests", "_gloo_connect_worker.py")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", MASTER_PORT=str(29540 + world), PYTHONPATH=REPO)
    procs = [subprocess.Popen([sys.executable, code, str(r), str(world)], env=env,
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE) for r in range(world)]
    outs = [p.communicate(timeout=120) for p in procs]
    for p, (o, e) in zip(procs, outs):
        assert p.returncode == 0, e.decode()[-2000:]
    res = [json.loads(o.decode().strip().splitlines()[-1]) for o, _ in outs]
    for r, d in enumerate(res):
        assert d["uid"] == "uid-of-rank-0"
        assert d["handles"] == list(range(world)) and d["lens"] == [64] * world
        assert d["calls"] == (["uid"] if r == 0 else []) + ["comm", "handle", "peers"]
        assert d["ret"] == world
