"""Host-buffer placement helper for the e2e path (paper_1806_02508_b200/hostio.py)."""
from paper_1806_02508_b200.hostio import _parse_cpulist, gpu_local_cpus


def test_parse_cpulist():
    assert _parse_cpulist("0-3,8,10-11\n") == {0, 1, 2, 3, 8, 10, 11}
    assert _parse_cpulist("") == set()


def test_gpu_local_cpus_without_gpu_is_empty_or_subset():
    import os
    cpus = gpu_local_cpus(0)
    assert cpus <= os.sched_getaffinity(0)
