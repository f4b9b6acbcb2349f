"""Host-side I/O placement for the per-round host buffers (e2e path).

Page-locked host memory is placed on the NUMA node of the thread that first
touches it. A buffer on the node far from the GPU's PCIe root crosses the
socket interconnect on every host->device copy, so the per-round dataset
upload (`lbbsp_mlp_load_data_async`) should read from memory on the GPU's
own node. `pinned_empty` allocates a page-locked tensor with the calling
thread temporarily bound to the GPU-local CPUs (read from sysfs), then
restores the previous affinity.
"""
import os

import torch


def _pci_bus_id(device):
    props = torch.cuda.get_device_properties(device)
    dom = getattr(props, "pci_domain_id", 0)
    return "%04x:%02x:%02x.0" % (dom, props.pci_bus_id, props.pci_device_id)


def _parse_cpulist(text):
    cpus = set()
    for part in text.strip().split(","):
        if not part:
            continue
        if "-" in part:
            a, b = part.split("-")
            cpus.update(range(int(a), int(b) + 1))
        else:
            cpus.add(int(part))
    return cpus


def gpu_local_cpus(device=0):
    """CPUs on the GPU's NUMA node that this process may run on (empty set if
    sysfs does not say)."""
    try:
        path = "/sys/bus/pci/devices/%s/local_cpulist" % _pci_bus_id(device)
        with open(path) as f:
            cpus = _parse_cpulist(f.read())
    except (OSError, ValueError, RuntimeError, AttributeError):
        return set()
    return cpus & os.sched_getaffinity(0)


def pinned_empty(shape, dtype, device=0):
    """torch.empty(shape, dtype, pin_memory=True) with its pages first-touched
    on the GPU's NUMA node."""
    local = gpu_local_cpus(device)
    prev = os.sched_getaffinity(0)
    if local:
        os.sched_setaffinity(0, local)
    try:
        t = torch.empty(shape, dtype=dtype, pin_memory=True)
        t.zero_()  # first touch happens here, on the local node
    finally:
        if local:
            os.sched_setaffinity(0, prev)
    return t
