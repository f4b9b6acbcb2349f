"""Host-side I/O placement for the per-round host buffers (e2e path).

Page-locked host memory is placed on the NUMA node of the thread that first
touches it. A buffer on the node far from the GPU's PCIe root crosses the
socket interconnect on every host->device copy, so the per-round dataset
upload (`lbbsp_mlp_load_data_async`) should read from memory on the GPU's
own node. `pinned_empty` allocates a page-locked tensor with the calling
thread temporarily bound to the GPU-local CPUs (read from sysfs), then
restores the previous affinity.

The pages are 2 MB transparent huge pages where the kernel grants them: a
2 MB-aligned anonymous mapping, madvise(MADV_HUGEPAGE), first-touched on
the local node and page-locked with cudaHostRegister. DMA out of 4 KB-page
pinned memory (torch pin_memory) needs one IOMMU translation per 4 KB and
ran the 1.57 MB C2 upload at 12-28 GB/s for its first ~1000-3000 copies on
this pool's boxes, against 45 GB/s from the first copy out of huge pages
(profiles/r02_h2d_hugepages.txt, scripts/h2d_hugepage_probe.py). Without
THP support it falls back to torch's pin_memory. Huge-page buffers stay
mapped and registered for the life of the process.
"""
import ctypes
import mmap
import os

import torch

_HUGE = 2 << 20
_keep = []  # (mapping, ctypes view) of every huge-page buffer: process lifetime


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


def _huge_pinned(nbytes):
    """a zeroed, page-locked, 2 MB-aligned THP mapping of >= nbytes (uint8
    tensor), or None when THP or the registration is unavailable"""
    if not hasattr(mmap, "MADV_HUGEPAGE") or not torch.cuda.is_available():
        return None
    size = (max(nbytes, 1) + _HUGE - 1) // _HUGE * _HUGE
    mm = mmap.mmap(-1, size + _HUGE, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    base = ctypes.addressof(ctypes.c_char.from_buffer(mm))
    off = (-base) % _HUGE
    try:
        mm.madvise(mmap.MADV_HUGEPAGE, off, size)
    except (OSError, ValueError):
        mm.close()
        return None
    view = (ctypes.c_char * size).from_buffer(mm, off)
    ctypes.memset(view, 0, size)  # first touch (the caller's CPU binding applies)
    if int(torch.cuda.cudart().cudaHostRegister(base + off, size, 0)) != 0:
        del view
        mm.close()
        return None
    _keep.append((mm, view))
    return torch.frombuffer(view, dtype=torch.uint8, count=nbytes)


def pinned_empty(shape, dtype, device=0, huge_pages=True):
    """A zeroed page-locked host tensor whose pages are first-touched on the
    GPU's NUMA node: 2 MB huge pages registered with cudaHostRegister when
    available (huge_pages), else torch.empty(..., pin_memory=True)."""
    local = gpu_local_cpus(device)
    prev = os.sched_getaffinity(0)
    if local:
        os.sched_setaffinity(0, local)
    try:
        t = None
        if huge_pages:
            numel = 1
            for d in shape:
                numel *= int(d)
            nbytes = numel * torch.empty((), dtype=dtype).element_size()
            raw = _huge_pinned(nbytes)
            if raw is not None:
                t = raw.view(dtype).reshape(tuple(int(d) for d in shape))
        if t is None:
            t = torch.empty(shape, dtype=dtype, pin_memory=True)
            t.zero_()  # first touch happens here, on the local node
    finally:
        if local:
            os.sched_setaffinity(0, prev)
    return t
