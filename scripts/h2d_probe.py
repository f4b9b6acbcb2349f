"""Host->device copy bandwidth of page-locked buffers: tensor.pin_memory() vs
torch.empty(pin_memory=True), and the PCIe link state (debug helper)."""
import torch, ctypes

def bw(nbytes, pinned_kind="torch", reps=20, chunks=1):
    n = nbytes // 2
    if pinned_kind == "torch":
        x = torch.empty(n, dtype=torch.bfloat16).pin_memory()
    else:
        x = torch.empty(n, dtype=torch.bfloat16, pin_memory=True)
    dx = torch.empty(n, dtype=torch.bfloat16, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(chunks)]
    for _ in range(3): dx.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
    s.record()
    cs = n // chunks
    for _ in range(reps):
        if chunks == 1:
            dx.copy_(x, non_blocking=True)
        else:
            for i, st in enumerate(streams):
                st.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(st):
                    dx[i*cs:(i+1)*cs].copy_(x[i*cs:(i+1)*cs], non_blocking=True)
            for st in streams: torch.cuda.current_stream().wait_stream(st)
    e.record(); e.synchronize()
    t = s.elapsed_time(e) / reps * 1e3
    print(f"{nbytes/1e6:8.2f} MB {pinned_kind:6s} chunks={chunks}: {t:8.1f} us  {nbytes/t/1e3:6.1f} GB/s", flush=True)
for nb in (1568000, 16 << 20, 64 << 20):
    bw(nb)
bw(1568000, "alloc")
bw(1568000, chunks=4)
import subprocess
print(subprocess.run(["nvidia-smi", "--query-gpu=pcie.link.gen.current,pcie.link.width.current,pcie.link.gen.max", "--format=csv"], capture_output=True, text=True).stdout)
