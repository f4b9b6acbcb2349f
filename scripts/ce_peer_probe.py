"""Copy-engine peer bandwidth over NVLink (one process, 2 GPUs; debug probe).

Times a 33.5 MB / 134 MB bf16 device-to-peer copy (cudaMemcpyPeerAsync via
torch's copy_), alone and while a bf16 GEMM saturates the sending GPU's SMs,
to decide whether a copy-engine gradient exchange can overlap the backward.
"""
import torch


def t_ms(fn, stream, iters=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(iters):
        fn()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / iters


def main():
    assert torch.cuda.device_count() >= 2
    print("peer access 0->1:", torch.cuda.can_device_access_peer(0, 1))
    d0, d1 = torch.device("cuda", 0), torch.device("cuda", 1)
    for n in (4096 * 4096 + 4096, 4 * (4096 * 4096 + 4096)):
        a = torch.randn(n, device=d0, dtype=torch.bfloat16)
        b = torch.empty(n, device=d1, dtype=torch.bfloat16)
        cs = torch.cuda.Stream(d0)
        with torch.cuda.device(d0), torch.cuda.stream(cs):
            ms = t_ms(lambda: b.copy_(a, non_blocking=True), cs)
        print(f"CE copy {n * 2 / 1e6:.1f} MB alone: {ms:.3f} ms = {n * 2 / ms / 1e6:.0f} GB/s", flush=True)
        # split into 4 chunks on 4 streams (several copy engines?)
        streams = [torch.cuda.Stream(d0) for _ in range(4)]
        ch = n // 4

        def split():
            for i, st in enumerate(streams):
                with torch.cuda.stream(st):
                    b[i * ch:(i + 1) * ch].copy_(a[i * ch:(i + 1) * ch], non_blocking=True)
            for st in streams:
                cs.wait_stream(st)
            for st in streams:
                st.wait_stream(cs)
        with torch.cuda.device(d0), torch.cuda.stream(cs):
            ms = t_ms(split, cs)
        print(f"CE copy {n * 2 / 1e6:.1f} MB as 4 streams: {ms:.3f} ms = {n * 2 / ms / 1e6:.0f} GB/s", flush=True)
    # overlap with a GEMM on GPU 0
    x = torch.randn(8192, 4096, device=d0, dtype=torch.bfloat16)
    w = torch.randn(4096, 4096, device=d0, dtype=torch.bfloat16)
    gs = torch.cuda.Stream(d0)
    with torch.cuda.device(d0), torch.cuda.stream(gs):
        g_ms = t_ms(lambda: torch.mm(x, w), gs, iters=40)
    print(f"GEMM 8192x4096x4096 alone: {g_ms:.3f} ms", flush=True)
    n = 4 * (4096 * 4096 + 4096)
    a = torch.randn(n, device=d0, dtype=torch.bfloat16)
    b = torch.empty(n, device=d1, dtype=torch.bfloat16)
    cs = torch.cuda.Stream(d0)
    with torch.cuda.device(d0):
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        sc = torch.cuda.Event(enable_timing=True)
        ec = torch.cuda.Event(enable_timing=True)
        s.record(gs)
        with torch.cuda.stream(gs):
            for _ in range(40):
                torch.mm(x, w)
        e.record(gs)
        sc.record(cs)
        with torch.cuda.stream(cs):
            for _ in range(10):
                b.copy_(a, non_blocking=True)
        ec.record(cs)
        torch.cuda.synchronize()
        print(f"concurrent: GEMMs {s.elapsed_time(e) / 40:.3f} ms each, copies "
              f"{sc.elapsed_time(ec) / 10:.3f} ms each ({n * 2 / (sc.elapsed_time(ec) / 10) / 1e6:.0f} GB/s)",
              flush=True)


if __name__ == "__main__":
    main()
