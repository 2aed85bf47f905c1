"""Dev tool: host->device copy rate from pinned memory with 1, 2, 4 concurrent
copy streams (does one cudaMemcpyAsync saturate the host link?)."""
import torch

GB = 4
n = GB << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h.fill_(1)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for k in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(k)]
    best = 1e9
    for rep in range(4):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for s in streams:
            s.wait_event(a)
        part = n // k
        ends = []
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * part:(i + 1) * part].copy_(h[i * part:(i + 1) * part], non_blocking=True)
                e = torch.cuda.Event()
                e.record()
                ends.append(e)
        for e in ends:
            torch.cuda.current_stream().wait_event(e)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b)
        if rep:
            best = min(best, ms)
    print(f"streams={k}: {n / best / 1e6:.1f} GB/s")
