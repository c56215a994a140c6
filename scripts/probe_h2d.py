"""Probe: pinned H2D bandwidth of one 64 MiB copy split over 1/2/4 copy streams."""
import torch

n = 64 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        evs = []
        for i, st in enumerate(streams):
            st.wait_event(e0)
            with torch.cuda.stream(st):
                sl = slice(i * n // ns, (i + 1) * n // ns)
                d[sl].copy_(h[sl], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(st)
                evs.append(ev)
        for ev in evs:
            torch.cuda.current_stream().wait_event(ev)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        if rep == 2:
            print(f"streams={ns}: {ms:.3f} ms, {n / ms / 1e6:.1f} GB/s")
