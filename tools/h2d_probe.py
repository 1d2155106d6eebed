"""Pinned host->device copy bandwidth for the headline's e2e input volume
(2 MiB: cd and cv, C=2 ciphertexts each) split over 1, 2 or 4 copies on one
stream, and over 2 / 4 concurrent streams (copy engines)."""
import torch

MB = 1 << 20
x = torch.empty(2 * MB, dtype=torch.uint8).pin_memory()
y = torch.empty(2 * MB, dtype=torch.uint8, device="cuda")
main = torch.cuda.Stream()
side = [torch.cuda.Stream() for _ in range(4)]


def run(parts, nstreams):
    sz = (2 * MB) // parts
    ev0 = torch.cuda.Event()
    ev0.record(main)
    for i in range(parts):
        st = side[i % nstreams] if nstreams > 1 else main
        if nstreams > 1:
            st.wait_event(ev0)
        with torch.cuda.stream(st):
            y[i * sz:(i + 1) * sz].copy_(x[i * sz:(i + 1) * sz], non_blocking=True)
    if nstreams > 1:
        for st in side[:nstreams]:
            e = torch.cuda.Event()
            e.record(st)
            main.wait_event(e)


for parts, ns in ((1, 1), (2, 1), (4, 1), (2, 2), (4, 2), (4, 4), (8, 4)):
    for _ in range(5):
        run(parts, ns)
    torch.cuda.synchronize()
    ts = []
    for _ in range(30):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(main)
        run(parts, ns)
        b.record(main)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    med = ts[len(ts) // 2]
    print(f"2 MiB H2D as {parts} copies on {ns} stream(s): median {med * 1e3:.1f} us = {2 * MB / (med * 1e-3) / 1e9:.1f} GB/s", flush=True)
