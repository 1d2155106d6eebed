import torch, time
x = torch.empty(2 << 20, dtype=torch.uint8).pin_memory()
y = torch.empty(2 << 20, dtype=torch.uint8, device="cuda")
o = torch.empty(128 << 10, dtype=torch.uint8).pin_memory()
z = torch.empty(128 << 10, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for name, fn in (("h2d 2MB x1", lambda: y.copy_(x, non_blocking=True)),
                 ("h2d 1MB x2", lambda: (y[:1 << 20].copy_(x[:1 << 20], non_blocking=True), y[1 << 20:].copy_(x[1 << 20:], non_blocking=True))),
                 ("d2h 128KB", lambda: o.copy_(z, non_blocking=True))):
    with torch.cuda.stream(s):
        for _ in range(5): fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(20)]
        for a, b in ev:
            a.record(s); fn(); b.record(s)
        torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) for a, b in ev)
    print(name, f"median {ts[10]*1e3:.1f} us")
