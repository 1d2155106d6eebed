"""Device-resident Comp latency (warm, or median with L2 flushed: --flush) over (N, s) points with random level-3
residues as inputs (timing only; parity is covered by tests/ and
tools/large_config.py).  usage: python tools/sweep.py N:s [N:s ...] [--lanes K]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib

args = [a for a in sys.argv[1:] if ":" in a]
cbs = [int(x) for x in sys.argv[sys.argv.index("--cb") + 1].split(",")] if "--cb" in sys.argv else [0]
vts = [int(x) for x in sys.argv[sys.argv.index("--vt2") + 1].split(",")] if "--vt2" in sys.argv else [0]
lanes = [int(x) for x in sys.argv[sys.argv.index("--lanes") + 1].split(",")] if "--lanes" in sys.argv else [4]
keys_cache = {}
for pt in args:
    N, s = (int(x) for x in pt.split(":"))
    p = 65537 if N < 65537 else next(c for c in (786433, 1097729, 4423681) if c > N)
    he = P.HeParams(8192, p, 3)
    params = P.CompressionParams(N, s, he)
    if (p, s) not in keys_cache:
        be = P.B200BgvBackend(he, seed=0, noise_guard=False)
        keys_cache[(p, s)] = (be, be.keygen(*P.plan_rotation_amounts(s, 8192)))
    be, keys = keys_cache[(p, s)]
    rng = np.random.default_rng(1)
    C = params.num_ciphertexts
    qs = np.array(be.q, dtype=np.uint64).reshape(1, 1, 4, 1)
    cd = (rng.integers(0, 2**63, (C, 2, 4, 8192), dtype=np.uint64) % qs).astype(np.uint64)
    cv = (rng.integers(0, 2**63, (C, 2, 4, 8192), dtype=np.uint64) % qs).astype(np.uint64)
    for ln, cb, vt in [(a, b, c) for a in lanes for b in cbs for c in vts]:
        _lib.lib().hc_set_lane_blocks(ln)
        if vt:
            _lib.lib().hc_set_vt2_jobs(vt)
        be._planned = None  # force a re-plan with this setting
        dc = P.DeviceComp(be, params, keys, chunk_blocks=cb)
        dc.set_inputs(cd, cv)
        for _ in range(3):
            dc.launch()
        torch.cuda.synchronize()
        iters = int(os.environ.get("SWEEP_ITERS", "0")) or max(3, min(50, int(2000 / max(1, N >> 14))))
        st = torch.cuda.Stream()
        if "--flush" in sys.argv:  # L2 flushed (256 MiB write) before every timed Comp, as bench.py
            flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(iters)]
            with torch.cuda.stream(st):
                for a, b in evs:
                    flush.zero_()
                    a.record(st)
                    dc.launch(st.cuda_stream)
                    b.record(st)
            torch.cuda.synchronize()
            ms = sorted(a.elapsed_time(b) for a, b in evs)[iters // 2]
        else:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(iters):
                dc.launch(st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / iters
        print(f"N={N:8d} s={s:4d} cb={cb:3d} vt2>={vt:10d} lanes<={ln:5d} blocks={params.num_blocks:5d}  {ms:9.3f} ms  {N/ms/1e3:8.1f} M entries/s", flush=True)
_lib.lib().hc_set_lane_blocks(4)
