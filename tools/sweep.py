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
        if "--profile" in sys.argv:  # un-graphed, event-timed launch table (hc_comp_profile_ex)
            sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
            from bench import STEP_KINDS, kernel_name
            mx = 4096
            sm_, sk, sj, tg = (np.zeros(mx, dtype=t) for t in (np.float32, np.int32, np.int32, np.int32))
            ns = _lib.lib().hc_comp_profile_ex(be._ctx(), st.cuda_stream, mx, _lib.ptr(sm_), _lib.ptr(sk), _lib.ptr(sj), _lib.ptr(tg))
            agg = {}
            for i in range(ns):
                nm = kernel_name(int(tg[i])) if int(sk[i]) == 0 else STEP_KINDS.get(int(sk[i]), str(sk[i]))
                a = agg.setdefault(nm, [0.0, 0, 0]); a[0] += float(sm_[i]); a[1] += int(sj[i]); a[2] += 1
                if "--launches" in sys.argv:
                    print(f"  {i:4d} {nm:34s} jobs {int(sj[i]):6d} {float(sm_[i])*1e3:9.1f} us")
            for nm, (t, j, l) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
                extra = f" {j*53248/(t*1e-3)/1e9:7.1f} Gbfly/s" if nm.startswith("k_xf") else ""
                print(f"  {nm:34s} launches {l:4d} jobs {j:7d} {t*1e3:9.1f} us{extra}")
        import hashlib
        sha = hashlib.sha256(np.ascontiguousarray(dc.output()).tobytes()).hexdigest()[:12]  # A/B builds/switches must agree
        print(f"N={N:8d} s={s:4d} cb={cb:3d} vt2>={vt:10d} lanes<={ln:5d} blocks={params.num_blocks:5d}  {ms:9.3f} ms  {N/ms/1e3:8.1f} M entries/s  out {sha}", flush=True)
_lib.lib().hc_set_lane_blocks(4)
