import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
L = _lib.lib()
for N, s in ((16384, 16), (8192, 8), (32768, 16)):
    he = P.HeParams(8192, 65537, 3); params = P.CompressionParams(N, s, he)
    be = P.B200BgvBackend(he, seed=0, noise_guard=False)
    keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
    rng = np.random.default_rng(1); C = params.num_ciphertexts
    qs = np.array(be.q, dtype=np.uint64).reshape(1, 1, 4, 1)
    cd = (rng.integers(0, 2**63, (C, 2, 4, 8192), dtype=np.uint64) % qs).astype(np.uint64)
    for thr in (0, 16, 32, 48, 64, 100, 150):
        L.hc_set_cluster_threshold(thr)
        be._planned = None
        dc = P.DeviceComp(be, params, keys); dc.set_inputs(cd, cd)
        for _ in range(3): dc.launch()
        torch.cuda.synchronize()
        st = torch.cuda.Stream(); e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(50): dc.launch(st.cuda_stream)
        e1.record(st); torch.cuda.synchronize()
        print(f"N={N} s={s} cluster<= {thr:4d}: {e0.elapsed_time(e1)/50:.4f} ms", flush=True)
L.hc_set_cluster_threshold(48)
