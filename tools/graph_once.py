"""Warm Comp graph launches inside an NVTX range "comp" (for ncu --nvtx)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_17063_b200 as P
N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
p = 65537 if N < 65537 else 786433
he = P.HeParams(8192, p, 3); params = P.CompressionParams(N, s, he)
be = P.B200BgvBackend(he, seed=0, noise_guard=False)
keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
rng = np.random.default_rng(1); C = params.num_ciphertexts
cd = np.stack([np.stack([rng.integers(0, q, 8192, dtype=np.uint64) for q in be.q]) for _ in range(2 * C)]).reshape(C, 2, 4, 8192)
dc = P.DeviceComp(be, params, keys); dc.set_inputs(cd, cd.copy())
for _ in range(3): dc.launch()
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("comp")
dc.launch()
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("ok")
