"""One device-resident Comp (keygen, plan/graph capture, one graph launch,
output read) for compute-sanitizer runs:

  compute-sanitizer --tool {memcheck,racecheck,synccheck} python tools/sanitize_comp.py N s

Inputs are random level-3 residues (the kernels' memory behaviour does not
depend on the values); exits non-zero if the output is not reproducible."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2408_17063_b200 as P

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
s = int(sys.argv[2]) if len(sys.argv) > 2 else 16
p = 65537 if N < 65537 else next(c for c in (786433, 1097729, 4423681) if c > N)
he = P.HeParams(8192, p, 3)
params = P.CompressionParams(N, s, he)
be = P.B200BgvBackend(he, seed=0, noise_guard=False)
keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
rng = np.random.default_rng(1)
C = params.num_ciphertexts
qs = np.array(be.q, dtype=np.uint64).reshape(1, 1, 4, 1)
cd = (rng.integers(0, 2**63, (C, 2, 4, 8192), dtype=np.uint64) % qs).astype(np.uint64)
cv = (rng.integers(0, 2**63, (C, 2, 4, 8192), dtype=np.uint64) % qs).astype(np.uint64)
dc = P.DeviceComp(be, params, keys)
dc.set_inputs(cd, cv)
dc.launch()
o1 = dc.output()
dc.launch()
o2 = dc.output()
torch.cuda.synchronize()
assert np.array_equal(o1, o2), "graph replay not reproducible"
print(f"sanitize_comp N={N} s={s}: ok", flush=True)
