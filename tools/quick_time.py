import sys, time, random
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2408_17063_b200 as P
from oracle import bgv_oracle as O
N, s = 16384, 16
he = P.HeParams(8192, 65537, 3); params = P.CompressionParams(N, s, he)
t = time.time(); be = P.B200BgvBackend(he, seed=0); keys = be.keygen(*P.plan_rotation_amounts(s, 8192)); print('keygen', time.time()-t, flush=True)
rng = random.Random(0); dense = O.plant_sparse(rng, N, s, 65537)
cts = P.encrypt_vector(dense, params, be, keys); hint = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
dc = P.DeviceComp(be, params, keys)
print(be.plan_info())
cd = np.stack([c.payload.res for c in cts]); cv = np.stack([c.payload.res for c in hint])
dc.set_inputs(cd, cv)
for _ in range(3): dc.launch()
torch.cuda.synchronize()
s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
K = 20
torch.cuda.synchronize(); t0 = time.perf_counter()
for _ in range(K): dc.launch()
torch.cuda.synchronize(); t1 = time.perf_counter()
print('comp ms (wall, avg of %d, default ctx stream)' % K, (t1-t0)/K*1e3)
print(be.plan_info())
