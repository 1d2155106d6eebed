import sys, random
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2408_17063_b200 as P
from oracle import bgv_oracle as O
n = 8192
he = P.HeParams(n, 65537, 3)
be = P.B200BgvBackend(he, seed=0)
keys = be.keygen(*P.plan_rotation_amounts(8, n))
obe = O.OracleBgv(n, 65537, 3, seed=0)
okeys = obe.keygen(*O.plan_rotation_amounts(8, n))
params = P.CompressionParams(8192, 8, he)
rng = random.Random(0); dense = O.plant_sparse(rng, 8192, 8, 65537)
ct = P.encrypt_vector(dense, params, be, keys)[0]
oct_ = O.encrypt_vector(dense, 8192, obe, okeys)[0]
assert np.array_equal(ct.payload.res, oct_.c)
rows = np.random.default_rng(5).integers(0, 65537, (2, n//2)).astype(np.int64)
m = P.SlotMatrix(65537, rows)
cur, ocur = ct, oct_
for lvl in (3, 2, 1):
    for r in sorted(keys.rotation_keys):
        a = be.rot_row(cur, r, keys); b = obe.rot_row(ocur, r, okeys)
        bad = [(i, k, int((a.payload.res[i, k] != b.c[i, k]).sum())) for i in range(2) for k in range(lvl + 1)]
        bad = [x for x in bad if x[2]]
        print('level', lvl, 'r', r, 't', keys.rotation_keys[r][0], 'mismatch (poly,k,count):', bad, flush=True)
    a = be.rot_col(cur, keys); b = obe.rot_col(ocur, okeys)
    print('level', lvl, 'col', [(i, k, int((a.payload.res[i, k] != b.c[i, k]).sum())) for i in range(2) for k in range(lvl + 1)])
    cur = be.mul_plain(cur, m); ocur = obe.mul_plain(ocur, rows)
