"""Keygen + encryption time with the native random.Random restatement."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_17063_b200 as P
for N, s in ((1 << 14, 16), (1 << 16, 64)):
    he = P.HeParams(8192, 65537, 3)
    params = P.CompressionParams(N, s, he)
    be = P.B200BgvBackend(he, seed=3, noise_guard=False)
    t0 = time.perf_counter()
    keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
    t1 = time.perf_counter()
    cts = P.encrypt_vector([0] * N, params, be, keys)
    t2 = time.perf_counter()
    print(f"N={N} s={s}: keygen {t1 - t0:.2f} s ({len(keys.rotation_keys) + 1} rotation keys), encrypt {params.num_ciphertexts} cts {t2 - t1:.2f} s")
