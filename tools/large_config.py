"""Config 4: large Comp, N in {2^20, 2^22}, s in {16, 128}.

Real keygen and encryption of the seeded sparse payload, one Comp through
the package API (`comp`), the decrypted (w, e) slots checked against the
power sums of the planted pairs (what the reference's decomp inverts,
compress.py:1-16), then warm device-resident timing (`DeviceComp`).

With --oracle the CPU oracle (oracle/, C + OpenMP restatement of the
reference Comp) runs the same seed end to end and the answer must be
bit-exact (ciphertext residues and serialized bytes).

  python tools/large_config.py --N 1048576 --s 16 [--iters 5] [--oracle] [--json out.json]
"""
import argparse
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

import paper_2408_17063_b200 as P
from paper_2408_17063_b200.compress import DeviceComp, _stack_level3


def plant(N, s, p, seed):
    rng = random.Random(seed)
    support = sorted(rng.sample(range(1, N + 1), s))
    d = [0] * N
    for i in support:
        d[i - 1] = rng.randrange(1, p)
    return d


def power_sums(dense, s, p):
    w = [0] * s
    e = [0] * s
    nz = [(i, v) for i, v in enumerate(dense, start=1) if v]
    for i, v in nz:
        pw = i % p
        for j in range(s):
            w[j] = (w[j] + pw) % p
            e[j] = (e[j] + pw * v) % p
            pw = pw * i % p
    return w, e


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=1 << 20)
    ap.add_argument("--s", type=int, default=16)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--json", default="")
    ap.add_argument("--oracle", action="store_true",
                    help="also run the CPU oracle (oracle/, C + OpenMP) on the same seed and require a bit-exact answer")
    a = ap.parse_args()
    p = 65537 if a.N < 65537 else next(c for c in (786433, 1097729, 4423681) if c > a.N)
    t0 = time.perf_counter()
    he = P.HeParams(8192, p, 3)
    params = P.CompressionParams(a.N, a.s, he)
    be = P.B200BgvBackend(he, seed=a.seed, noise_guard=False)  # past the heuristic bound
    keys = be.keygen(*P.plan_rotation_amounts(a.s, 8192))
    t1 = time.perf_counter()
    dense = plant(a.N, a.s, p, a.seed)
    cd = P.encrypt_vector(dense, params, be, keys)
    cv = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
    t2 = time.perf_counter()
    ans = P.comp(cd, params, be, keys, index_hint=cv)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    w, e = ans.payload_slots(be, keys)
    ok = (w, e) == power_sums(dense, a.s, p)
    dc = DeviceComp(be, params, keys)
    dc.set_inputs(_stack_level3(cd, 3), _stack_level3(cv, 3))
    dc.launch()
    torch.cuda.synchronize()
    same = np.array_equal(dc.output(), ans.cts[0].payload.res)
    st = torch.cuda.Stream()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ms = []
    for _ in range(a.iters):
        torch.cuda.synchronize()
        ev[0].record(st)
        dc.launch(st.cuda_stream)
        ev[1].record(st)
        torch.cuda.synchronize()
        ms.append(ev[0].elapsed_time(ev[1]))
    ms.sort()
    med = ms[len(ms) // 2]
    oracle_ok = None
    if a.oracle:
        sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
        from oracle import bgv_oracle as O

        t4 = time.perf_counter()
        obe = O.OracleBgv(8192, p, 3, seed=a.seed, check_noise=False)
        okeys = obe.keygen(*O.plan_rotation_amounts(a.s, 8192))
        ocd = O.encrypt_vector(dense, a.N, obe, okeys)
        ocv = O.encrypt_vector([1 if x else 0 for x in dense], a.N, obe, okeys)
        oout = O.comp(ocd, a.N, a.s, obe, okeys, ocv)
        oracle_s = time.perf_counter() - t4
        oracle_ok = bool(np.array_equal(ans.cts[0].payload.res, oout.c))
        oracle_ser = O.sha256(O.serialize_answer(obe, oout, a.s))
        gpu_ser = O.sha256(ans.serialize(be))
    r = {
        "N": a.N, "s": a.s, "p": p, "blocks": params.num_blocks, "ciphertexts": params.num_ciphertexts,
        "decomp_slots_match": ok, "device_rerun_identical": bool(same),
        "comp_ms_median": med, "comp_ms_min": ms[0], "entries_per_s": a.N / (med * 1e-3),
        "first_call_s": t3 - t2, "keygen_s": t1 - t0, "encrypt_s": t2 - t1,
    }
    if a.oracle:
        r.update({"oracle_bit_exact": oracle_ok, "answer_sha256_gpu": gpu_ser, "answer_sha256_oracle": oracle_ser,
                  "oracle_keygen_encrypt_comp_s": oracle_s, "oracle_threads": O.lib().orc_num_threads()})
        ok = ok and oracle_ok and gpu_ser == oracle_ser
    print(json.dumps(r))
    if a.json:
        with open(a.json, "a") as f:
            f.write(json.dumps(r) + "\n")
    if not (ok and same):
        sys.exit(1)


if __name__ == "__main__":
    main()
