"""Config 5 shape on one GPU: Q independent queries, each with its own seeded
key set (real keygen) and its own s-sparse payload, over N = 2^16, s = 64.
Every query has its own context (keys, plan, CUDA graph); their Comps run on
separate streams.  Reports aggregate compressed entries/s for 1, 2, 4, 8
concurrent queries and checks every query's output decrypts to its power sums.

  python tools/multi_query.py [--Q 8] [--N 65536] [--s 64] [--rounds 20]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--Q", type=int, default=8)
    ap.add_argument("--N", type=int, default=1 << 16)
    ap.add_argument("--s", type=int, default=64)
    ap.add_argument("--rounds", type=int, default=20)
    ap.add_argument("--oracle", type=int, default=0,
                    help="check the first K queries bit-exact against the CPU oracle (own keygen/encrypt/Comp per seed)")
    a = ap.parse_args()
    p = 65537 if a.N < 65537 else next(c for c in (786433, 1097729, 4423681) if c > a.N)
    he = P.HeParams(8192, p, 3)
    params = P.CompressionParams(a.N, a.s, he)
    qs = []
    t0 = time.perf_counter()
    for q in range(a.Q):
        be = P.B200BgvBackend(he, seed=q, noise_guard=False)
        keys = be.keygen(*P.plan_rotation_amounts(a.s, 8192))
        rng = random.Random(1000 + q)
        support = sorted(rng.sample(range(1, a.N + 1), a.s))
        dense = [0] * a.N
        for i in support:
            dense[i - 1] = rng.randrange(1, p)
        cd = P.encrypt_vector(dense, params, be, keys)
        cv = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
        dc = P.DeviceComp(be, params, keys)
        dc.set_inputs(np.stack([c.payload.res for c in cd]), np.stack([c.payload.res for c in cv]))
        qs.append(dict(be=be, keys=keys, dense=dense, dc=dc, stream=torch.cuda.Stream()))
    setup_s = time.perf_counter() - t0
    # correctness: every query decrypts to its own power sums
    for d in qs:
        d["dc"].launch(d["stream"].cuda_stream)
    torch.cuda.synchronize()
    ok = True
    for d in qs:
        out = d["dc"].output()
        be = d["be"]
        ct = P.Ciphertext(be.backend_id, d["keys"].key_id, 0, P.RnsPayload(out, 0.0, (be.q[0],)))
        m = be.decrypt(ct, d["keys"])
        w = [int(x) for x in m.rows[0][: a.s]]
        want = [sum(pow(i + 1, j + 1, p) for i, v in enumerate(d["dense"]) if v) % p for j in range(a.s)]
        ok &= w == want
    res = {"N": a.N, "s": a.s, "p": p, "queries": a.Q, "decrypt_ok": ok, "setup_s": round(setup_s, 1), "concurrency": {}}
    if a.oracle:
        from oracle import bgv_oracle as O

        exact = []
        for q, d in enumerate(qs[: a.oracle]):
            obe = O.OracleBgv(8192, p, 3, seed=q, check_noise=False)
            okeys = obe.keygen(*O.plan_rotation_amounts(a.s, 8192))
            ocd = O.encrypt_vector(d["dense"], a.N, obe, okeys)
            ocv = O.encrypt_vector([1 if x else 0 for x in d["dense"]], a.N, obe, okeys)
            oout = O.comp(ocd, a.N, a.s, obe, okeys, ocv)
            exact.append(bool(np.array_equal(d["dc"].output(), oout.c)))
            print(f"query {q}: GPU Comp == oracle Comp: {exact[-1]}", flush=True)
        res["oracle_bit_exact"] = exact
        ok &= all(exact)
    for conc in (1, 2, 4, 8):
        if conc > a.Q:
            break
        active = qs[:conc]
        for _ in range(3):
            for d in active:
                d["dc"].launch(d["stream"].cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream()
        e0.record(main)
        for d in active:
            d["stream"].wait_event(e0)
        for _ in range(a.rounds):
            for d in active:
                d["dc"].launch(d["stream"].cuda_stream)
        for d in active:
            ev = torch.cuda.Event()
            ev.record(d["stream"])
            main.wait_event(ev)
        e1.record(main)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        comps = conc * a.rounds
        res["concurrency"][conc] = {
            "ms_per_comp": ms / comps,
            "aggregate_entries_per_s": comps * a.N / (ms * 1e-3),
        }
        print(f"concurrent queries {conc}: {ms / comps:.3f} ms/Comp amortised, "
              f"{comps * a.N / (ms * 1e-3) / 1e6:.1f} M entries/s aggregate", flush=True)
    print(json.dumps(res))
    if not ok:
        sys.exit(1)


if __name__ == "__main__":
    main()
