"""Mask + Comp (pdq.answer after Match) on the 5-prime chain:
wall time of each stage through the package API (host buffers in and out,
synchronous calls), next to the fused level-3 Comp at the same (N, s).

  python tools/answer_bench.py [--N 8192] [--s 8] [--iters 5]
"""
import argparse
import ctypes
import json
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_17063_b200 as P  # noqa: E402
from oracle import bgv_oracle as O  # noqa: E402  (payload recipe + expected slots only)


def med(f, iters):
    ts = []
    out = None
    for _ in range(iters):
        t0 = time.perf_counter()
        out = f()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2] * 1e3, out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--N", type=int, default=8192)
    ap.add_argument("--s", type=int, default=8)
    ap.add_argument("--iters", type=int, default=5)
    a = ap.parse_args()
    N, s, p, seed = a.N, a.s, 65537, 6
    he = P.HeParams(8192, p, 4)
    params = P.CompressionParams(N, s, he)
    # noise guard off (as the oracle's guard-disabled goldens): the reference's
    # heuristic bound trips from s = 32 at these levels; values never depend on it
    be = P.B200BgvBackend(he, seed=seed, noise_guard=False)
    keys = be.keygen(*P.plan_rotation_amounts(s, 8192))
    support, db, dense = O.masked_payload(N, s, p, seed)
    hint = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
    P.answer_from_match(hint, db, params, be, keys)  # warm: plan + graph capture
    t_mask, cd = med(lambda: P.mask(hint, db, params, be, keys), a.iters)
    t_comp, ans = med(lambda: P.comp(cd, params, be, keys, index_hint=hint), a.iters)
    t_ans, ans2 = med(lambda: P.answer_from_match(hint, db, params, be, keys), a.iters)
    assert ans.payload_slots(be, keys) == O.expected_slots(dense, s, p)
    # the packed-input BSGS graph alone (device part of the glue path)
    import numpy as np
    from paper_2408_17063_b200 import _lib
    from paper_2408_17063_b200.compress import _pack_pair_ops

    t_pack, u = med(lambda: _pack_pair_ops(hint, cd, params, be, keys), a.iters)
    u_arr = np.ascontiguousarray(np.stack([c.payload.res for c in u]), dtype=np.uint64)
    out = np.empty((2, 1, 8192), dtype=np.uint64)
    L = _lib.lib(4)
    t_bsgs, _ = med(lambda: _lib.check(L.hc_comp_packed(be._ctx(), _lib.ptr(u_arr), len(u), _lib.ptr(out))), a.iters)
    # the fused level-3 Comp at the same point (4-prime chain)
    he3 = P.HeParams(8192, p, 3)
    be3 = P.B200BgvBackend(he3, seed=seed, noise_guard=False)
    k3 = be3.keygen(*P.plan_rotation_amounts(s, 8192))
    d3 = O.plant_sparse(random.Random(seed), N, s, p)
    c3 = P.encrypt_vector(d3, P.CompressionParams(N, s, he3), be3, k3)
    h3 = P.encrypt_vector([1 if x else 0 for x in d3], P.CompressionParams(N, s, he3), be3, k3)
    P.comp(c3, P.CompressionParams(N, s, he3), be3, k3, index_hint=h3)
    t_fused, _ = med(lambda: P.comp(c3, P.CompressionParams(N, s, he3), be3, k3, index_hint=h3), a.iters)
    # device-resident: the answer graph (Mask + pack_pair + BSGS) replayed on one
    # stream, CUDA events around each launch, L2 flushed in between (untimed)
    import torch

    P.answer_from_match(hint, db, params, be, keys)
    st = torch.cuda.Stream()
    flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    dev = []
    with torch.cuda.stream(st):
        for i in range(a.iters + 3):
            flush.fill_(i)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            _lib.check(L.hc_mixed_launch(be._ctx(), ctypes.c_void_p(st.cuda_stream)))
            e1.record(st)
            st.synchronize()
            if i >= 3:
                dev.append(e0.elapsed_time(e1))
    dev.sort()
    t_dev = dev[len(dev) // 2]
    out_dev = np.empty((2, 1, 8192), dtype=np.uint64)
    _lib.check(L.hc_comp_get_output(be._ctx(), _lib.ptr(out_dev)))
    assert np.array_equal(out_dev, ans2.cts[0].payload.res)
    print(json.dumps({
        "workload": f"answer after Match: mask + comp, N={N} s={s} max_level=4 (cv level 4, cd level 3)",
        "ms": {"mask": round(t_mask, 3), "comp_mixed": round(t_comp, 3), "answer_from_match": round(t_ans, 3),
               "pack_pair_single_ops": round(t_pack, 3), "bsgs_graph_from_u (hc_comp_packed)": round(t_bsgs, 3),
               "fused_comp_level3_same_point": round(t_fused, 3),
               "answer_graph_device_resident (CUDA events, L2 flushed)": round(t_dev, 4)},
        "entries_per_s_answer": round(N / (t_ans / 1e3), 1),
        "entries_per_s_answer_device": round(N / (t_dev / 1e3), 1),
        "note": "wall clock, synchronous API calls with host buffers (H2D/D2H inside), median of iters",
    }))


if __name__ == "__main__":
    main()
