"""TEST INFRASTRUCTURE ONLY -- generate tests/golden/*.json by running the
read-only Python REFERENCE (imported with the gmpy2 stand-in, see
oracle/refimport.py) in the build container.  The GPU box has no
/root/reference; the fixtures travel instead.

For each case the reference runs exactly the bench.run_point recipe
(bench.py:72-94): BgvBackend(HeParams(n, p, 3), seed), keygen over
plan_rotation_amounts, a sparse payload planted with random.Random(seed)
(bench.py:65-69), encrypt d then the index hint, then the timed
`comp(..., index_hint=hint)`.  Recorded: SHA-256 of the serialized
CompressedAnswer, decrypted (w, e), final noise_bits, Comp's counter
deltas, key_id, and SHA-256 digests of the key material and input
ciphertexts in RNS residue form (pins the oracle's keygen/encrypt).

Small-ring cases (n=64) also store every residue (inputs, keys, output) so
the oracle can be checked without regenerating anything.

Usage:  python oracle/make_golden.py [case-name ...]
"""

from __future__ import annotations

import hashlib
import json
import os
import random
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
sys.path.insert(0, ROOT)

from oracle import refimport  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")

# name: (n, p, N, s, seed, guard_disabled)
CASES = {
    "small_n64_N200_s5": (64, 257, 200, 5, 11, True),
    "small_n64_N64_s8": (64, 257, 64, 8, 12, True),
    "c1_N8192_s8": (8192, 65537, 8192, 8, 0, False),
    "c3_N8192_s16": (8192, 65537, 8192, 16, 1, False),
    "c2_N16384_s16": (8192, 65537, 16384, 16, 0, False),
    "odd_N10000_s5": (8192, 65537, 10000, 5, 3, True),
    "c2_N16384_s32": (8192, 65537, 16384, 32, 0, True),
    # round 2: the rest of config 2's sparsity sweep (baby = 4 / 8 / 16 in the
    # latency schedule) and config 3's N = 2^15, 2^16 points
    "c2_N16384_s8": (8192, 65537, 16384, 8, 0, False),
    "c2_N16384_s64": (8192, 65537, 16384, 64, 0, True),
    "c2_N16384_s128": (8192, 65537, 16384, 128, 0, True),
    "c3_N32768_s16": (8192, 65537, 32768, 16, 0, True),
    "c3_N65536_s16": (8192, 65537, 65536, 16, 0, True),
    # comp_masked (compress.py:521-530): cleartext DB on every position,
    # encrypted 0/1 index vector on the support (masked_payload below)
    "masked_small_n64_N200_s5": (64, 257, 200, 5, 13, True),
    "masked_c1_N8192_s8": (8192, 65537, 8192, 8, 4, False),
    "masked_c2_N16384_s16": (8192, 65537, 16384, 16, 5, False),
    # Mask + Comp (pdq.answer after Match, pdq.py:238-256) on a 5-prime chain
    # (max_level 4): cv = encrypted 0/1 index vector at level 4, cd =
    # pdq.mask(cv, db) at level 3, then comp(cd, index_hint=cv) -- mixed input
    # levels, reconciled by add's _at_level (bgv.py:656-658)
    "answer_small_n64_N200_s5": (64, 257, 200, 5, 14, True),
    "answer_c1_N8192_s8": (8192, 65537, 8192, 8, 6, False),
    "answer_c2_N16384_s16": (8192, 65537, 16384, 16, 7, False),
    # answer() on the protocol's own chain: max_level = pdq.protocol_max_level(p)
    # = 21 (pdq.py:181-184; Match's depth 17 + mask + 3), 22 primes.  The index
    # vector is encrypted at level 21 and brought to level 4 -- where Match
    # leaves it -- by the backend's own _at_level (bgv.py:610-614), then
    # pdq.mask and comp run exactly as in pdq.answer (pdq.py:248-256)
    "answer_deep_c1_N8192_s8": (8192, 65537, 8192, 8, 8, False),
}

# max_level per case (default 3, the BASELINE chain)
MAX_LEVEL = {"answer_small_n64_N200_s5": 4, "answer_c1_N8192_s8": 4, "answer_c2_N16384_s16": 4,
             "answer_deep_c1_N8192_s8": 21}
# level the index vector enters Mask at (Match's output level on the protocol chain)
ANSWER_LEVEL = {"answer_deep_c1_N8192_s8": 4}


def masked_payload(N, s, p, seed):
    """support = sorted(rng.sample(range(1, N+1), s)); db[i] = rng.randrange(1, p)
    for every position i (the server's cleartext database)."""
    rng = random.Random(seed)
    support = sorted(rng.sample(range(1, N + 1), s))
    db = [rng.randrange(1, p) for _ in range(N)]
    return support, db


def residues_of(vals, primes_rns):
    return np.array([[int(v) % q for v in vals] for q in primes_rns], dtype=np.uint64)


def digest_arrays(arrs) -> str:
    h = hashlib.sha256()
    for a in arrs:
        h.update(np.ascontiguousarray(a, dtype=np.uint64).tobytes())
    return h.hexdigest()


def keys_residues(be, keys):
    """Key material in RNS order: pk_b, pk_a, relin pairs, rotation keys by
    amount, col-swap key; each ring element [L+1][n]."""
    L = be.params.max_level
    primes = [be.chain.level_prime(k) for k in range(L + 1)]
    out = [residues_of(keys.public.pk_b, primes), residues_of(keys.public.pk_a, primes)]

    def ksk(k):
        for b, a in k.pairs:
            out.append(residues_of(b, primes))
            out.append(residues_of(a, primes))

    ksk(keys.relin_key)
    for r in sorted(keys.rotation_keys):
        ksk(keys.rotation_keys[r][1])
    if keys.col_swap_key is not None:
        ksk(keys.col_swap_key[1])
    return out


def keys_residues_low(be, keys, levels=4, digits=14):
    primes = [be.chain.level_prime(k) for k in range(levels)]
    out = []

    def ksk(k):
        for b, a in k.pairs[:digits]:
            out.append(residues_of(b, primes))
            out.append(residues_of(a, primes))

    for r in sorted(keys.rotation_keys):
        ksk(keys.rotation_keys[r][1])
    if keys.col_swap_key is not None:
        ksk(keys.col_swap_key[1])
    return out


def ct_residues(be, c):
    primes = [be.chain.level_prime(k) for k in range(c.level + 1)]
    return np.stack([residues_of(c.payload.c0, primes), residues_of(c.payload.c1, primes)])


def run_case(name):
    n, p, N, s, seed, guard_off = CASES[name]
    hc = refimport.load()
    from hcpdq.bgv import BgvBackend
    from hcpdq.compress import (
        CompressionParams,
        comp,
        comp_masked,
        decomp,
        encrypt_vector,
        plan_rotation_amounts,
        precompute_masked_matrix,
    )
    from hcpdq.heiface import HeParams

    he = HeParams(n, p, MAX_LEVEL.get(name, 3))
    params = CompressionParams(N, s, he)
    be = BgvBackend(he, seed=seed)
    amounts, col = plan_rotation_amounts(s, n)
    t0 = time.time()
    keys = be.keygen(amounts, col_swap=col)
    masked = name.startswith("masked_")
    answer = name.startswith("answer_")
    mask_counters = None
    if answer:
        import types

        from hcpdq import pdq

        support, db = masked_payload(N, s, p, seed)
        dense = [0] * N
        for i in support:
            dense[i - 1] = db[i - 1]
        hint = encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
        if name in ANSWER_LEVEL:
            hint = [be._at_level(c, ANSWER_LEVEL[name]) for c in hint]
        m0 = be.counters.snapshot()
        cts = pdq.mask(hint, types.SimpleNamespace(values=db), params, be, keys)
        mask_counters = be.counters.delta(m0).as_dict()

        def run():
            return comp(cts, params, be, keys, index_hint=hint)
    elif masked:
        support, db = masked_payload(N, s, p, seed)
        dense = [0] * N
        for i in support:
            dense[i - 1] = db[i - 1]
        table = precompute_masked_matrix(db, params)
        hint = encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
        cts = hint

        def run():
            return comp_masked(hint, table, params, be, keys)
    else:
        rng = random.Random(seed)
        support = sorted(rng.sample(range(1, N + 1), s))
        dense = [0] * N
        for i in support:
            dense[i - 1] = rng.randrange(1, p)
        cts = encrypt_vector(dense, params, be, keys)
        hint = encrypt_vector([1 if x else 0 for x in dense], params, be, keys)

        def run():
            return comp(cts, params, be, keys, index_hint=hint)
    t1 = time.time()
    before = be.counters.snapshot()
    if guard_off:
        with refimport.noise_guard_disabled():
            ans = run()
    else:
        ans = run()
    t2 = time.time()
    delta = be.counters.delta(before)
    blob = ans.serialize(be)
    w, e = ans.payload_slots(be, keys)
    rec = decomp(ans, params, be, keys)
    assert rec.entries == tuple((i, dense[i - 1]) for i in support), "reference round trip failed"
    out = ans.cts[0]
    L = he.max_level
    rec_json = {
        "case": name,
        "generator": "oracle/make_golden.py (reference hcpdq run in the build container)",
        "n": n,
        "p": p,
        "max_level": L,
        "N": N,
        "s": s,
        "seed": seed,
        "noise_guard_disabled": guard_off,
        "masked": masked,
        "answer": answer,
        "mask_counters": mask_counters,
        "cts_levels": [c.level for c in cts],
        "hint_levels": [c.level for c in hint],
        "chain_primes_desc": list(be.chain.primes),
        "key_id": keys.key_id.hex(),
        "support": support,
        "values": [dense[i - 1] for i in support],
        "answer_sha256": hashlib.sha256(blob).hexdigest(),
        "answer_len": len(blob),
        "w": w,
        "e": e,
        "noise_bits": out.payload.noise_bits,
        "out_level": out.level,
        "counters": delta.as_dict(),
        "keys_sha256": digest_arrays(keys_residues(be, keys)) if L <= 4 else None,
        # deep chains: the key digits levels <= 3 use (_KskPair.at_level,
        # bgv.py:304-312) -- first 14 pairs on the 4 smallest primes
        "keys_low_sha256": digest_arrays(keys_residues_low(be, keys)) if L > 4 else None,
        "cts_sha256": digest_arrays([ct_residues(be, c) for c in cts]),
        "hint_sha256": digest_arrays([ct_residues(be, c) for c in hint]),
        "out_sha256": digest_arrays([ct_residues(be, out)]),
        "ref_comp_seconds": round(t2 - t1, 3),
        "ref_setup_seconds": round(t1 - t0, 3),
    }
    if n <= 256:
        rec_json["full"] = {
            "cts": [ct_residues(be, c).tolist() for c in cts],
            "hint": [ct_residues(be, c).tolist() for c in hint],
            "out": ct_residues(be, out).tolist(),
            "secret": list(keys.secret),
        }
    path = os.path.join(GOLDEN, f"{name}.json")
    with open(path, "w") as fh:
        json.dump(rec_json, fh, indent=1)
    print(f"{name}: comp {t2 - t1:.1f}s sha {rec_json['answer_sha256'][:16]} -> {path}", flush=True)


if __name__ == "__main__":
    os.makedirs(GOLDEN, exist_ok=True)
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        run_case(nm)
