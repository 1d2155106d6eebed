"""CPU tests of the product's host side: the C-ABI library loads and exports
every symbol declared in include/hcomp.h, the pure-host helpers match the
reference's maps, and the host mirror of the reference API (parameters,
rotation plan, noise/counter bookkeeping, live diagonals) matches the
reference / oracle."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_names, load_golden

import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import _lib
from paper_2408_17063_b200.compress import comp_noise, live_diagonals


def header_symbols():
    src = open(os.path.join(ROOT, "include", "hcomp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(hc_[a-z0-9_]+)\s*\(", src)))


@pytest.mark.parametrize("max_level,plain_row", [(3, 4), (4, 5), (21, 23)])
def test_library_exports_every_declared_symbol(max_level, plain_row):
    """Every build (4-prime libhcomp.so, 5-prime libhcomp_l4.so, protocol-chain
    libhcomp_deep.so) exports the ABI."""
    L = _lib.lib(max_level)
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib.EXPORTS) | {"hc_trace_reset", "hc_trace_read", "hc_trace_read_tail"}
    assert L.hc_plain_row() == plain_row  # csrc/ctx.cuh PIDX = MAXL + 1: rows 0..MAXL are chain primes


def test_host_helpers_without_gpu(oracle):
    L = _lib.lib()
    be = oracle.OracleBgv(8192, 65537, 3, seed=0)
    for q in be.q:
        assert L.hc_prim_root_2n(q, 8192) == oracle.prim_root_2n(q, 8192)
    coef = np.empty(8192, dtype=np.uint16)
    perm = np.empty(8192, dtype=np.uint16)
    t = pow(3, 7, 2 * 8192)
    assert L.hc_galois_tables(8192, t, _lib.ptr(coef), _lib.ptr(perm)) == 0
    assert np.array_equal(perm.astype(np.int64), be.galois_perm(t))
    assert L.hc_galois_tables(8192, 2, _lib.ptr(coef), _lib.ptr(perm)) == _lib.HC_ERR_ARG


def test_params_mirror_reference_behaviour():
    with pytest.raises(ValueError):
        P.HeParams(8192, 40961, 3)  # p != 1 mod 2n
    with pytest.raises(ValueError):
        P.CompressionParams(1 << 17, 16, P.HeParams(8192, 65537, 3))  # p must exceed N (F4)
    he = P.HeParams(8192, 65537, 3)
    cp = P.CompressionParams(10000, 5, he)
    assert (cp.num_blocks, cp.num_ciphertexts, cp.s_pad) == (3, 2, 8)
    assert P.bsgs_shape(16) == (4, 4) and P.bsgs_shape(128) == (16, 8) and P.bsgs_shape(32) == (8, 4)


def test_rotation_plan_matches_reference(oracle):
    for s in (1, 2, 5, 8, 16, 32, 64, 128, 2048):
        assert P.plan_rotation_amounts(s, 8192) == oracle.plan_rotation_amounts(s, 8192)
    assert P.find_chain_primes(8192, 65537, 4) == sorted(oracle.OracleBgv(8192, 65537, 3).q, reverse=True)


def test_rotation_plan_matches_real_reference_if_present():
    from oracle import refimport

    if not refimport.available():
        pytest.skip("reference not present (GPU box)")
    hc = refimport.load()
    for s in (3, 8, 16, 64, 128):
        assert P.plan_rotation_amounts(s, 8192) == hc.compress.plan_rotation_amounts(s, 8192)
        assert P.bsgs_shape(s) == hc.compress.bsgs_shape(s)


@pytest.mark.parametrize("name", golden_names())
def test_noise_and_counters_replay_reference(name):
    """comp's deterministic noise_bits and op-counter deltas equal the
    reference's (golden), without running any ring arithmetic."""
    g = load_golden(name)
    if g["n"] != 8192:
        pytest.skip("the B200 backend is n = 8192 only")
    if g.get("answer"):  # mask (level 4 -> 3), then comp with mixed input levels
        from paper_2408_17063_b200.compress import FUSED_LEVEL, _NoiseSim, bsgs_noise, pack_noise_mixed

        he = P.HeParams(g["n"], g["p"], g["max_level"])
        params = P.CompressionParams(g["N"], g["s"], he)
        be = P.B200BgvBackend(he, seed=0, noise_guard=not g["noise_guard_disabled"])
        fresh = be._fresh_noise_bits()
        C = params.num_ciphertexts
        msim = _NoiseSim(be)
        cd = [(msim.mul_plain(fresh, 4), 3) for _ in range(C)]
        assert {"keyswitches": msim.ks, "pt_mults": msim.pt, "adds": msim.adds, "ct_mults": 0} == g["mask_counters"]
        sim = _NoiseSim(be)
        u = pack_noise_mixed(sim, params, [(fresh, 4)] * C, cd)
        bits, sim = bsgs_noise(sim, params, u, live_diagonals(params), FUSED_LEVEL - 1)
        assert bits == g["noise_bits"]
        assert {"keyswitches": sim.ks, "pt_mults": sim.pt, "adds": sim.adds, "ct_mults": 0} == g["counters"]
        return
    he = P.HeParams(g["n"], g["p"], 3)
    params = P.CompressionParams(g["N"], g["s"], he)
    be = P.B200BgvBackend(he, seed=0, noise_guard=not g["noise_guard_disabled"])
    fresh = be._fresh_noise_bits()
    C = params.num_ciphertexts
    bits, sim = comp_noise(be, params, [fresh] * C, [fresh] * C, live_diagonals(params))
    assert bits == g["noise_bits"]
    assert {"keyswitches": sim.ks, "pt_mults": sim.pt, "adds": sim.adds, "ct_mults": 0} == g["counters"]


def test_noise_guard_raises_where_reference_does():
    he = P.HeParams(8192, 65537, 3)
    params = P.CompressionParams(1 << 14, 32, he)
    be = P.B200BgvBackend(he, seed=0, noise_guard=True)
    f = be._fresh_noise_bits()
    with pytest.raises(P.NoiseOverflow):
        comp_noise(be, params, [f] * 2, [f] * 2, live_diagonals(params))


def test_live_diagonals_match_reference_plan(oracle):
    for N, s in ((10000, 5), (4097, 3), (8192, 8), (12289, 7)):
        params = P.CompressionParams(N, s, P.HeParams(8192, 65537, 3))
        plan = oracle.build_plan(N, s, 8192, 65537)
        want = np.array([[d is not None for d in row] for row in plan.diagonals])
        assert np.array_equal(live_diagonals(params), want)


def test_slot_index_matches_reference(oracle):
    from paper_2408_17063_b200.backend import slot_index

    be = oracle.OracleBgv(8192, 65537, 3, seed=0)
    assert np.array_equal(slot_index(8192), be.slot_index)


def test_comp_rejects_bad_inputs_like_reference():
    he = P.HeParams(8192, 65537, 3)
    params = P.CompressionParams(8192, 8, he)
    be = P.B200BgvBackend(he, seed=0)
    with pytest.raises(NotImplementedError):
        P.comp([], params, be, None)  # no index hint: power_fermat path not built
    ct = P.Ciphertext(be.backend_id, b"x" * 16, 3, P.RnsPayload(np.zeros((2, 4, 8192), np.uint64), 0.0))
    keys = P.KeySet(be.backend_id, he, b"x" * 16, {}, None, None, None, None)
    with pytest.raises(ValueError):
        P.comp([ct, ct], params, be, keys, index_hint=[ct])  # wrong count (compress.py:348-349)
    with pytest.raises(P.MissingRotationKey):
        P.comp([ct], params, be, keys, index_hint=[ct])  # no col-swap key (bgv.py:767-768)


def test_masked_matrix_mirrors_vandermonde_table_checks():
    """precompute_masked_matrix (compress.py:154-157 -> VandermondeTable,
    compress.py:107-116): wrong length raises ValueError; values are reduced
    with Python's int(v) % p (negatives included)."""
    he = P.HeParams(8192, 65537, 3)
    params = P.CompressionParams(200, 5, he)
    with pytest.raises(ValueError):
        P.precompute_masked_matrix([1] * 199, params)
    db = [-1, 65537, 70000, 3] + [0] * 196
    m = P.precompute_masked_matrix(db, params)
    assert m.db_mod_p.dtype == np.uint64 and len(m.db_mod_p) == 200
    assert list(m.db_mod_p[:4]) == [65536, 0, 70000 % 65537, 3]


def test_comp_masked_argument_checks():
    he = P.HeParams(8192, 65537, 3)
    params = P.CompressionParams(8192, 8, he)
    be = P.B200BgvBackend(he, seed=0)
    ct = P.Ciphertext(be.backend_id, b"x" * 16, 3, P.RnsPayload(np.zeros((2, 4, 8192), np.uint64), 0.0))
    keys = P.KeySet(be.backend_id, he, b"x" * 16, {}, None, None, None, None)
    with pytest.raises(TypeError):  # only tables from precompute_masked_matrix
        P.comp([ct], params, be, keys, masked=object())
    table = P.precompute_masked_matrix([1] * 8192, params)
    with pytest.raises(P.MissingRotationKey):  # same input checks as the hint path
        P.comp_masked([ct], table, params, be, keys)


def test_shard_input_ranges_cover_the_blocks_sources():
    """A rank running blocks [b0, b1) reads input ciphertexts b // 2; the
    range it uploads (hc_comp_set_inputs_range) is [b0 // 2, (b1 + 1) // 2)."""
    from paper_2408_17063_b200.dist import shard_blocks

    for B in (1, 2, 3, 4, 7, 256, 1023):
        for world in (1, 2, 3, 8):
            for rank in range(world):
                b0, b1 = shard_blocks(B, world, rank)
                if b1 == b0:
                    continue
                c0, c1 = b0 // 2, (b1 + 1) // 2
                assert {b // 2 for b in range(b0, b1)} == set(range(c0, c1))
                assert c1 <= (B + 1) // 2


def test_bench_helpers():
    import bench

    assert bench.metric_name(1 << 14, 16) == "Comp encrypted entries/sec (N=2^14, s=16)"
    assert bench.metric_name(10000, 5) == "Comp encrypted entries/sec (N=10000, s=5)"
    assert bench.pick_p(1 << 14, 0) == 65537
    assert bench.pick_p(1 << 17, 0) == 786433
    assert bench.pick_p(1 << 20, 0) == 1097729
    assert bench.pick_p(1 << 22, 0) == 4423681


@pytest.mark.parametrize("seed", [0, 1, 7, 2**32 - 1, 2**32, 12345678901234567890, -5])
def test_host_rng_reproduces_python_random(seed):
    """HostRng (csrc/pyrng.hpp) consumes random.Random(seed)'s stream exactly:
    interleaved getrandbits of every width class, randrange(3), the CBD
    sampler and randrange of a 216-bit modulus (the samplers of bgv.py:398-414)."""
    import random

    from paper_2408_17063_b200.backend import HostRng

    py = random.Random(seed)
    hr = HostRng(seed)
    for k in (1, 2, 5, 21, 31, 32, 33, 63, 64, 65, 128, 216):
        assert hr.getrandbits(k) == py.getrandbits(k), k
    assert list(hr.ternary(1000)) == [py.randrange(3) - 1 for _ in range(1000)]
    want = []
    for _ in range(500):
        a = py.getrandbits(21).bit_count()
        b = py.getrandbits(21).bit_count()
        want.append(a - b)
    assert list(hr.cbd(500, 21)) == want
    primes = P.find_chain_primes(8192, 65537, 4)[::-1]  # ascending = level order
    Q = 1
    for q in primes:
        Q *= q
    got = hr.uniform(300, Q, primes)
    vals = [py.randrange(Q) for _ in range(300)]
    assert np.array_equal(got, np.array([[v % q for v in vals] for q in primes], dtype=np.uint64))
    assert hr.getrandbits(128) == py.getrandbits(128)  # still in lockstep


def test_bench_options_pass_through_torchrun():
    """Every bench.py option has a spelling torchrun hands to the script.

    argparse prefix-matches, so torchrun's parser takes an option such as
    "--s" for its own (--standalone / --start-method / ...) and exits before
    bench.py runs; the N>1 driver launch goes through that parser."""
    import bench
    from torch.distributed.run import get_args_parser

    tr = get_args_parser()
    for act in bench.make_parser()._actions:
        longs = [o for o in act.option_strings if o.startswith("--") and o != "--help"]
        if not longs:
            continue
        ok = []
        for o in longs:
            argv = [o] if act.nargs == 0 else [o, act.choices[0] if act.choices else "1"]
            try:
                got = tr.parse_args(["--nproc-per-node", "2", "bench.py", *argv]).training_script_args
            except SystemExit:
                continue
            if got == argv:
                ok.append(o)
        assert ok, f"no spelling of {longs} survives torchrun's parser"
    a = bench.parse(["--gpus", "2", "--steps", "3", "--warmup", "3", "--sparsity", "32", "--N", "1048576"])
    assert (a.gpus, a.steps, a.warmup, a.s, a.N) == (2, 3, 3, 32, 1 << 20)
