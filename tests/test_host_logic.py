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


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    assert set(syms) <= set(_lib.EXPORTS) | {"hc_trace_reset", "hc_trace_read"}


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
