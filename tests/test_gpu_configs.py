"""GPU parity at the BASELINE config points the reference goldens do not
reach (configs 4 and 5), plus serving-path edge cases.  Every Comp here is
compared residue for residue with the CPU oracle run end to end on the same
seed (keys, payload and encryption regenerated independently on both sides),
and decrypted against the planted payload.  Configs 1-3 (every point of the
sparsity and size sweeps) are pinned to the reference itself through
tests/golden/ in test_gpu_parity.py.  Run on a B200 with `pytest -m gpu`."""

import random

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu

RING = 8192


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("CUDA GPU required for -m gpu tests")
    import paper_2408_17063_b200 as P
    from paper_2408_17063_b200 import build

    build.build_lib()
    return P


def _gpu_case(P, O, N, s, p, seed):
    he = P.HeParams(RING, p, 3)
    params = P.CompressionParams(N, s, he)
    be = P.B200BgvBackend(he, seed=seed, noise_guard=False)
    keys = be.keygen(*P.plan_rotation_amounts(s, RING))
    dense = O.plant_sparse(random.Random(seed), N, s, p)
    cts = P.encrypt_vector(dense, params, be, keys)
    hint = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
    return be, params, keys, dense, cts, hint


def _oracle_answer(O, N, s, p, seed):
    obe = O.OracleBgv(RING, p, 3, seed=seed, check_noise=False)
    okeys = obe.keygen(*O.plan_rotation_amounts(s, RING))
    dense = O.plant_sparse(random.Random(seed), N, s, p)
    ocd = O.encrypt_vector(dense, N, obe, okeys)
    ocv = O.encrypt_vector([1 if x else 0 for x in dense], N, obe, okeys)
    obe.counters = O.OCounters()
    out = O.comp(ocd, N, s, obe, okeys, ocv)
    return obe, out


def _check_vs_oracle(P, O, N, s, p, seed):
    be, params, keys, dense, cts, hint = _gpu_case(P, O, N, s, p, seed)
    before = be.counters.snapshot()
    ans = P.comp(cts, params, be, keys, index_hint=hint)
    delta = be.counters.delta(before).as_dict()
    obe, out = _oracle_answer(O, N, s, p, seed)
    assert np.array_equal(ans.cts[0].payload.res, out.c), f"(N={N}, s={s}, seed={seed}) differs from the oracle"
    assert ans.cts[0].payload.noise_bits == out.noise_bits
    assert delta == vars(obe.counters)
    assert O.sha256(ans.serialize(be)) == O.sha256(O.serialize_answer(obe, out, s))
    assert ans.payload_slots(be, keys) == O.expected_slots(dense, s, p)
    return be, ans


def test_config5_independent_queries_vs_oracle(pkg, oracle):
    """Config 5 shape: (N=2^16, s=64) queries, each with its own seeded key
    pair and rotation keys (baby 8 x giant 8, 16 blocks: the wide schedule
    with k_ksmac_mb grouping), over one GPU; two seeds, both bit-exact."""
    P, O = pkg, oracle
    answers = [_check_vs_oracle(P, O, 1 << 16, 64, 65537, seed)[1] for seed in (100, 101)]
    assert not np.array_equal(answers[0].cts[0].payload.res, answers[1].cts[0].payload.res)


@pytest.mark.slow
@pytest.mark.parametrize("N,s,p", [(1 << 20, 128, 1097729), (1 << 22, 16, 4423681)])
def test_config4_large_vs_oracle(pkg, oracle, N, s, p):
    """Config 4: (2^20, 128) -- 256 blocks, baby 16 in the throughput
    schedule, 4 chunks of 64 -- and (2^22, 16) -- 1024 blocks, 16 chunks;
    real keygen and encryption on both sides, bit-exact against the oracle."""
    _check_vs_oracle(pkg, oracle, N, s, p, 0)


def test_answer_db_after_key_change(pkg, oracle):
    """Serving two clients against one database: answer_from_match with key
    set A, then key set B (a re-plan with an identical plan tag), then A
    again -- the device mask plaintexts are regenerated each time the plan is
    (a stale answer_db tag used to skip hc_answer_db)."""
    P, O = pkg, oracle
    g = load_golden("answer_c1_N8192_s8")
    n, p, N, s, seed = g["n"], g["p"], g["N"], g["s"], g["seed"]
    he = P.HeParams(n, p, g["max_level"])
    params = P.CompressionParams(N, s, he)
    be = P.B200BgvBackend(he, seed=seed, noise_guard=not g["noise_guard_disabled"])
    keys_a = be.keygen(*P.plan_rotation_amounts(s, n))
    support, db, dense = O.masked_payload(N, s, p, seed)
    hint_a = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys_a)
    keys_b = be.keygen(*P.plan_rotation_amounts(s, n))
    hint_b = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys_b)
    want = O.expected_slots(dense, s, p)
    a1 = P.answer_from_match(hint_a, db, params, be, keys_a)
    assert O.sha256(a1.serialize(be)) == g["answer_sha256"]
    b1 = P.answer_from_match(hint_b, db, params, be, keys_b)
    assert b1.payload_slots(be, keys_b) == want
    a2 = P.answer_from_match(hint_a, db, params, be, keys_a)
    assert O.sha256(a2.serialize(be)) == g["answer_sha256"]
    # a different plan in between (other chunking), same keys
    P.DeviceComp(be, params, keys_a, chunk_blocks=1)
    a3 = P.answer_from_match(hint_a, db, params, be, keys_a)
    assert O.sha256(a3.serialize(be)) == g["answer_sha256"]


def test_chunked_lane_plans_vs_single_chunk(pkg, oracle):
    """chunk_blocks 3 and 4 with more blocks than a chunk (N=2^16: 16 blocks):
    several latency-regime chunks in one range now accumulate through the
    non-atomic diagonal MAC; the answer equals the default plan's."""
    P, O = pkg, oracle
    be, params, keys, dense, cts, hint = _gpu_case(P, O, 1 << 16, 16, 65537, 3)
    cd = np.stack([c.payload.res for c in cts])
    cv = np.stack([c.payload.res for c in hint])
    ref = P.DeviceComp(be, params, keys).run_host(cd, cv)
    for cb in (3, 4, 5):
        out = P.DeviceComp(be, params, keys, chunk_blocks=cb).run_host(cd, cv)
        assert np.array_equal(out, ref), f"chunk_blocks={cb}"
    ans = P.comp(cts, params, be, keys, index_hint=hint)
    assert ans.payload_slots(be, keys) == O.expected_slots(dense, 16, 65537)


def test_reference_shaped_objects_and_wire_round_trip(pkg, oracle):
    """The INTEGRATION.md dispatch path with reference-shaped arguments:
    parameter objects that only carry the reference's public attributes and a
    comp_masked table that only offers VandermondeTable.block (compress.py:
    103-157).  The answer is byte-identical to the reference golden, and
    CompressedAnswer.deserialize / deserialize_ciphertext (compress.py:419-430,
    bgv.py:792-814) read it back to the same residues and slots."""
    import types

    P, O = pkg, oracle
    g = load_golden("masked_c1_N8192_s8")
    n, p, N, s, seed = g["n"], g["p"], g["N"], g["s"], g["seed"]
    he_ref = types.SimpleNamespace(n=n, p=p, max_level=3)
    cp_ref = types.SimpleNamespace(N=N, s=s, he=he_ref)
    be = P.make_backend("bgv-b200", he_ref, seed=seed)
    keys = be.keygen(*P.plan_rotation_amounts(s, n))
    support, db, dense = O.masked_payload(N, s, p, seed)
    hint = P.encrypt_vector([1 if x else 0 for x in dense], cp_ref, be, keys)

    class Table:  # what hcpdq.compress.precompute_masked_matrix returns, public API only
        def block(self, k):
            return O.vandermonde_block(N, s, p, n // 2, k, db)

    ans = P.comp(hint, cp_ref, be, keys, masked=Table())
    blob = ans.serialize(be)
    assert O.sha256(blob) == g["answer_sha256"]
    back = P.CompressedAnswer.deserialize(blob, be)
    assert back.s == s and back.packed
    assert np.array_equal(back.cts[0].payload.res, ans.cts[0].payload.res)
    assert back.cts[0].payload.noise_bits == ans.cts[0].payload.noise_bits
    assert back.cts[0].key_id == keys.key_id
    assert back.payload_slots(be, keys) == (g["w"], g["e"])
    # a level-3 ciphertext (4-limb integers on the wire) round-trips too
    c = hint[0]
    c2 = be.deserialize_ciphertext(be.serialize_ciphertext(c))
    assert c2.level == 3 and np.array_equal(c2.payload.res, c.payload.res)


def test_block_range_plans_sum_to_the_full_comp(pkg, oracle):
    """Per-rank plans (hc_plan_range): each range plan holds only its blocks'
    diagonals and input ciphertexts; the partials of [0, 7) and [7, 16) summed
    as uint64 and finished equal the whole-matrix Comp (N = 2^16, 16 blocks).
    Whole-matrix entry points refuse a range plan."""
    import ctypes

    import torch

    from paper_2408_17063_b200 import _lib

    P, O = pkg, oracle
    be, params, keys, dense, cts, hint = _gpu_case(P, O, 1 << 16, 16, 65537, 5)
    cd = np.stack([c.payload.res for c in cts])
    cv = np.stack([c.payload.res for c in hint])
    ref = P.DeviceComp(be, params, keys).run_host(cd, cv)
    L = _lib.lib()
    h = be._ctx()
    total = None
    for b0, b1 in ((0, 7), (7, 16)):
        be.plan(params.N, params.s, keys, block_range=(b0, b1))
        c0, c1 = b0 // 2, (b1 + 1) // 2
        cdr = np.ascontiguousarray(cd[c0:c1])
        cvr = np.ascontiguousarray(cv[c0:c1])
        _lib.check(L.hc_comp_set_inputs_range(h, _lib.ptr(cdr), _lib.ptr(cvr), c0, c1, None))
        part = torch.zeros(L.hc_partial_words(h), dtype=torch.int64, device="cuda")
        _lib.check(L.hc_comp_partial(h, b0, b1, ctypes.c_void_p(part.data_ptr()), None))
        torch.cuda.synchronize()
        total = part if total is None else total + part
        with pytest.raises(_lib.HcompError, match="covers blocks"):
            out = np.empty((2, 1, 8192), dtype=np.uint64)
            _lib.check(L.hc_comp(h, _lib.ptr(cd), _lib.ptr(cv), cd.shape[0], _lib.ptr(out)))
    _lib.check(L.hc_comp_finish(h, ctypes.c_void_p(total.data_ptr()), None))
    out = np.empty((2, 1, 8192), dtype=np.uint64)
    _lib.check(L.hc_comp_get_output(h, _lib.ptr(out)))
    assert np.array_equal(out, ref)


def test_shared_plan_queries_vs_oracle(pkg, oracle):
    """Config 5's memory layout: query B's plan reuses query A's diagonals
    (hc_plan_shared) with its own keys and inputs; both answers equal the
    oracle's for their seeds, and A re-planning does not disturb B."""
    P, O = pkg, oracle
    N, s, p = 1 << 14, 16, 65537
    qa = _gpu_case(P, O, N, s, p, 200)
    qb = _gpu_case(P, O, N, s, p, 201)
    dca = P.DeviceComp(qa[0], qa[1], qa[2])
    dcb = P.DeviceComp(qb[0], qb[1], qb[2], share_with=dca)
    outs = []
    for (be, params, keys, dense, cts, hint), dc in ((qa, dca), (qb, dcb)):
        out = dc.run_host(np.stack([c.payload.res for c in cts]), np.stack([c.payload.res for c in hint]))
        outs.append(out)
    # the source re-plans (other chunking); the shared buffers stay alive
    P.DeviceComp(qa[0], qa[1], qa[2], chunk_blocks=1)
    be, params, keys, dense, cts, hint = qb
    again = dcb.run_host(np.stack([c.payload.res for c in cts]), np.stack([c.payload.res for c in hint]))
    assert np.array_equal(again, outs[1])
    for seed, out in zip((200, 201), outs):
        _, oout = _oracle_answer(O, N, s, p, seed)
        assert np.array_equal(out, oout.c), f"seed {seed}"


def test_device_decrypt_vs_oracle_every_level(pkg, oracle):
    """hc_decrypt (phase, INTT, CRT lift, centring, slot decode in one device
    call) against the oracle's decrypt (bgv.py:559-575) at levels 3, 2, 1, 0."""
    P, O = pkg, oracle
    be, params, keys, dense, cts, hint = _gpu_case(P, O, 8192, 8, 65537, 31)
    obe = O.OracleBgv(8192, 65537, 3, seed=31, check_noise=False)
    okeys = obe.keygen(*O.plan_rotation_amounts(8, 8192))
    octs = O.encrypt_vector(dense, 8192, obe, okeys)
    rows = np.random.default_rng(2).integers(0, 65537, (2, 4096)).astype(np.int64)
    m = P.SlotMatrix(65537, rows)
    cur, ocur = cts[0], octs[0]
    for lvl in (3, 2, 1, 0):
        assert cur.level == lvl
        got = be.decrypt(cur, keys).rows
        want = obe.decrypt(ocur, okeys)
        assert np.array_equal(np.asarray(got, dtype=np.int64), np.asarray(want, dtype=np.int64)), f"level {lvl}"
        if lvl:
            cur = be.mul_plain(cur, m)
            ocur = obe.mul_plain(ocur, rows)


def test_comp_inputs_above_level_3_on_both_sides_vs_oracle(pkg, oracle):
    """Fresh ciphertexts at level 4 on a 5-prime chain (both inputs above the
    fused schedule's level 3): pack_pair at level 4, BSGS at level 3, the
    answer at level 1 -- as the reference computes it -- through the backend's
    single GPU operations; bit-exact with the oracle (residues, noise bits,
    counters, serialized bytes) and decrypting to the power sums."""
    P, O = pkg, oracle
    n, p, N, s, seed = 8192, 65537, 8192, 8, 41
    he = P.HeParams(n, p, 4)
    params = P.CompressionParams(N, s, he)
    be = P.B200BgvBackend(he, seed=seed)
    keys = be.keygen(*P.plan_rotation_amounts(s, n))
    dense = O.plant_sparse(random.Random(seed), N, s, p)
    cts = P.encrypt_vector(dense, params, be, keys)
    hint = P.encrypt_vector([1 if x else 0 for x in dense], params, be, keys)
    before = be.counters.snapshot()
    ans = P.comp(cts, params, be, keys, index_hint=hint)
    delta = be.counters.delta(before).as_dict()
    assert ans.cts[0].level == 1
    obe = O.OracleBgv(n, p, 4, seed=seed)
    okeys = obe.keygen(*O.plan_rotation_amounts(s, n))
    octs = O.encrypt_vector(dense, N, obe, okeys)
    ohint = O.encrypt_vector([1 if x else 0 for x in dense], N, obe, okeys)
    obe.counters = O.OCounters()
    out = O.comp(octs, N, s, obe, okeys, ohint)
    assert out.level == 1
    assert np.array_equal(ans.cts[0].payload.res, out.c)
    assert ans.cts[0].payload.noise_bits == out.noise_bits
    assert delta == vars(obe.counters)
    assert O.sha256(ans.serialize(be)) == O.sha256(O.serialize_answer(obe, out, s))
    assert ans.payload_slots(be, keys) == O.expected_slots(dense, s, p)


def test_fused_key_switch_kernel_matches_multi_launch(pkg, oracle):
    """k_ksfused (one kernel per rotation: digit NTTs + key MAC + c0
    automorphism, hc_set_ksfused) gives the multi-launch throughput schedule's
    answer bit for bit at N = 2^17 (32-block chunks: column swap with
    tinv = 1 and three baby rotations through the closed-form gather), and the
    multi-launch answer is the oracle's."""
    from paper_2408_17063_b200 import _lib

    P, O = pkg, oracle
    N, s, p, seed = 1 << 17, 16, 786433, 5
    be, params, keys, dense, cts, hint = _gpu_case(P, O, N, s, p, seed)
    cd = np.ascontiguousarray(np.stack([c.payload.res for c in cts]))
    cv = np.ascontiguousarray(np.stack([c.payload.res for c in hint]))
    outs = {}
    try:
        for on in (0, 1):
            _lib.check(_lib.lib().hc_set_ksfused(on))
            be._planned = None  # re-plan with this setting
            dc = P.DeviceComp(be, params, keys)
            dc.set_inputs(cd, cv)
            dc.launch()
            dc.launch()  # replay: the fused kernel leaves no state behind
            outs[on] = dc.output().copy()
            kinds = be.plan_info()["kernel_launches"]
            outs[("launches", on)] = kinds
    finally:
        _lib.check(_lib.lib().hc_set_ksfused(0))
        be._planned = None
    assert np.array_equal(outs[0], outs[1])
    assert outs[("launches", 1)] < outs[("launches", 0)]  # S3+S4 and S7+S8 are one launch each
    _, oout = _oracle_answer(O, N, s, p, seed)
    assert np.array_equal(outs[0], np.asarray(oout.c, dtype=np.uint64).reshape(outs[0].shape))


def test_serving_pipeline_upload_launch_readback(pkg, oracle):
    """The streamed serving path of bench.py's e2e: two query
    contexts with their own keys; hc_comp_upload_async on a copy stream,
    hc_comp_launch on the compute stream, hc_comp_get_output_async on a third,
    chained by events over six steps.  Every answer equals the context's own
    hc_comp result (itself pinned to the oracle by the tests above)."""
    import torch

    from paper_2408_17063_b200 import _lib

    P, O = pkg, oracle
    N, s, p = 1 << 13, 8, 65537
    L = _lib.lib()
    ctxs = []
    for seed in (21, 22):
        be, params, keys, dense, cts, hint = _gpu_case(P, O, N, s, p, seed)
        cd = np.ascontiguousarray(np.stack([c.payload.res for c in cts]))
        cv = np.ascontiguousarray(np.stack([c.payload.res for c in hint]))
        want = P.comp(cts, params, be, keys, index_hint=hint).cts[0].payload.res.copy()
        dc = P.DeviceComp(be, params, keys)
        # start from wrong inputs: the pipeline's uploads must be what the Comps read
        dc.set_inputs(np.zeros_like(cd), np.zeros_like(cv))
        ctxs.append(dict(be=be, dc=dc, h=be._ctx(), want=want, C=cd.shape[0],
                         cd_h=torch.from_numpy(cd).pin_memory(), cv_h=torch.from_numpy(cv).pin_memory(),
                         out_h=torch.zeros((2, 1, RING), dtype=torch.int64).pin_memory()))
    comp_s, h2d_s, d2h_s = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    steps, R = 6, len(ctxs)
    up = [torch.cuda.Event() for _ in range(steps)]
    done = [torch.cuda.Event() for _ in range(steps)]
    back = [torch.cuda.Event() for _ in range(steps)]

    def upload(i):
        c = ctxs[i % R]
        if i >= R:
            h2d_s.wait_event(done[i - R])
        _lib.check(L.hc_comp_upload_async(c["h"], c["cd_h"].data_ptr(), c["cv_h"].data_ptr(), c["C"], h2d_s.cuda_stream))
        up[i].record(h2d_s)

    upload(0)
    for i in range(steps):
        c = ctxs[i % R]
        comp_s.wait_event(up[i])
        if i >= R:
            comp_s.wait_event(back[i - R])
        c["dc"].launch(comp_s.cuda_stream)
        done[i].record(comp_s)
        if i + 1 < steps:
            upload(i + 1)
        d2h_s.wait_event(done[i])
        _lib.check(L.hc_comp_get_output_async(c["h"], c["out_h"].data_ptr(), d2h_s.cuda_stream))
        back[i].record(d2h_s)
    torch.cuda.synchronize()
    for c in ctxs:
        assert np.array_equal(c["out_h"].numpy().view(np.uint64).reshape(c["want"].shape), c["want"])
    # argument checks of the new entry point
    assert L.hc_comp_upload_async(ctxs[0]["h"], ctxs[0]["cd_h"].data_ptr(), ctxs[0]["cv_h"].data_ptr(), 99, None) != 0
