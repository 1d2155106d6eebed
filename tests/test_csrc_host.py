"""CPU check of the exact device code: the CUDA headers' arithmetic, the
256-thread NTT schedule (emulated thread by thread, same passes/swizzles as
on the GPU), the CRT/digit split and the modulus-switch correction are
compiled for the host (paper_2408_17063_b200/csrc/hosttest.cpp) and compared
bit-for-bit with the oracle."""

import ctypes

PIDX = 5  # csrc/ctx.cuh: RNS table row of the plaintext prime p (chains of up to 5 primes)

import numpy as np
import pytest

from paper_2408_17063_b200 import build as hbuild

N8K = 8192


@pytest.fixture(scope="module")
def ht():
    path = hbuild.build_selftest()
    L = ctypes.CDLL(path)
    P = ctypes.c_void_p
    L.ht_init.argtypes = [P, ctypes.c_int, ctypes.c_uint64]
    L.ht_ntt.argtypes = [ctypes.c_int, P, ctypes.c_int]
    L.ht_ntt_cl.argtypes = [ctypes.c_int, P, ctypes.c_int]
    L.ht_ntt_edge.argtypes = [ctypes.c_int, P, ctypes.c_int]
    L.ht_compose.argtypes = [ctypes.c_int, P, P, ctypes.c_int, P]
    L.ht_compose2_check.argtypes = [P, P, ctypes.c_int]
    L.ht_rescale_rd_check.argtypes = [ctypes.c_int, P, ctypes.c_int]
    L.ht_rescale_corr.argtypes = [ctypes.c_int, P, P]
    L.ht_modops.argtypes = [ctypes.c_int, ctypes.c_int, P, P, P, ctypes.c_int]
    L.ht_galois.argtypes = [ctypes.c_uint32, P, P]
    L.ht_ksfused_ntt.argtypes = [ctypes.c_int, ctypes.c_uint32, P, P, P]
    L.ht_slot_of.argtypes = [P]
    L.ht_digits.argtypes = [ctypes.c_int]
    return L


def p_(a):
    return a.ctypes.data_as(ctypes.c_void_p)


@pytest.fixture(scope="module", params=[65537, 786433])
def setup(request, ht, oracle):
    p = request.param
    be = oracle.OracleBgv(N8K, p, 3, seed=0)
    primes = np.asarray(be.q, dtype=np.uint64)
    ht.ht_init(p_(primes), 3, p)
    return ht, be, p


def rand_res(rng, q, n=N8K):
    return np.array([rng.randrange(q) for _ in range(n)], dtype=np.uint64)


def test_ntt_schedule_matches_reference_transform(setup):
    ht, be, p = setup
    import random

    rng = random.Random(5)
    for k, q in enumerate(be.q + [p]):
        a = rand_res(rng, q)
        want_f = (be.ntt if k < 4 else be.ntt_p).fwd(a[None, :], [k if k < 4 else 0])[0]
        want_i = (be.ntt if k < 4 else be.ntt_p).inv(a[None, :], [k if k < 4 else 0])[0]
        t = k if k < 4 else PIDX  # table row of the plaintext prime
        got = a.copy()
        ht.ht_ntt(t, p_(got), 0)
        assert np.array_equal(got, want_f), f"forward NTT mismatch for prime {k}"
        got = a.copy()
        ht.ht_ntt(t, p_(got), 1)
        assert np.array_equal(got, want_i), f"inverse NTT mismatch for prime {k}"
        # k_xf's form (bit-0 stage in registers at the kernel's edge) on the same data
        got = a.copy()
        ht.ht_ntt_edge(t, p_(got), 0)
        assert np.array_equal(got, want_f), f"edge-stage forward NTT mismatch for prime {k}"
        got = a.copy()
        ht.ht_ntt_edge(t, p_(got), 1)
        assert np.array_equal(got, want_i), f"edge-stage inverse NTT mismatch for prime {k}"
        # cluster schedule (8 CTAs, DSMEM exchange) on the same data
        got = a.copy()
        ht.ht_ntt_cl(t, p_(got), 0)
        assert np.array_equal(got, want_f), f"cluster forward NTT mismatch for prime {k}"
        got = a.copy()
        ht.ht_ntt_cl(t, p_(got), 1)
        assert np.array_equal(got, want_i), f"cluster inverse NTT mismatch for prime {k}"
    # lazy-range inputs up to 4q (forward) are accepted
    q = be.q[0]
    a = rand_res(rng, q)
    lazy = a + np.uint64(3 * q) * (np.arange(N8K) % 2 == 0).astype(np.uint64)
    ht.ht_ntt(0, p_(lazy), 0)
    assert np.array_equal(lazy, be.ntt.fwd(a[None, :], [0])[0])


def test_crt_digits_match_reference_digit_split(setup, oracle):
    ht, be, p = setup
    import random

    rng = random.Random(7)
    for level in (1, 2, 3):
        P = level + 1
        x = np.stack([rand_res(rng, q) for q in be.q[:P]])
        # edge values: 0, Q-1, and q_k-1 everywhere
        x[:, 0] = 0
        for k in range(P):
            x[k, 1] = be.q[k] - 1
        D = be.digits[level]
        assert ht.ht_digits(level) == D
        want = np.empty((D, N8K), dtype=np.uint64)
        qv = np.asarray(be.q[:P], dtype=np.uint64)
        oracle.lib().orc_digits(p_(np.ascontiguousarray(x)), p_(want), P, N8K, p_(qv), D, 16)
        got = np.empty((2 * D, N8K), dtype=np.uint16)
        assert ht.ht_compose(level, p_(np.ascontiguousarray(x)), None, 1, p_(got)) == 0
        assert np.array_equal(got[:D].astype(np.uint64), want)
        # negated image digits = digits of (Q - X) (0 stays 0)
        Q = be.moduli[level]
        ints = be.compose(x, level)
        neg = [(Q - v) % Q for v in ints]
        want_neg = np.array([[(v >> (16 * j)) & 0xFFFF for v in neg] for j in range(D)], dtype=np.uint16)
        assert np.array_equal(got[D:], want_neg)


def test_garner_compose2_matches_crt(setup):
    """compose2 (the level-1 Garner CRT in the fold INTT) == crt_compose<1>,
    random residues plus 0 / q_k - 1 edges."""
    ht, be, _ = setup
    import random

    rng = random.Random(11)
    n = 4096
    x0 = np.array([rng.randrange(be.q[0]) for _ in range(n)], dtype=np.uint64)
    x1 = np.array([rng.randrange(be.q[1]) for _ in range(n)], dtype=np.uint64)
    x0[:4] = [0, be.q[0] - 1, 0, be.q[0] - 1]
    x1[:4] = [0, 0, be.q[1] - 1, be.q[1] - 1]
    assert ht.ht_compose2_check(p_(x0), p_(x1), n) == 0


def test_rescale_rd_sums_equal_summed_corrections(setup):
    """EP_RESCALE_RD + k_diagx: the correction rebuilt from (r, d) equals
    rescale_corr per term, and from summed (r, d) over 1024 terms (the most a
    k_diagx job sums) equals the sum of the corrections."""
    ht, be, _ = setup
    import random

    rng = random.Random(13)
    for level in (1, 2, 3):
        q = be.q[level]
        x = np.array([rng.randrange(q) for _ in range(1024)], dtype=np.uint64)
        x[:6] = [0, 1, q // 2, q // 2 + 1, q - 1, q - 2]
        assert ht.ht_rescale_rd_check(level, p_(x), len(x)) == 0
        # worst case for the int64 sums: every r near -q/2 or +q/2
        hi = np.full(1024, q // 2, dtype=np.uint64)
        lo = np.full(1024, q // 2 + 1, dtype=np.uint64)
        assert ht.ht_rescale_rd_check(level, p_(hi), 1024) == 0
        assert ht.ht_rescale_rd_check(level, p_(lo), 1024) == 0


def test_rescale_correction_equals_mod_switch(setup, oracle):
    """out_k = x_k * q^-1 + e_k (coefficient domain) must equal the
    reference's modulus switch evaluated on the composed integer."""
    ht, be, p = setup
    import random

    rng = random.Random(9)
    for level in (1, 2, 3):
        P = level + 1
        x = np.stack([rand_res(rng, q) for q in be.q[:P]])
        x[:, :4] = 0
        x[level, 1] = be.q[level] >> 1          # r = +floor(q/2)
        x[level, 2] = (be.q[level] >> 1) + 1    # r = -floor(q/2)
        # boundaries of both centrings: r around 0 and +-q/2, d = centered_p(r mod p)
        # around 0 and +-p/2 (residues k p + {p/2 - 1 .. p/2 + 2}, from both ends)
        qd_, edge = be.q[level], []
        for t in range(24):
            edge += [t, qd_ - 1 - t, (qd_ >> 1) - t, (qd_ >> 1) + 1 + t]
        for kk in (0, 1, 5, qd_ // (2 * p) - 1, qd_ // (2 * p), qd_ // p - 2):
            for dlt in (-1, 0, 1, 2):
                for sgn in (0, 1):  # r = +(k p + p/2 + dlt) and r = -(...)
                    v = kk * p + (p >> 1) + dlt
                    edge.append(v if sgn == 0 else qd_ - v)
        edge = [v % qd_ for v in edge]
        x[level, 8:8 + len(edge)] = edge
        want = np.empty((level, N8K), dtype=np.uint64)
        qv = np.asarray(be.q[:P], dtype=np.uint64)
        oracle.lib().orc_rescale(p_(np.ascontiguousarray(x)), p_(want), P, N8K, p_(qv), p)
        e = np.empty((level, N8K), dtype=np.uint64)
        ht.ht_rescale_corr(level, p_(np.ascontiguousarray(x[level])), p_(e))
        qd = be.q[level]
        for k in range(level):
            q = be.q[k]
            qinv = pow(qd, -1, q)
            got = [(int(a) * qinv + int(b)) % q for a, b in zip(x[k], e[k])]
            assert np.array_equal(np.array(got, dtype=np.uint64), want[k]), f"level {level} prime {k}"


def test_modular_helpers(setup):
    ht, be, p = setup
    import random

    rng = random.Random(11)
    for k, q in enumerate(be.q):
        a = np.array([rng.randrange(q) for _ in range(2000)] + [0, q - 1], dtype=np.uint64)
        b = np.array([rng.randrange(q) for _ in range(2000)] + [q - 1, q - 1], dtype=np.uint64)
        want = np.array([int(x) * int(y) % q for x, y in zip(a, b)], dtype=np.uint64)
        for op in (0, 1):
            out = np.empty_like(a)
            ht.ht_modops(k, op, p_(a), p_(b), p_(out), a.size)
            assert np.array_equal(out, want)
        big = np.array([rng.getrandbits(64) for _ in range(2000)] + [2**64 - 1, 0], dtype=np.uint64)
        out = np.empty_like(big)
        ht.ht_modops(k, 2, p_(big), p_(big), p_(out), big.size)
        assert np.array_equal(out, np.array([int(v) % q for v in big], dtype=np.uint64))


def test_galois_tables_match_reference_maps(setup):
    """NTT-domain permutation == galois_permutation (bgv.py:258-261, via the
    oracle's calibrated eval exponents); coefficient gather == coeff_automorphism."""
    ht, be, p = setup
    n = N8K
    for t in (3, pow(3, 5, 2 * n), pow(3, 1024, 2 * n), 2 * n - 1):
        coef = np.empty(n, dtype=np.uint16)
        perm = np.empty(n, dtype=np.uint16)
        ht.ht_galois(t, p_(coef), p_(perm))
        assert np.array_equal(perm.astype(np.int64), be.galois_perm(t))
        c = np.arange(1, n + 1, dtype=np.int64)
        want = np.asarray(be.coeff_automorphism(list(c), t))
        src = coef & 0x7FFF
        sign = np.where(coef >> 15, -1, 1)
        assert np.array_equal(sign * c[src], want)


def test_fused_key_switch_digit_ntt(setup):
    """k_ksfused's digit transform on the host (ksfused.cuh: closed-form Galois
    gather from [digits of X | digits of Q - X], the three leading stages as a
    linear form of the 16-bit digits per output chunk, phase B on the chunk)
    equals the reference NTT (bgv.py:178-199) of the rotation's digit
    polynomial as LD_DIGGAL gathers it through the coefficient table
    (bgv.py:273-284, 622-631), for every level-2 prime and for the identity,
    three rotations and the column swap."""
    ht, be, p = setup
    import random

    n = N8K
    rng = random.Random(11)
    dpos = np.array([rng.randrange(1 << 16) for _ in range(n)], dtype=np.uint16)
    dneg = np.array([rng.randrange(1 << 16) for _ in range(n)], dtype=np.uint16)
    dpos[:4] = (0, 1, 0xFFFF, 0x8000)  # extreme digits
    for t in (1, 3, pow(3, 2, 2 * n), pow(3, 1024, 2 * n), 2 * n - 1):
        coef = np.empty(n, dtype=np.uint16)
        perm = np.empty(n, dtype=np.uint16)
        ht.ht_galois(t, p_(coef), p_(perm))
        x = np.where(coef >> 15, dneg[coef & 0x7FFF], dpos[coef & 0x7FFF]).astype(np.uint64)
        for k in range(3):
            want = be.ntt.fwd(x[None, :], [k])[0]
            got = np.empty(n, dtype=np.uint64)
            ht.ht_ksfused_ntt(k, t, p_(dpos), p_(dneg), p_(got))
            assert np.array_equal(got, want), f"fused digit NTT mismatch: t={t}, prime {k}"


def test_slot_map_matches_reference(setup):
    ht, be, p = setup
    slot_of = np.empty(N8K, dtype=np.uint16)
    ht.ht_slot_of(p_(slot_of))
    for r in range(2):
        for c in range(0, N8K // 2, 97):
            i = be.slot_index[r][c]
            assert slot_of[i] == (r << 12 | c)
