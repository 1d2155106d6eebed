"""TEST INFRASTRUCTURE ONLY -- CPU oracle for the BGV Comp hot path.

A restatement, in RNS form, of the reference's BGV backend
(/root/reference/pkg/src/hcpdq/bgv.py) and Comp schedule (compress.py).
It is the parity checker for the CUDA path and the CPU arm of
`bench.py --impl reference`; nothing in the product package imports it.

Representation: a ring element at level l is `uint64[l+1][n]`, row k holding
the residue modulo `level_prime(k)` (so row l is the prime a modulus switch
divides out, bgv.py:104-106).  The reference keeps the composite integer mod
Q_l; its composite NTT's residues equal the per-prime NTTs because the
composite root is CRT(per-prime roots) (bgv.py:343-348), and
every non-linear step (modulus switch, key-switch digits, decrypt centering,
serialization) is evaluated here on the exactly composed integer.

Randomness is consumed from one `random.Random(seed)` in exactly the
reference's order (bgv.py:338,398-414,464-520,537-557), so keys, key_id and
ciphertexts are bit-identical to the reference's for the same seed.
"""

from __future__ import annotations

import ctypes
import hashlib
import math
import os
import random
import struct
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

CBD_HALF_WIDTH = 21  # bgv.py:48


def lib():
    """Load oracle/liboracle.so (built by oracle/Makefile)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            import subprocess

            subprocess.check_call(["make", "-s", "-C", _HERE])
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        I = ctypes.c_int
        U = ctypes.c_uint64
        L.orc_ntt_tables.argtypes = [U, U, I, P, P, P]
        L.orc_ntt_fwd.argtypes = [P, I, I, P, P, P]
        L.orc_ntt_inv.argtypes = [P, I, I, P, P, P, P]
        L.orc_pointwise.argtypes = [P, P, P, I, I, I, P, I]
        L.orc_rescale.argtypes = [P, P, I, I, P, U]
        L.orc_digits.argtypes = [P, P, I, I, P, I, I]
        L.orc_mac_digits.argtypes = [P, P, P, P, P, I, I, I, P]
        L.orc_compose.argtypes = [P, P, I, I, P, I]
        L.orc_num_threads.restype = I
        L.orc_set_num_threads.argtypes = [I]
        L.orc_set_num_threads.restype = None
        _LIB = L
    return _LIB


def _p(a: np.ndarray):
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(ctypes.c_void_p)


# ---------------------------------------------------------------------------
# number theory (bgv.py:60-76, 115-126)
# ---------------------------------------------------------------------------

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin (exact below 3.3e24)."""
    if n < 2:
        return False
    for b in _MR_BASES:
        if n % b == 0:
            return n == b
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    for a in _MR_BASES:
        x = pow(a, d, n)
        if x in (1, n - 1):
            continue
        for _ in range(r - 1):
            x = x * x % n
            if x == n - 1:
                break
        else:
            return False
    return True


def find_chain_primes(n: int, p: int, count: int, bits: int = 54) -> list[int]:
    """bgv.py:60-76: largest-first primes = 1 (mod 2n) and = 1 (mod p)."""
    step = 2 * n * p // math.gcd(2 * n, p)
    top = (1 << bits) - 1
    cand = top - (top - 1) % step
    out = []
    floor = 1 << (bits - 1)
    while len(out) < count and cand > floor:
        if is_prime(cand):
            out.append(cand)
        cand -= step
    if len(out) < count:
        raise RuntimeError("no NTT prime chain")
    return out


def prim_root_2n(q: int, n: int) -> int:
    """bgv.py:120-126."""
    for g in range(2, q):
        w = pow(g, (q - 1) // (2 * n), q)
        if pow(w, n, q) == q - 1:
            return w
    raise RuntimeError("no root")


def bitrev(n: int) -> list[int]:
    bits = n.bit_length() - 1
    return [int(format(i, f"0{bits}b")[::-1], 2) for i in range(n)]


# ---------------------------------------------------------------------------
# per-prime NTT contexts
# ---------------------------------------------------------------------------


class PrimeNtt:
    """Tables for a set of primes (one row each)."""

    def __init__(self, n: int, primes: list[int]):
        self.n = n
        self.q = np.asarray(primes, dtype=np.uint64)
        k = len(primes)
        self.tbl = np.zeros((k, n), dtype=np.uint64)
        self.itbl = np.zeros((k, n), dtype=np.uint64)
        self.ninv = np.zeros(k, dtype=np.uint64)
        L = lib()
        for i, q in enumerate(primes):
            psi = prim_root_2n(q, n)
            ninv = ctypes.c_uint64()
            t = np.zeros(n, dtype=np.uint64)
            it = np.zeros(n, dtype=np.uint64)
            L.orc_ntt_tables(q, psi, n, _p(t), _p(it), ctypes.byref(ninv))
            self.tbl[i] = t
            self.itbl[i] = it
            self.ninv[i] = ninv.value

    def fwd(self, a: np.ndarray, which) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        rows = a.reshape(-1, self.n)
        w = np.ascontiguousarray(np.asarray(which, dtype=np.int32).reshape(-1))
        assert w.size == rows.shape[0]
        lib().orc_ntt_fwd(_p(rows), rows.shape[0], self.n, _p(self.q), _p(self.tbl), _p(w))
        return a

    def inv(self, a: np.ndarray, which) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        rows = a.reshape(-1, self.n)
        w = np.ascontiguousarray(np.asarray(which, dtype=np.int32).reshape(-1))
        assert w.size == rows.shape[0]
        lib().orc_ntt_inv(
            _p(rows), rows.shape[0], self.n, _p(self.q), _p(self.itbl), _p(self.ninv), _p(w)
        )
        return a


# ---------------------------------------------------------------------------
# data model (heiface.py:203-213, bgv.py:287-291)
# ---------------------------------------------------------------------------


class MissingRotationKey(KeyError):
    pass


class LevelExhausted(RuntimeError):
    pass


class NoiseOverflow(RuntimeError):
    pass


@dataclass
class OCt:
    """Ciphertext at `level`: c uint64[2][level+1][n] NTT-domain residues."""

    key_id: bytes
    level: int
    c: np.ndarray
    noise_bits: float


@dataclass
class OKeys:
    key_id: bytes
    secret: list  # ternary coefficients
    pk_b: np.ndarray  # [L+1][n]
    pk_a: np.ndarray
    relin: np.ndarray  # [D_L][2][L+1][n]   (b_j, a_j)
    rotation_keys: dict  # r -> (t, ksk[D_L][2][L+1][n])
    col_swap_key: tuple | None


@dataclass
class OCounters:
    keyswitches: int = 0
    ct_mults: int = 0
    pt_mults: int = 0
    adds: int = 0


class OracleBgv:
    """Restatement of `BgvBackend` (bgv.py:321-770) over RNS residues."""

    def __init__(self, n: int, p: int, max_level: int, seed=None, check_noise: bool = True):
        self.n, self.p, self.L = n, p, max_level
        self.slots = n // 2
        self.rng = random.Random(seed)
        self.check_noise = check_noise
        self.counters = OCounters()
        primes_desc = sorted(find_chain_primes(n, p, max_level + 1, 54), reverse=True)
        self.primes_desc = primes_desc
        # RNS row k <-> level_prime(k) = primes[L - k]  (bgv.py:104-106)
        self.q = [primes_desc[max_level - k] for k in range(max_level + 1)]
        self.ntt = PrimeNtt(n, self.q)
        self.ntt_p = PrimeNtt(n, [p])
        self.moduli = [math.prod(self.q[: l + 1]) for l in range(max_level + 1)]
        self.digits = [-(-self.moduli[l].bit_length() // 16) for l in range(max_level + 1)]
        # evaluation exponents: NTT(X) gives psi^{e_i} at index i (bgv.py:170-174)
        self.eval_exponents = self._calibrate()
        self.index_of_exponent = {e: i for i, e in enumerate(self.eval_exponents)}
        two_n = 2 * n
        idx = np.zeros((2, self.slots), dtype=np.int64)  # bgv.py:367-377
        e = 1
        for c in range(self.slots):
            idx[0, c] = self.index_of_exponent[e]
            idx[1, c] = self.index_of_exponent[two_n - e]
            e = (e * 3) % two_n
        self.slot_index = idx
        self._perm_cache = {}

    # -- helpers -------------------------------------------------------------

    def _calibrate(self) -> list[int]:
        q = int(self.q[0])
        psi = prim_root_2n(q, self.n)
        pows = {}
        v = 1
        for e in range(2 * self.n):
            pows[v] = e
            v = v * psi % q
        x = np.zeros((1, self.n), dtype=np.uint64)
        x[0, 1] = 1
        y = self.ntt.fwd(x, [0])[0]
        return [pows[int(t)] for t in y]

    def rows(self, level: int) -> list[int]:
        return list(range(level + 1))

    def fwd(self, a: np.ndarray, level: int) -> np.ndarray:
        """NTT of [..., level+1, n] residues (bgv.py:178-199 per prime)."""
        shp = a.shape
        which = np.broadcast_to(np.arange(level + 1), shp[:-1]).reshape(-1)
        return self.ntt.fwd(a, which).reshape(shp)

    def inv(self, a: np.ndarray, level: int) -> np.ndarray:
        shp = a.shape
        which = np.broadcast_to(np.arange(level + 1), shp[:-1]).reshape(-1)
        return self.ntt.inv(a, which).reshape(shp)

    def residues(self, ints, level: int) -> np.ndarray:
        """Signed/big Python ints -> [level+1][n] residues (Python %)."""
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        for k in range(level + 1):
            q = self.q[k]
            out[k] = np.array([int(v) % q for v in ints], dtype=np.uint64)
        return out

    def small_residues(self, vals: np.ndarray, level: int) -> np.ndarray:
        """Small signed int64 values -> residues (vectorised)."""
        vals = np.asarray(vals, dtype=np.int64)
        out = np.empty((level + 1, self.n), dtype=np.uint64)
        for k in range(level + 1):
            q = np.int64(self.q[k])
            out[k] = np.mod(vals, q).astype(np.uint64)
        return out

    def pointwise(self, x: np.ndarray, y: np.ndarray, level: int, op: str) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(np.broadcast_to(y, x.shape), dtype=np.uint64)
        out = np.empty_like(x)
        rows = x.size // self.n
        qv = np.asarray(self.q[: level + 1], dtype=np.uint64)
        lib().orc_pointwise(
            _p(x), _p(y), _p(out), rows, level + 1, self.n, _p(qv), {"mul": 0, "add": 1, "sub": 2}[op]
        )
        return out

    def compose(self, res: np.ndarray, level: int) -> list[int]:
        """Exact integers in [0, Q_level) from residues [level+1][n]."""
        W = 4
        out = np.empty((self.n, W), dtype=np.uint64)
        qv = np.asarray(self.q[: level + 1], dtype=np.uint64)
        lib().orc_compose(_p(np.ascontiguousarray(res)), _p(out), level + 1, self.n, _p(qv), W)
        return [
            int(a) | (int(b) << 64) | (int(c) << 128) | (int(d) << 192) for a, b, c, d in out
        ]

    # -- slots (bgv.py:379-394) ------------------------------------------------

    def slot_encode(self, rows: np.ndarray) -> np.ndarray:
        evals = np.zeros(self.n, dtype=np.uint64)
        r = np.asarray(rows, dtype=np.int64) % self.p
        evals[self.slot_index[0]] = r[0]
        evals[self.slot_index[1]] = r[1]
        return self.ntt_p.inv(evals[None, :], [0])[0]

    def slot_decode(self, coeffs: np.ndarray) -> np.ndarray:
        ev = self.ntt_p.fwd(np.asarray(coeffs, dtype=np.uint64)[None, :] % np.uint64(self.p), [0])[0]
        return np.stack([ev[self.slot_index[0]], ev[self.slot_index[1]]]).astype(np.int64)

    def plain_ntt(self, rows: np.ndarray, level: int) -> np.ndarray:
        """bgv.py:452-460: slot_encode (coeffs in [0,p)) then NTT mod Q_level."""
        coeffs = self.slot_encode(rows)
        res = np.broadcast_to(coeffs, (level + 1, self.n)).copy()
        return self.fwd(res, level)

    # -- sampling (bgv.py:398-414) -----------------------------------------------

    def sample_ternary(self) -> list[int]:
        return [self.rng.randrange(3) - 1 for _ in range(self.n)]

    def sample_cbd(self) -> list[int]:
        rng = self.rng
        k = CBD_HALF_WIDTH
        out = []
        for _ in range(self.n):
            a = bin(rng.getrandbits(k)).count("1")
            b = bin(rng.getrandbits(k)).count("1")
            out.append(a - b)
        return out

    def sample_uniform_ntt(self, level: int) -> np.ndarray:
        modulus = self.moduli[level]
        vals = [self.rng.randrange(modulus) for _ in range(self.n)]
        return self.residues(vals, level)

    # -- keys (bgv.py:464-520) -----------------------------------------------------

    def coeff_automorphism(self, coeffs, t: int) -> list[int]:
        """bgv.py:273-284 on small signed coefficients (result as signed ints
        whose residues equal the reference's values mod Q)."""
        n = self.n
        out = [0] * n
        two_n = 2 * n
        for i, c in enumerate(coeffs):
            if c:
                j = (i * t) % two_n
                if j >= n:
                    out[j - n] = -c
                else:
                    out[j] = c
        return out

    def keygen(self, rotation_amounts, col_swap: bool = True) -> OKeys:
        n, p, L = self.n, self.p, self.L
        amounts = sorted(set(int(r) for r in rotation_amounts))
        for r in amounts:
            if not (0 <= r < self.slots):
                raise ValueError(f"rotation amount {r} outside [0, n/2)")
        s = self.sample_ternary()
        s_ntt = self.fwd(self.small_residues(s, L), L)
        pk_a = self.sample_uniform_ntt(L)
        e = self.sample_cbd()
        pe_ntt = self.fwd(self.small_residues(np.asarray(e) * p, L), L)
        pk_b = self.pointwise(pe_ntt, self.pointwise(pk_a, s_ntt, L, "mul"), L, "sub")

        D = self.digits[L]
        # deep protocol chains (L > 4): keep the slice levels <= 3 read (first
        # D_3 pairs on the 4 smallest primes, _KskPair.at_level bgv.py:304-312)
        # while drawing every pair's samples in the reference's order
        kl = 3 if L > 4 else L
        dk = self.digits[3] if L > 4 else D
        s_k = np.ascontiguousarray(s_ntt[: kl + 1])

        def make_ksk(target_res: np.ndarray) -> np.ndarray:
            target_ntt = self.fwd(np.ascontiguousarray(target_res[: kl + 1]), kl)
            ksk = np.empty((dk, 2, kl + 1, n), dtype=np.uint64)
            for j in range(D):
                vals = [self.rng.randrange(self.moduli[L]) for _ in range(n)]  # a_j (bgv.py:412-414)
                e_j = self.sample_cbd()
                if j >= dk:
                    continue
                a_j = self.residues(vals, kl)
                pej = self.fwd(self.small_residues(np.asarray(e_j) * p, kl), kl)
                shift = np.array([pow(2, 16 * j, int(q)) for q in self.q[: kl + 1]], dtype=np.uint64)
                sh_t = self.pointwise(target_ntt, np.repeat(shift[:, None], n, axis=1), kl, "mul")
                b_j = self.pointwise(
                    self.pointwise(pej, self.pointwise(a_j, s_k, kl, "mul"), kl, "sub"), sh_t, kl, "add"
                )
                ksk[j, 0] = b_j
                ksk[j, 1] = a_j
            return ksk

        s_sq = self.inv(self.pointwise(s_k, s_k, kl, "mul"), kl)  # residues of [0,Q) ints
        relin = make_ksk(s_sq)
        two_n = 2 * n
        rot = {}
        for r in amounts:
            if r == 0:
                continue
            t = pow(3, r, two_n)
            rot[r] = (t, make_ksk(self.small_residues(self.coeff_automorphism(s, t), kl)))
        col = None
        if col_swap:
            t = two_n - 1
            col = (t, make_ksk(self.small_residues(self.coeff_automorphism(s, t), kl)))
        key_id = self.rng.getrandbits(128).to_bytes(16, "little")
        return OKeys(key_id, s, pk_b, pk_a, relin, rot, col)

    # -- enc / dec (bgv.py:533-575) --------------------------------------------------

    def fresh_noise_bits(self) -> float:
        return math.log2(self.p) + math.log2(CBD_HALF_WIDTH) + math.log2(2 * self.n + 2)

    def encrypt(self, rows: np.ndarray, keys: OKeys) -> OCt:
        L, p = self.L, self.p
        m = self.slot_encode(rows).astype(np.int64)
        u_ntt = self.fwd(self.small_residues(self.sample_ternary(), L), L)
        e0 = np.asarray(self.sample_cbd(), dtype=np.int64)
        e1 = np.asarray(self.sample_cbd(), dtype=np.int64)
        body0 = self.fwd(self.small_residues(p * e0 + m, L), L)
        body1 = self.fwd(self.small_residues(p * e1, L), L)
        c0 = self.pointwise(self.pointwise(keys.pk_b, u_ntt, L, "mul"), body0, L, "add")
        c1 = self.pointwise(self.pointwise(keys.pk_a, u_ntt, L, "mul"), body1, L, "add")
        return OCt(keys.key_id, L, np.stack([c0, c1]), self.fresh_noise_bits())

    def decrypt(self, ct: OCt, keys: OKeys) -> np.ndarray:
        l = ct.level
        s_ntt = self.fwd(self.small_residues(keys.secret, l), l)
        phase = self.inv(
            self.pointwise(ct.c[0], self.pointwise(ct.c[1], s_ntt, l, "mul"), l, "add"), l
        )
        Q = self.moduli[l]
        half = Q >> 1
        ints = self.compose(phase, l)
        centered = np.array([(x - Q if x > half else x) % self.p for x in ints], dtype=np.uint64)
        return self.slot_decode(centered)

    # -- noise (bgv.py:421-429) ----------------------------------------------------

    def _threshold_bits(self, level: int) -> float:
        return self.moduli[level].bit_length() - 1

    def _check(self, bits: float, level: int) -> float:
        if self.check_noise and bits >= self._threshold_bits(level):
            raise NoiseOverflow(f"noise estimate 2^{bits:.1f} crosses the level-{level} threshold")
        return bits

    # -- level plumbing (bgv.py:579-647) ------------------------------------------

    def _rescale_deep(self, res: np.ndarray, level: int) -> np.ndarray:
        """bgv.py:592-603 literally on Python integers for levels past the C
        oracle's 4-limb compose: x = CRT(res), r = centred(x mod q),
        y = (x - r) / q, d = centred_p((x - y) mod p), out = (y + d) mod Q_{l-1}."""
        primes = [int(q) for q in self.q[: level + 1]]
        Q = self.moduli[level]
        q = primes[level]
        p = self.p
        coef = []
        for k, qk in enumerate(primes):
            Mk = Q // qk
            coef.append(Mk * pow(Mk, -1, qk))
        rows = [res[k].tolist() for k in range(level + 1)]
        out = np.empty((level, self.n), dtype=np.uint64)
        Qn = self.moduli[level - 1]
        ys = []
        for j in range(self.n):
            x = sum(int(rows[k][j]) * coef[k] for k in range(level + 1)) % Q
            r = x % q
            if r > q // 2:
                r -= q
            y = (x - r) // q
            d = (x - y) % p
            if d > p // 2:
                d -= p
            ys.append((y + d) % Qn)
        for k in range(level):
            qk = primes[k]
            out[k] = np.array([v % qk for v in ys], dtype=np.uint64)
        return out

    def mod_switch(self, c: np.ndarray, noise: float, level: int):
        """_mod_switch_once: INTT mod Q_l, rescale (orc_rescale), NTT mod Q_{l-1}."""
        coeffs = self.inv(c, level)  # [2][l+1][n]
        out = np.empty((2, level, self.n), dtype=np.uint64)
        qv = np.asarray(self.q[: level + 1], dtype=np.uint64)
        for i in range(2):
            src = np.ascontiguousarray(coeffs[i])
            if level > 4:
                out[i] = self._rescale_deep(src, level)
                continue
            dst = np.empty((level, self.n), dtype=np.uint64)
            lib().orc_rescale(_p(src), _p(dst), level + 1, self.n, _p(qv), self.p)
            out[i] = dst
        out = self.fwd(out, level - 1)
        qd = self.q[level]
        floor_bits = math.log2(self.p) + math.log2(self.n)
        bits = max(noise - math.log2(qd), floor_bits) + 1
        return out, bits

    def key_switch(self, poly_ntt: np.ndarray, ksk: np.ndarray, level: int):
        """_key_switch (bgv.py:616-647).  ksk: [D_L][2][L+1][n]; the level's
        key is its first D_l pairs reduced mod Q_l, i.e. rows 0..l (bgv.py:304-312)."""
        D = self.digits[level]
        P = level + 1
        coeffs = np.ascontiguousarray(self.inv(poly_ntt, level))
        dig = np.empty((D, self.n), dtype=np.uint64)
        qv = np.asarray(self.q[:P], dtype=np.uint64)
        lib().orc_digits(_p(coeffs), _p(dig), P, self.n, _p(qv), D, 16)
        dig_res = np.ascontiguousarray(np.broadcast_to(dig[:, None, :], (D, P, self.n)))
        dig_ntt = self.fwd(dig_res, level)
        b = np.ascontiguousarray(ksk[:D, 0, :P])
        a = np.ascontiguousarray(ksk[:D, 1, :P])
        out0 = np.empty((P, self.n), dtype=np.uint64)
        out1 = np.empty((P, self.n), dtype=np.uint64)
        lib().orc_mac_digits(_p(dig_ntt), _p(b), _p(a), _p(out0), _p(out1), D, P, self.n, _p(qv))
        noise = (
            math.log2(self.p) + math.log2(D) + 16 + math.log2(self.n) + math.log2(CBD_HALF_WIDTH)
        )
        return out0, out1, noise

    # -- homomorphic ops (bgv.py:651-770) -----------------------------------------

    def add(self, a: OCt, b: OCt) -> OCt:
        if a.key_id != b.key_id:
            raise ValueError("ciphertexts under different key sets")
        lvl = min(a.level, b.level)
        a = self.at_level(a, lvl)
        b = self.at_level(b, lvl)
        self.counters.adds += 1
        bits = self._check(max(a.noise_bits, b.noise_bits) + 1, lvl)
        return OCt(a.key_id, lvl, self.pointwise(a.c, b.c, lvl, "add"), bits)

    def at_level(self, c: OCt, level: int) -> OCt:
        while c.level > level:
            out, bits = self.mod_switch(c.c, c.noise_bits, c.level)
            c = OCt(c.key_id, c.level - 1, out, bits)
        return c

    def mul_plain(self, c: OCt, rows: np.ndarray) -> OCt:
        lvl = c.level
        if lvl < 1:
            raise LevelExhausted("plaintext multiply at level 0")
        pt = self.plain_ntt(rows, lvl)
        bits = c.noise_bits + math.log2(self.p) + math.log2(self.n)
        self._check(bits, lvl)
        self.counters.pt_mults += 1
        prod = self.pointwise(c.c, pt[None], lvl, "mul")
        out, bits = self.mod_switch(prod, bits, lvl)
        return OCt(c.key_id, lvl - 1, out, bits)

    def galois_perm(self, t: int) -> np.ndarray:
        """bgv.py:258-261."""
        perm = self._perm_cache.get(t)
        if perm is None:
            two_n = 2 * self.n
            perm = np.array(
                [self.index_of_exponent[(e * t) % two_n] for e in self.eval_exponents], dtype=np.int64
            )
            self._perm_cache[t] = perm
        return perm

    def apply_galois(self, c: OCt, t: int, ksk: np.ndarray) -> OCt:
        lvl = c.level
        perm = self.galois_perm(t)
        s = np.ascontiguousarray(c.c[:, :, perm])
        ks0, ks1, ks_noise = self.key_switch(s[1], ksk, lvl)
        c0 = self.pointwise(s[0], ks0, lvl, "add")
        bits = self._check(max(c.noise_bits, ks_noise) + 1, lvl)
        self.counters.keyswitches += 1
        return OCt(c.key_id, lvl, np.stack([c0, ks1]), bits)

    def rot_row(self, c: OCt, r: int, keys: OKeys) -> OCt:
        r = r % self.slots
        if r == 0:
            return OCt(c.key_id, c.level, c.c.copy(), c.noise_bits)
        entry = keys.rotation_keys.get(r)
        if entry is None:
            raise MissingRotationKey(f"rotation by {r} was not declared at keygen")
        t, ksk = entry
        return self.apply_galois(c, t, ksk)

    def rot_col(self, c: OCt, keys: OKeys) -> OCt:
        if keys.col_swap_key is None:
            raise MissingRotationKey("column-swap key was not declared at keygen")
        t, ksk = keys.col_swap_key
        return self.apply_galois(c, t, ksk)

    # -- serialization (bgv.py:774-790, heiface.py:256-257) -----------------------

    def serialize_ciphertext(self, c: OCt) -> bytes:
        l = c.level
        W = -(-self.moduli[l].bit_length() // 64)
        head = struct.pack("<BBIQB", 0x01, l, self.n, self.p, self.L)
        parts = [head, c.key_id, struct.pack("<d", c.noise_bits)]
        coeffs = self.inv(c.c, l)
        for i in range(2):
            for x in self.compose(coeffs[i], l):
                parts.append(int(x).to_bytes(8 * W, "little"))
        return b"HCV1" + struct.pack("<BH", 0x02, 1) + b"".join(parts)


# ---------------------------------------------------------------------------
# Comp schedule (compress.py restated)
# ---------------------------------------------------------------------------


def bsgs_shape(s: int) -> tuple[int, int]:
    """compress.py:76-84."""
    s_pad = 1 << (s - 1).bit_length()
    log_target = ((2 * s_pad).bit_length() - 1) / 2
    baby = 1 << int(log_target)
    baby = min(max(baby, 1), s_pad)
    return baby, s_pad // baby


def plan_rotation_amounts(s: int, n: int) -> tuple[list[int], bool]:
    """compress.py:87-100."""
    m = n // 2
    s_pad = 1 << (s - 1).bit_length()
    baby, giant = bsgs_shape(s)
    amounts = set(range(1, baby))
    amounts.update((g * baby) % m for g in range(1, giant))
    step = s_pad
    while step < m:
        amounts.add(step)
        step <<= 1
    amounts.discard(0)
    return sorted(amounts), True


def vandermonde_block(N: int, s: int, p: int, m: int, k: int, db=None) -> np.ndarray:
    """compress.py:120-141: rows j=0..s-1 hold col^(j+1) mod p for the
    block's columns k*m+1..(k+1)*m, zero past N; with a cleartext database
    (compress.py:107-116,131-135) each column is scaled by db[col-1] mod p."""
    cols = np.arange(k * m + 1, (k + 1) * m + 1, dtype=np.int64)
    valid = cols <= N
    base = np.where(valid, cols % p, 0).astype(object if p >= (1 << 31) else np.int64)
    table = np.zeros((s, m), dtype=base.dtype)
    row = base.copy()
    for j in range(s):
        table[j] = row
        row = row * base % p
    if db is not None:
        scale = np.zeros(m, dtype=table.dtype)
        nv = int(valid.sum())
        scale[:nv] = [int(v) % p for v in db[k * m : k * m + nv]]
        table = table * scale[None, :] % p
    return table


def diag_vector(table: np.ndarray, g: int, b: int, baby: int, s_pad: int, m: int) -> np.ndarray:
    """compress.py:186-195."""
    pos = np.arange(m)
    rows = (pos - g * baby) % s_pad
    cols = (pos + b) % m
    live = rows < table.shape[0]
    out = np.zeros(m, dtype=np.int64)
    out[live] = table[rows[live], cols[live]]
    return out


@dataclass
class OPlan:
    baby: int
    giant: int
    fold: tuple
    diagonals: list  # [t][g*baby+b] -> rows (2, m) int64 or None
    output_mask: np.ndarray


def build_plan(N: int, s: int, n: int, p: int, db=None) -> OPlan:
    """compress.py:198-255, mode "packed"; `db` = the cleartext database of
    precompute_masked_matrix (bottom lane evaluates D = C diag(DB))."""
    m = n // 2
    s_pad = 1 << (s - 1).bit_length()
    baby, giant = bsgs_shape(s)
    B = -(-N // m)
    diagonals = []
    for t in range(B):
        tab = vandermonde_block(N, s, p, m, t)
        tab_d = tab if db is None else vandermonde_block(N, s, p, m, t, db)
        per = []
        for g in range(giant):
            for b in range(baby):
                r0 = diag_vector(tab, g, b, baby, s_pad, m)
                r1 = r0 if db is None else diag_vector(tab_d, g, b, baby, s_pad, m)
                if not np.any(r0) and not np.any(r1):
                    per.append(None)
                else:
                    per.append(np.stack([r0, r1]) % p)
        diagonals.append(per)
    fold = []
    step = s_pad
    while step < m:
        fold.append(step)
        step <<= 1
    row = np.array([1] * s + [0] * (m - s), dtype=np.int64)
    return OPlan(baby, giant, tuple(fold), diagonals, np.stack([row, row]))


def encode_vector(values, N: int, n: int, p: int) -> list[np.ndarray]:
    """compress.py:318-329 + SlotMatrix.from_vector (heiface.py:105-113)."""
    vals = list(values)
    assert len(vals) == N
    half = n // 2
    out = []
    C = -(-(-(-N // half)) // 2)
    for t in range(C):
        chunk = vals[t * n : (t + 1) * n]
        chunk = chunk + [0] * (n - len(chunk))
        out.append(np.array([chunk[:half], chunk[half:]], dtype=np.int64) % p)
    return out


def encrypt_vector(values, N: int, be: OracleBgv, keys: OKeys) -> list[OCt]:
    return [be.encrypt(m, keys) for m in encode_vector(values, N, be.n, be.p)]


def pack_pair(cv, cd, N: int, be: OracleBgv, keys: OKeys) -> list[OCt]:
    """compress.py:338-367."""
    m = be.slots
    B = -(-N // m)
    top = np.array([[1] * m, [0] * m], dtype=np.int64)
    bot = np.array([[0] * m, [1] * m], dtype=np.int64)
    out = []
    for j in range(B):
        src = j // 2
        if j % 2 == 0:
            u = be.add(be.mul_plain(cv[src], top), be.rot_col(be.mul_plain(cd[src], top), keys))
        else:
            u = be.add(be.rot_col(be.mul_plain(cv[src], bot), keys), be.mul_plain(cd[src], bot))
        out.append(u)
    return out


def bsgs_matvec(plan: OPlan, inputs, be: OracleBgv, keys: OKeys) -> OCt:
    """compress.py:273-310 (packed mode)."""
    baby, giant = plan.baby, plan.giant
    acc = [None] * giant
    for t, ct in enumerate(inputs):
        rotated = [ct]
        for b in range(1, baby):
            rotated.append(be.rot_row(ct, b, keys))
        diags = plan.diagonals[t]
        for g in range(giant):
            for b in range(baby):
                d = diags[g * baby + b]
                if d is None:
                    continue
                prod = be.mul_plain(rotated[b], d)
                acc[g] = prod if acc[g] is None else be.add(acc[g], prod)
    res = acc[0]
    for g in range(1, giant):
        if acc[g] is None:
            continue
        part = be.rot_row(acc[g], (g * baby) % be.slots, keys)
        res = part if res is None else be.add(res, part)
    for amount in plan.fold:
        res = be.add(res, be.rot_row(res, amount, keys))
    return be.mul_plain(res, plan.output_mask)


def comp(cd, N: int, s: int, be: OracleBgv, keys: OKeys, index_hint=None, masked_db=None) -> OCt:
    """compress.py:488-514, packed: with an index hint, or (comp_masked,
    compress.py:521-530) with masked_db, where cd is the index vector."""
    cv = list(cd) if masked_db is not None else list(index_hint)
    u = pack_pair(cv, cd, N, be, keys)
    plan = build_plan(N, s, be.n, be.p, masked_db)
    return bsgs_matvec(plan, u, be, keys)


def mask(cv, db, N: int, be: OracleBgv) -> list[OCt]:
    """pdq.mask (pdq.py:238-245): d_i = v_i * value_i, plaintext multiply by
    the cleartext database block matrices (_db_block_matrices, pdq.py:207-208)."""
    return [be.mul_plain(c, m) for c, m in zip(cv, encode_vector(db, N, be.n, be.p))]


def serialize_answer(be: OracleBgv, ct: OCt, s: int) -> bytes:
    """CompressedAnswer.serialize (compress.py:403-416), packed, one ct."""
    head = struct.pack("<HIBBBIIB", 1, s, 1, 0, 1, 0, 0, 1)
    blob = be.serialize_ciphertext(ct)
    return head + struct.pack("<I", len(blob)) + blob


def plant_sparse(rng: random.Random, N: int, s: int, p: int) -> list[int]:
    """bench.py:65-69 (dense form)."""
    support = sorted(rng.sample(range(1, N + 1), s))
    d = [0] * N
    for i in support:
        d[i - 1] = rng.randrange(1, p)
    return d


def masked_payload(N: int, s: int, p: int, seed: int):
    """comp_masked fixture recipe (oracle/make_golden.py): the encrypted index
    vector's support and a cleartext database value on every position."""
    rng = random.Random(seed)
    support = sorted(rng.sample(range(1, N + 1), s))
    db = [rng.randrange(1, p) for _ in range(N)]
    dense = [0] * N
    for i in support:
        dense[i - 1] = db[i - 1]
    return support, db, dense


def expected_slots(dense, s: int, p: int) -> tuple[list[int], list[int]]:
    """What Comp must decrypt to: w_j = sum_i i^(j+1) v_i, e_j = sum_i i^(j+1) d_i
    (compress.py:1-16)."""
    w = [0] * s
    e = [0] * s
    for i, v in enumerate(dense, start=1):
        if v:
            pw = i % p
            for j in range(s):
                w[j] = (w[j] + pw) % p
                e[j] = (e[j] + pw * v) % p
                pw = pw * i % p
    return w, e


def sha256(b: bytes) -> str:
    return hashlib.sha256(b).hexdigest()
