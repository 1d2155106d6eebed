"""B200 BGV backend: the reference's `BgvBackend` surface (bgv.py:321-931)
with every ring operation executed by libhcomp on the GPU.

Host side (this file): parameter/chain setup, the random sampling of keygen
and encryption (one `random.Random(seed)` consumed in exactly the
reference's order, bgv.py:338,398-414,464-557, so keys and ciphertexts are
bit-identical to the reference's for the same seed), the deterministic
noise-bits bookkeeping and the op counters.  Device side (libhcomp): NTTs,
pointwise ring arithmetic, modulus switching, key switching and the fused
Comp schedule.

Ciphertexts carry RNS residues: `payload.res` is uint64[2][level+1][n], row k
modulo level_prime(k) (bgv.py:104-106).  `payload.c0` / `payload.c1` give the
reference's composite-modulus integer lists on demand.
"""

from __future__ import annotations

import ctypes
import hashlib
import os
import math
import struct
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from .params import (
    BACKEND_BGV,
    BackendMismatch,
    HeParams,
    LevelExhausted,
    MissingRotationKey,
    NoiseOverflow,
    find_chain_primes,
)

CBD_HALF_WIDTH = 21  # bgv.py:48
_OBJ_KIND_CIPHERTEXT = 0x01
MAGIC = b"HCV1"
FORMAT_VERSION = 1


# ---------------------------------------------------------------------------
# data model (heiface.py:73-248, bgv.py:287-312)
# ---------------------------------------------------------------------------


class SlotMatrix:
    """2 x (n/2) matrix over Z_p (heiface.py:73-171, the parts Comp uses)."""

    __slots__ = ("p", "rows")

    def __init__(self, p: int, rows: np.ndarray):
        if rows.shape[0] != 2:
            raise ValueError("slot matrix has exactly two rows")
        self.p = p
        self.rows = rows

    @classmethod
    def zeros(cls, n: int, p: int) -> "SlotMatrix":
        return cls(p, np.zeros((2, n // 2), dtype=np.int64))

    @classmethod
    def from_rows(cls, row0, row1, p: int) -> "SlotMatrix":
        return cls(p, np.array([list(row0), list(row1)], dtype=np.int64) % p)

    @classmethod
    def from_vector(cls, values, n: int, p: int) -> "SlotMatrix":
        half = n // 2
        vals = list(values)
        if len(vals) > n:
            raise ValueError(f"vector of length {len(vals)} does not fit n={n}")
        vals = vals + [0] * (n - len(vals))
        return cls.from_rows(vals[:half], vals[half:], p)

    @property
    def cols(self) -> int:
        return self.rows.shape[1]

    def __eq__(self, other) -> bool:
        return (
            isinstance(other, SlotMatrix)
            and self.p == other.p
            and self.rows.shape == other.rows.shape
            and bool(np.all(self.rows == other.rows))
        )

    def __repr__(self) -> str:
        return f"SlotMatrix(p={self.p}, shape={self.rows.shape})"


@dataclass
class OpCounters:
    """heiface.py:174-200."""

    keyswitches: int = 0
    ct_mults: int = 0
    pt_mults: int = 0
    adds: int = 0

    def snapshot(self) -> "OpCounters":
        return OpCounters(self.keyswitches, self.ct_mults, self.pt_mults, self.adds)

    def delta(self, earlier: "OpCounters") -> "OpCounters":
        return OpCounters(
            self.keyswitches - earlier.keyswitches,
            self.ct_mults - earlier.ct_mults,
            self.pt_mults - earlier.pt_mults,
            self.adds - earlier.adds,
        )

    def as_dict(self) -> dict[str, int]:
        return {
            "keyswitches": self.keyswitches,
            "ct_mults": self.ct_mults,
            "pt_mults": self.pt_mults,
            "adds": self.adds,
        }


@dataclass(frozen=True)
class Ciphertext:
    """heiface.py:203-213."""

    backend_id: int
    key_id: bytes
    level: int
    payload: object

    def with_payload(self, payload: object, level: int | None = None) -> "Ciphertext":
        return replace(self, payload=payload, level=self.level if level is None else level)


@dataclass
class RnsPayload:
    """BgvPayload (bgv.py:287-291) in RNS form."""

    res: np.ndarray  # uint64[2][level+1][n], NTT domain
    noise_bits: float
    primes: tuple = ()

    def _compose(self, i: int) -> list[int]:
        return crt_compose(self.res[i], self.primes)

    @property
    def c0(self) -> list[int]:
        return self._compose(0)

    @property
    def c1(self) -> list[int]:
        return self._compose(1)


@dataclass
class KeySet:
    """heiface.py:216-248.  KSKs are uint64[D_L][2][L+1][n] (b_j, a_j) arrays."""

    backend_id: int
    params: HeParams
    key_id: bytes
    rotation_keys: dict
    col_swap_key: object | None
    relin_key: object | None
    public: object | None
    secret: object | None

    def public_only(self) -> "KeySet":
        return replace(self, secret=None)

    @property
    def rotation_amounts(self) -> frozenset[int]:
        return frozenset(self.rotation_keys)


@dataclass
class BgvPublic:
    pk_b: np.ndarray
    pk_a: np.ndarray


def crt_compose(res: np.ndarray, primes) -> list[int]:
    """Residue rows -> integers in [0, prod primes) (bgv.py:129-137)."""
    primes = [int(q) for q in primes]
    Q = math.prod(primes)
    acc = [0] * res.shape[-1]
    for k, q in enumerate(primes):
        Mi = Q // q
        c = Mi * pow(Mi, -1, q)
        row = res[k].tolist()
        acc = [a + int(v) * c for a, v in zip(acc, row)]
    return [a % Q for a in acc]


def write_envelope(backend_id: int, payload: bytes) -> bytes:
    return MAGIC + struct.pack("<BH", backend_id, FORMAT_VERSION) + payload


def read_envelope(data: bytes) -> tuple[int, int, bytes]:
    """heiface.py:273-279."""
    if len(data) < 7 or data[:4] != MAGIC:
        raise ValueError("not an HCV1 blob")
    backend_id, version = struct.unpack("<BH", data[4:7])
    if version != FORMAT_VERSION:
        raise ValueError(f"unsupported format version {version}")
    return backend_id, version, data[7:]


# ---------------------------------------------------------------------------
# tables shared with libhcomp (bgv.py:115-117, 170-174, 258-261, 367-377)
# ---------------------------------------------------------------------------


def bitrev_table(n: int) -> np.ndarray:
    bits = n.bit_length() - 1
    idx = np.arange(n, dtype=np.int64)
    out = np.zeros(n, dtype=np.int64)
    for b in range(bits):
        out |= ((idx >> b) & 1) << (bits - 1 - b)
    return out


def slot_index(n: int) -> np.ndarray:
    """_build_slot_map: NTT index of slot (r, c); index_of_exponent[e] =
    bitrev((e-1)/2) because NTT index i evaluates at psi^(2*bitrev(i)+1)."""
    br = bitrev_table(n)
    two_n = 2 * n
    half = n // 2
    e = np.ones(half, dtype=np.int64)
    for c in range(1, half):
        e[c] = e[c - 1] * 3 % two_n
    return np.stack([br[(e - 1) // 2], br[(two_n - e - 1) // 2]])


# ---------------------------------------------------------------------------
# backend
# ---------------------------------------------------------------------------


class HostRng:
    """random.Random(seed) restated natively (csrc/pyrng.hpp, CPython's
    MT19937): the reference backend's samplers (bgv.py:398-414) consume the
    same stream, so keys and ciphertexts stay bit-identical, ~100x faster than
    the Python loops."""

    def __init__(self, seed):
        if seed is None:  # random.Random(None): fresh entropy
            seed = int.from_bytes(os.urandom(32), "little")
        n = abs(int(seed))
        words = []
        while n:
            words.append(n & 0xFFFFFFFF)
            n >>= 32
        key = np.array(words or [0], dtype=np.uint32)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().hc_rng_create(_lib.ptr(key), len(key), ctypes.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                _lib.lib().hc_rng_destroy(self._h)
        except Exception:
            pass

    def getrandbits(self, k: int) -> int:
        w = np.zeros(max(1, (k + 31) // 32), dtype=np.uint32)
        _lib.check(_lib.lib().hc_rng_getrandbits(self._h, k, _lib.ptr(w)))
        return int.from_bytes(w.tobytes(), "little")

    def ternary(self, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        _lib.check(_lib.lib().hc_rng_ternary(self._h, n, _lib.ptr(out)))
        return out

    def cbd(self, n: int, k: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        _lib.check(_lib.lib().hc_rng_cbd(self._h, n, k, _lib.ptr(out)))
        return out

    def uniform(self, n: int, modulus: int, primes) -> np.ndarray:
        """[randrange(modulus) for _ in range(n)] as residues [len(primes)][n]."""
        kbits = modulus.bit_length()
        nw = (kbits + 31) // 32
        q = np.frombuffer(modulus.to_bytes(4 * nw, "little"), dtype=np.uint32).copy()
        pr = np.ascontiguousarray(primes, dtype=np.uint64)
        out = np.empty((len(pr), n), dtype=np.uint64)
        _lib.check(_lib.lib().hc_rng_uniform(self._h, n, _lib.ptr(q), nw, kbits, _lib.ptr(pr), len(pr), _lib.ptr(out)))
        return out


class B200BgvBackend:
    """BGV evaluation session on a B200 (reference: BgvBackend, bgv.py:321)."""

    backend_id = BACKEND_BGV
    name = "bgv-b200"

    def __init__(
        self,
        params: HeParams,
        seed: int | None = None,
        chain_bits: int = 54,
        ksw_base_bits: int = 16,
        chain_primes: list[int] | None = None,
        device: int = 0,
        noise_guard: bool = True,
    ):
        from .refcompat import he_params

        params = he_params(params)  # an hcpdq HeParams passes through
        if params.n != 8192:
            raise ValueError("the B200 backend supports n = 8192 only")
        if not (1 <= params.max_level <= 22):
            raise ValueError("the B200 backend supports max_level 1..22")
        if ksw_base_bits != 16:
            raise ValueError("ksw_base_bits must be 16")
        self.params = params
        self.counters = OpCounters()
        self._rng = HostRng(seed)
        self.w = ksw_base_bits
        self.noise_guard = noise_guard
        n, p = params.n, params.p
        primes = chain_primes or find_chain_primes(n, p, params.max_level + 1, chain_bits)
        self.chain_primes = tuple(sorted(primes, reverse=True))  # ModulusChain.primes
        L = params.max_level
        self.q = [self.chain_primes[L - k] for k in range(L + 1)]  # level order
        self.moduli = [math.prod(self.q[: l + 1]) for l in range(L + 1)]
        self.digits = [-(-self.moduli[l].bit_length() // self.w) for l in range(L + 1)]
        self.device = device
        self._h = None
        self._slot_index = slot_index(n)
        self._loaded_keys = None
        self._planned = None
        self._plan_gen = 0  # bumped whenever the device plan is rebuilt (hc_plan*)
        self._answer_db_tag = None

    # -- GPU context ------------------------------------------------------------

    def _ctx(self):
        if self._h is None:
            L = _lib.lib(self.params.max_level)
            h = ctypes.c_void_p()
            primes = np.asarray(self.q, dtype=np.uint64)
            _lib.check(
                L.hc_ctx_create(
                    self.params.n, self.params.max_level, _lib.ptr(primes), self.params.p, self.w,
                    self.device, ctypes.byref(h),
                )
            )
            self._h = h
        return self._h

    def close(self) -> None:
        if self._h is not None:
            _lib.lib(self.params.max_level).hc_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _pidx(self, rows: int, level: int) -> np.ndarray:
        return np.ascontiguousarray(np.resize(np.arange(level + 1, dtype=np.int32), rows))

    def ntt(self, a: np.ndarray, level: int, inverse: bool = False) -> np.ndarray:
        """NttContext.fwd/inv per RNS row on the GPU; a: [..., level+1, n]."""
        a = np.ascontiguousarray(a, dtype=np.uint64).copy()
        rows = a.size // self.params.n
        pidx = self._pidx(rows, level)
        _lib.check(_lib.lib(self.params.max_level).hc_ntt(self._ctx(), _lib.ptr(a), rows, _lib.ptr(pidx), 1 if inverse else 0))
        return a

    def ntt_p(self, a: np.ndarray, inverse: bool) -> np.ndarray:
        a = np.ascontiguousarray(a, dtype=np.uint64).copy().reshape(1, -1)
        pidx = np.array([_lib.lib(self.params.max_level).hc_plain_row()], dtype=np.int32)
        _lib.check(_lib.lib(self.params.max_level).hc_ntt(self._ctx(), _lib.ptr(a), 1, _lib.ptr(pidx), 1 if inverse else 0))
        return a[0]

    def pointwise(self, x: np.ndarray, y: np.ndarray, level: int, op: str) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.uint64)
        y = np.ascontiguousarray(np.broadcast_to(y, x.shape), dtype=np.uint64)
        out = np.empty_like(x)
        rows = x.size // self.params.n
        pidx = self._pidx(rows, level)
        code = {"mul": 0, "add": 1, "sub": 2}[op]
        _lib.check(
            _lib.lib(self.params.max_level).hc_pointwise(self._ctx(), _lib.ptr(x), _lib.ptr(y), _lib.ptr(out), rows, _lib.ptr(pidx), code)
        )
        return out

    # -- residues --------------------------------------------------------------

    def small_residues(self, vals, level: int) -> np.ndarray:
        v = np.asarray(vals, dtype=np.int64)
        return np.stack([np.mod(v, np.int64(q)).astype(np.uint64) for q in self.q[: level + 1]])

    def big_residues(self, vals, level: int) -> np.ndarray:
        return np.stack(
            [np.fromiter((int(x) % q for x in vals), dtype=np.uint64, count=len(vals)) for q in self.q[: level + 1]]
        )

    # -- slots (bgv.py:379-394) --------------------------------------------------

    def _check_plain(self, m: SlotMatrix) -> None:
        if m.p != self.params.p or m.cols != self.params.slots:
            raise BackendMismatch("plaintext does not match backend parameters")

    def _check_ct(self, c: Ciphertext) -> None:
        if c.backend_id != self.backend_id:
            raise BackendMismatch("ciphertext from a different backend")

    def _check_keys(self, c: Ciphertext, keys: KeySet) -> None:
        self._check_ct(c)
        if keys.backend_id != self.backend_id or keys.key_id != c.key_id:
            raise BackendMismatch("key set does not match ciphertext")

    def slot_encode(self, m: SlotMatrix) -> np.ndarray:
        evals = np.zeros(self.params.n, dtype=np.uint64)
        rows = np.asarray(m.rows, dtype=np.int64) % self.params.p
        evals[self._slot_index[0]] = rows[0]
        evals[self._slot_index[1]] = rows[1]
        return self.ntt_p(evals, inverse=True)

    def slot_decode(self, coeffs) -> SlotMatrix:
        ev = self.ntt_p(np.asarray(coeffs, dtype=np.uint64) % np.uint64(self.params.p), inverse=False)
        rows = np.stack([ev[self._slot_index[0]], ev[self._slot_index[1]]]).astype(np.int64)
        return SlotMatrix(self.params.p, rows)

    def plain_ntt(self, m: SlotMatrix, level: int) -> np.ndarray:
        """_plain_ntt (bgv.py:452-460): slot_encode then NTT mod Q_level."""
        self._check_plain(m)
        coeffs = self.slot_encode(m)
        return self.ntt(np.broadcast_to(coeffs, (level + 1, self.params.n)), level)

    # -- sampling (bgv.py:398-414) ---------------------------------------------

    def _sample_ternary(self) -> list[int]:
        return [int(v) for v in self._rng.ternary(self.params.n)]

    def _sample_cbd(self) -> np.ndarray:
        return self._rng.cbd(self.params.n, CBD_HALF_WIDTH)

    def _sample_uniform_ntt(self, level: int) -> np.ndarray:
        return self._rng.uniform(self.params.n, self.moduli[level], self.q[: level + 1])

    # -- keys (bgv.py:464-520) ----------------------------------------------------

    def _coeff_automorphism(self, coeffs, t: int) -> np.ndarray:
        n = self.params.n
        c = np.asarray(coeffs, dtype=np.int64)
        j = (np.arange(n, dtype=np.int64) * t) % (2 * n)
        out = np.zeros(n, dtype=np.int64)
        hi = j >= n
        out[j[~hi]] = c[~hi]
        out[j[hi] - n] = -c[hi]
        return out

    def keygen(self, rotation_amounts, col_swap: bool = True) -> KeySet:
        params = self.params
        n, p, L = params.n, params.p, params.max_level
        amounts = sorted(set(int(r) for r in rotation_amounts))
        for r in amounts:
            if not (0 <= r < params.slots):
                raise ValueError(f"rotation amount {r} outside [0, n/2)")
        s = self._sample_ternary()
        s_ntt = self.ntt(self.small_residues(s, L), L)
        pk_a = self._sample_uniform_ntt(L)
        e = self._sample_cbd()
        pe_ntt = self.ntt(self.small_residues(p * e, L), L)
        pk_b = self.pointwise(pe_ntt, self.pointwise(pk_a, s_ntt, L, "mul"), L, "sub")
        D = self.digits[L]
        # Deep protocol chains (max_level > 4: 75 digits x 22 primes at level 21)
        # keep only the key slice key switching ever reads -- the first D_3
        # digits on the 4 smallest primes (_KskPair.at_level at levels <= 3,
        # bgv.py:304-312) -- while every digit's samples are still drawn, so
        # the random stream, key_id and all later encryptions stay the
        # reference's.  Shallow chains keep the whole key.
        deep = L > 4
        kl = 3 if deep else L  # key rows 0..kl (level order)
        dk = self.digits[3] if deep else D
        s_k = s_ntt[: kl + 1]

        def make_ksk(target_res: np.ndarray) -> np.ndarray:
            target_ntt = self.ntt(target_res[: kl + 1], kl)
            ksk = np.empty((dk, 2, kl + 1, n), dtype=np.uint64)
            pe = np.empty((dk, kl + 1, n), dtype=np.uint64)
            for j in range(D):  # the reference's sampling order: a_j then e_j
                a_j = self._rng.uniform(n, self.moduli[L], self.q[: kl + 1])  # randrange(Q_L) residues
                e_j = self._sample_cbd()
                if j < dk:
                    ksk[j, 1] = a_j
                    pe[j] = self.small_residues(p * e_j, kl)
            ksk[:, 0] = self.ntt(pe, kl)  # p*e_j in one batched transform, finished below
            # b_j = p e_j - a_j s + 2^(16 j) t  (bgv.py:488-493), batched on the GPU
            shifts = np.array(
                [[pow(2, self.w * j, int(q)) for q in self.q[: kl + 1]] for j in range(dk)], dtype=np.uint64
            )
            shift_t = self.pointwise(
                np.broadcast_to(target_ntt, (dk, kl + 1, n)), np.repeat(shifts[:, :, None], n, axis=2), kl, "mul"
            )
            a_s = self.pointwise(ksk[:, 1], np.broadcast_to(s_k, (dk, kl + 1, n)), kl, "mul")
            ksk[:, 0] = self.pointwise(self.pointwise(ksk[:, 0], a_s, kl, "sub"), shift_t, kl, "add")
            return ksk

        s_sq = self.ntt(self.pointwise(s_k, s_k, kl, "mul"), kl, inverse=True)
        relin = make_ksk(s_sq)
        two_n = 2 * n
        rot_keys = {}
        for r in amounts:
            if r == 0:
                continue
            t = pow(3, r, two_n)
            rot_keys[r] = (t, make_ksk(self.small_residues(self._coeff_automorphism(s, t), kl)))
        col_key = None
        if col_swap:
            t = two_n - 1
            col_key = (t, make_ksk(self.small_residues(self._coeff_automorphism(s, t), kl)))
        return KeySet(
            backend_id=self.backend_id,
            params=params,
            key_id=self._rng.getrandbits(128).to_bytes(16, "little"),
            rotation_keys=rot_keys,
            col_swap_key=col_key,
            relin_key=relin,
            public=BgvPublic(pk_b, pk_a),
            secret=s,
        )

    # -- encryption (bgv.py:533-575) -----------------------------------------------

    def _fresh_noise_bits(self) -> float:
        n, p = self.params.n, self.params.p
        return math.log2(p) + math.log2(CBD_HALF_WIDTH) + math.log2(2 * n + 2)

    def _payload(self, res: np.ndarray, bits: float, level: int) -> RnsPayload:
        return RnsPayload(res, bits, tuple(self.q[: level + 1]))

    def encrypt(self, m: SlotMatrix, keys: KeySet) -> Ciphertext:
        self._check_plain(m)
        if keys.public is None:
            raise BackendMismatch("key set lacks public key material")
        L, p = self.params.max_level, self.params.p
        m_coeffs = self.slot_encode(m).astype(np.int64)
        u_ntt = self.ntt(self.small_residues(self._sample_ternary(), L), L)
        e0 = self._sample_cbd()
        e1 = self._sample_cbd()
        body = self.ntt(np.stack([self.small_residues(p * e0 + m_coeffs, L), self.small_residues(p * e1, L)]), L)
        pk = np.stack([keys.public.pk_b, keys.public.pk_a])
        c = self.pointwise(self.pointwise(pk, np.broadcast_to(u_ntt, pk.shape), L, "mul"), body, L, "add")
        return Ciphertext(self.backend_id, keys.key_id, L, self._payload(c, self._fresh_noise_bits(), L))

    def decrypt(self, c: Ciphertext, keys: KeySet) -> SlotMatrix:
        self._check_keys(c, keys)
        if keys.secret is None:
            raise BackendMismatch("decryption requires the secret key")
        l = c.level
        if l <= 3:  # one device call: phase, INTT, CRT lift, centring, slot decode (hc_decrypt)
            ct = np.ascontiguousarray(c.payload.res, dtype=np.uint64)
            sec = np.ascontiguousarray(keys.secret, dtype=np.int64)
            rows = np.empty((2, self.params.slots), dtype=np.int64)
            _lib.check(_lib.lib(self.params.max_level).hc_decrypt(self._ctx(), _lib.ptr(ct), l, _lib.ptr(sec), _lib.ptr(rows)))
            return SlotMatrix(self.params.p, rows)
        s_ntt = self.ntt(self.small_residues(keys.secret, l), l)
        res = c.payload.res
        phase = self.ntt(self.pointwise(res[0], self.pointwise(res[1], s_ntt, l, "mul"), l, "add"), l, inverse=True)
        Q = self.moduli[l]
        half = Q >> 1
        p = self.params.p
        if l == 0:
            v = phase[0].astype(object)
            ints = v
        else:
            ints = crt_compose(phase, self.q[: l + 1])
        centered = np.array([(int(x) - Q if int(x) > half else int(x)) % p for x in ints], dtype=np.uint64)
        return self.slot_decode(centered)

    # -- noise bookkeeping (bgv.py:421-429, 606-607, 640-646, 660, 724, 745) -------

    def _threshold_bits(self, level: int) -> float:
        return self.moduli[level].bit_length() - 1

    def _check_noise(self, bits: float, level: int) -> float:
        if self.noise_guard and bits >= self._threshold_bits(level):
            raise NoiseOverflow(f"noise estimate 2^{bits:.1f} crosses the level-{level} threshold")
        return bits

    def _ms_bits(self, bits: float, level: int) -> float:
        q = self.q[level]
        floor_bits = math.log2(self.params.p) + math.log2(self.params.n)
        return max(bits - math.log2(q), floor_bits) + 1

    def _ks_noise(self, level: int) -> float:
        return (
            math.log2(self.params.p)
            + math.log2(self.digits[level])
            + self.w
            + math.log2(self.params.n)
            + math.log2(CBD_HALF_WIDTH)
        )

    # -- single homomorphic operations (bgv.py:651-770) ------------------------------

    def add(self, c1: Ciphertext, c2: Ciphertext) -> Ciphertext:
        self._check_ct(c1)
        self._check_ct(c2)
        if c1.key_id != c2.key_id:
            raise BackendMismatch("ciphertexts under different key sets")
        lvl = min(c1.level, c2.level)
        c1 = self._at_level(c1, lvl)
        c2 = self._at_level(c2, lvl)
        self.counters.adds += 1
        bits = self._check_noise(max(c1.payload.noise_bits, c2.payload.noise_bits) + 1, lvl)
        res = self.pointwise(c1.payload.res, c2.payload.res, lvl, "add")
        return Ciphertext(self.backend_id, c1.key_id, lvl, self._payload(res, bits, lvl))

    def _at_level(self, c: Ciphertext, level: int) -> Ciphertext:
        while c.level > level:
            one = SlotMatrix(self.params.p, np.ones((2, self.params.slots), dtype=np.int64))
            # _mod_switch_once == mul_plain by the all-ones plaintext minus its
            # noise/counter bookkeeping (slot_encode(1) is the constant 1)
            res = self._mul_plain_res(c.payload.res, c.level, self.plain_ntt(one, c.level))
            bits = self._ms_bits(c.payload.noise_bits, c.level)
            c = Ciphertext(self.backend_id, c.key_id, c.level - 1, self._payload(res, bits, c.level - 1))
        return c

    def _mul_plain_res(self, res: np.ndarray, level: int, pt: np.ndarray) -> np.ndarray:
        n = self.params.n
        ct = np.ascontiguousarray(res, dtype=np.uint64)
        pt = np.ascontiguousarray(pt, dtype=np.uint64)
        out = np.empty((2, level, n), dtype=np.uint64)
        _lib.check(_lib.lib(self.params.max_level).hc_mul_plain(self._ctx(), _lib.ptr(ct), level, _lib.ptr(pt), _lib.ptr(out)))
        return out

    def mul_plain(self, c: Ciphertext, m: SlotMatrix) -> Ciphertext:
        self._check_ct(c)
        self._check_plain(m)
        lvl = c.level
        if lvl < 1:
            raise LevelExhausted("plaintext multiply at level 0")
        pt = self.plain_ntt(m, lvl)
        bits = c.payload.noise_bits + math.log2(self.params.p) + math.log2(self.params.n)
        self._check_noise(bits, lvl)
        self.counters.pt_mults += 1
        res = self._mul_plain_res(c.payload.res, lvl, pt)
        return Ciphertext(self.backend_id, c.key_id, lvl - 1, self._payload(res, self._ms_bits(bits, lvl), lvl - 1))

    def _load_keys(self, keys: KeySet) -> None:
        if self._loaded_keys is keys:
            return
        L = _lib.lib(self.params.max_level)
        h = self._ctx()
        _lib.check(L.hc_clear_keys(h))
        entries = list(keys.rotation_keys.values())
        if keys.col_swap_key is not None:
            entries.append(keys.col_swap_key)
        for t, ksk in entries:
            arr = np.ascontiguousarray(ksk, dtype=np.uint64)  # [digits][2][rows][n]
            _lib.check(L.hc_load_ksk_slice(h, int(t), _lib.ptr(arr), arr.shape[0], arr.shape[2]))
        self._loaded_keys = keys
        self._planned = None

    def _apply_galois(self, c: Ciphertext, t: int, keys: KeySet) -> Ciphertext:
        lvl = c.level
        if lvl < 1:
            raise ValueError("the B200 backend key-switches at levels 1..max_level")
        self._load_keys(keys)
        ct = np.ascontiguousarray(c.payload.res, dtype=np.uint64)
        out = np.empty_like(ct)
        _lib.check(_lib.lib(self.params.max_level).hc_rotate(self._ctx(), _lib.ptr(ct), lvl, int(t), _lib.ptr(out)))
        bits = self._check_noise(max(c.payload.noise_bits, self._ks_noise(lvl)) + 1, lvl)
        self.counters.keyswitches += 1
        return Ciphertext(self.backend_id, c.key_id, lvl, self._payload(out, bits, lvl))

    def rot_row(self, c: Ciphertext, r: int, keys: KeySet) -> Ciphertext:
        self._check_keys(c, keys)
        r = r % self.params.slots
        if r == 0:
            return Ciphertext(self.backend_id, c.key_id, c.level, self._payload(c.payload.res.copy(), c.payload.noise_bits, c.level))
        entry = keys.rotation_keys.get(r)
        if entry is None:
            raise MissingRotationKey(f"rotation by {r} was not declared at keygen")
        return self._apply_galois(c, entry[0], keys)

    def rot_col(self, c: Ciphertext, keys: KeySet) -> Ciphertext:
        self._check_keys(c, keys)
        if keys.col_swap_key is None:
            raise MissingRotationKey("column-swap key was not declared at keygen")
        return self._apply_galois(c, keys.col_swap_key[0], keys)

    # -- serialization (bgv.py:774-790) -------------------------------------------

    def _words(self, level: int) -> int:
        return -(-self.moduli[level].bit_length() // 64)

    def serialize_ciphertext(self, c: Ciphertext) -> bytes:
        self._check_ct(c)
        level = c.level
        W = self._words(level)
        head = struct.pack("<BBIQB", _OBJ_KIND_CIPHERTEXT, level, self.params.n, self.params.p, self.params.max_level)
        parts = [head, c.key_id, struct.pack("<d", c.payload.noise_bits)]
        coeffs = self.ntt(c.payload.res, level, inverse=True)
        if level == 0:
            for i in range(2):
                parts.append(np.ascontiguousarray(coeffs[i, 0], dtype="<u8").tobytes())
        else:
            for i in range(2):
                for x in crt_compose(coeffs[i], self.q[: level + 1]):
                    parts.append(int(x).to_bytes(8 * W, "little"))
        return write_envelope(self.backend_id, b"".join(parts))

    def deserialize_ciphertext(self, data: bytes) -> Ciphertext:
        """bgv.py:792-814: coefficient-domain integers -> RNS residues -> NTT
        on the GPU (the inverse of serialize_ciphertext)."""
        backend_id, _, payload = read_envelope(data)
        if backend_id != self.backend_id:
            raise BackendMismatch("blob was produced by a different backend")
        kind, level, n, p, max_level = struct.unpack("<BBIQB", payload[:15])
        if kind != _OBJ_KIND_CIPHERTEXT:
            raise ValueError("blob is not a ciphertext")
        if (n, p, max_level) != (self.params.n, self.params.p, self.params.max_level):
            raise BackendMismatch("ciphertext parameters do not match backend")
        key_id = bytes(payload[15:31])
        (noise_bits,) = struct.unpack("<d", payload[31:39])
        W = self._words(level)
        body = np.frombuffer(payload, dtype="<u8", count=2 * n * W, offset=39).reshape(2, n, W)
        res = np.empty((2, level + 1, n), dtype=np.uint64)
        for k, q in enumerate(self.q[: level + 1]):
            # sum_i w_i 2^(64 i) mod q, limb by limb (every limb < 2^64)
            acc = np.zeros((2, n), dtype=object)
            for i in range(W):
                acc = acc + body[:, :, i].astype(object) * (pow(2, 64 * i, q))
            res[:, k] = (acc % q).astype(np.uint64)
        res = self.ntt(res, level)
        return Ciphertext(self.backend_id, key_id, level, self._payload(res, noise_bits, level))

    # -- the fused Comp (compress.py:488-514) ------------------------------------------

    def plan(
        self,
        N: int,
        s: int,
        keys: KeySet,
        chunk_blocks: int = 0,
        db: np.ndarray | None = None,
        block_range: tuple[int, int] | None = None,
        share_with: "B200BgvBackend | None" = None,
    ) -> None:
        """Device plan for (N, s); `db` (uint64[N], mod p) selects comp_masked's D = C diag(DB).

        block_range=(b0, b1): a sharded rank's plan (hc_plan_range), only its
        blocks' diagonals and input ciphertexts on the device.  share_with: a
        backend whose current (N, s) plan's plaintexts this one reuses
        (hc_plan_shared; independent queries over one database)."""
        self._load_keys(keys)
        rng = None if block_range is None else (int(block_range[0]), int(block_range[1]))
        src = None
        if share_with is not None:
            if db is not None or rng is not None:
                raise ValueError("a shared plan is a whole-matrix hint-path plan")
            sp = share_with._planned
            if sp is None or sp[:2] != (N, s) or sp[3] is not None or sp[4] is not None:
                raise ValueError("share_with has no hint-path plan for this (N, s)")
            src = share_with
        tag = (N, s, chunk_blocks, None if db is None else hashlib.sha256(db.tobytes()).digest(), rng, id(src) if src else None)
        if self._planned != tag:
            L = _lib.lib(self.params.max_level)
            if src is not None:
                _lib.check(L.hc_plan_shared(self._ctx(), src._ctx(), chunk_blocks))
                self._plan_src = src  # keep the source alive beside the shared buffers
            elif rng is not None:
                _lib.check(L.hc_plan_range(self._ctx(), N, s, chunk_blocks, rng[0], rng[1]))
            elif db is None:
                _lib.check(L.hc_plan(self._ctx(), N, s, chunk_blocks))
            else:
                db = np.ascontiguousarray(db, dtype=np.uint64)
                _lib.check(_lib.lib(self.params.max_level).hc_plan_masked(self._ctx(), N, s, chunk_blocks, _lib.ptr(db)))
            self._planned = tag
            # a new device Plan drops the previous plan's answer() mask
            # plaintexts (hc_answer_db), so their cache tag is stale too
            self._plan_gen += 1
            self._answer_db_tag = None

    def answer_db(self, db_mod_p: np.ndarray, level: int) -> None:
        """Mask plaintexts of the cleartext database for the current plan (hc_answer_db)."""
        db = np.ascontiguousarray(db_mod_p, dtype=np.uint64)
        tag = (self._plan_gen, level, hashlib.sha256(db.tobytes()).digest())
        if self._answer_db_tag != tag:
            _lib.check(_lib.lib(self.params.max_level).hc_answer_db(self._ctx(), level, _lib.ptr(db)))
            self._answer_db_tag = tag

    def plan_info(self) -> dict:
        info = np.zeros(8, dtype=np.int64)
        _lib.check(_lib.lib(self.params.max_level).hc_plan_info(self._ctx(), _lib.ptr(info)))
        keys = ["B", "C", "baby", "giant", "F", "s_pad", "live_diagonals", "kernel_launches"]
        return dict(zip(keys, (int(x) for x in info)))
