"""Parameter objects, shapes and exceptions of the reference API
(heiface.py:25-70, compress.py:39-100, bgv.py:52-76), restated so the
package is self-contained on the GPU box (the reference is not installed
there).  Names, argument meaning and error behaviour follow the reference.
"""

from __future__ import annotations

import math
from dataclasses import dataclass


class BackendMismatch(ValueError):
    """Ciphertexts/keys from different backends or key sets were mixed (heiface.py:25)."""


class LevelExhausted(RuntimeError):
    """An operation required a multiplicative level that is not available (heiface.py:29)."""


class MissingRotationKey(KeyError):
    """Rotation by an amount that was not declared at keygen (heiface.py:33)."""


class NoiseOverflow(RuntimeError):
    """The tracked noise bound crossed the decryption threshold (bgv.py:56)."""


class NoNttPrimes(RuntimeError):
    """No suitable NTT-friendly prime chain exists in the search window (bgv.py:52)."""


BACKEND_SIMULATOR = 0x01
BACKEND_BGV = 0x02

_MR_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)


def is_prime(n: int) -> bool:
    """Deterministic Miller-Rabin (exact below 3.3e24; chain primes are 54-bit)."""
    n = int(n)
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


@dataclass(frozen=True)
class HeParams:
    """Ring dimension, plaintext modulus and depth budget (heiface.py:50-70)."""

    n: int
    p: int
    max_level: int

    def __post_init__(self):
        if self.n < 4 or self.n & (self.n - 1):
            raise ValueError(f"n={self.n} must be a power of two >= 4")
        if not is_prime(self.p):
            raise ValueError(f"p={self.p} must be prime")
        if self.p % (2 * self.n) != 1:
            raise ValueError(f"p={self.p} must satisfy p = 1 (mod 2n = {2 * self.n})")
        if self.max_level < 1:
            raise ValueError("max_level must be >= 1")

    @property
    def slots(self) -> int:
        return self.n // 2


@dataclass(frozen=True)
class CompressionParams:
    """Vector length, sparsity bound, HE parameters (compress.py:39-73)."""

    N: int
    s: int
    he: HeParams

    def __post_init__(self):
        if self.N < 1:
            raise ValueError("N must be positive")
        if self.s < 1:
            raise ValueError("s must be positive")
        if self.he.p <= self.N:
            raise ValueError(f"p={self.he.p} must exceed N={self.N}")
        if 2 * self.s > self.he.n:
            raise ValueError(f"2s={2 * self.s} must fit the {self.he.n} slots of one ciphertext")

    @property
    def block_width(self) -> int:
        return self.he.slots

    @property
    def num_blocks(self) -> int:
        return -(-self.N // self.block_width)

    @property
    def num_ciphertexts(self) -> int:
        return -(-self.num_blocks // 2)

    @property
    def s_pad(self) -> int:
        return 1 << (self.s - 1).bit_length()


def bsgs_shape(s: int) -> tuple[int, int]:
    """(baby, giant) of compress.py:76-84."""
    s_pad = 1 << (s - 1).bit_length()
    log_target = ((2 * s_pad).bit_length() - 1) / 2
    baby = 1 << int(log_target)
    baby = min(max(baby, 1), s_pad)
    return baby, s_pad // baby


def plan_rotation_amounts(s: int, n: int) -> tuple[list[int], bool]:
    """Row-rotation amounts and the col-swap requirement (compress.py:87-100)."""
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


def fold_amounts(s_pad: int, m: int) -> list[int]:
    out = []
    step = s_pad
    while step < m:
        out.append(step)
        step <<= 1
    return out


def find_chain_primes(n: int, p: int, count: int, bits: int = 54) -> list[int]:
    """`count` primes = 1 (mod 2n) and = 1 (mod p), largest first (bgv.py:60-76)."""
    step = 2 * n * p // math.gcd(2 * n, p)
    top = (1 << bits) - 1
    cand = top - (top - 1) % step
    out: list[int] = []
    floor = 1 << (bits - 1)
    while len(out) < count and cand > floor:
        if is_prime(cand):
            out.append(int(cand))
        cand -= step
    if len(out) < count:
        raise NoNttPrimes(f"could not find {count} primes = 1 (mod {step}) of {bits} bits")
    return out
