"""TEST INFRASTRUCTURE ONLY -- stand-in for the `gmpy2` module so the
read-only reference package (/root/reference/pkg/src/hcpdq) imports in this
container, where gmpy2 is not installed.

The reference uses exactly three symbols (bgv.py:27-28,63,69; heiface.py:21,61;
zpcore.py:19,68): `is_prime`, `gcd` and `mpz`.  `mpz` is only ever used as an
arbitrary-precision integer container, so the builtin `int` is semantically
identical.  `is_prime` is a deterministic Miller-Rabin (exact for n < 3.3e24,
which covers every 54-bit chain prime and every plaintext modulus), with a
probabilistic tail for larger inputs.

Nothing in the product package imports this file.
"""

from math import gcd as _gcd

mpz = int

_BASES = (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41)


def gcd(a, b):
    return _gcd(int(a), int(b))


def is_prime(n, reps: int = 25) -> bool:
    n = int(n)
    if n < 2:
        return False
    for b in _BASES:
        if n % b == 0:
            return n == b
    d, r = n - 1, 0
    while d % 2 == 0:
        d //= 2
        r += 1
    bases = _BASES
    if n >= 3317044064679887385961981:
        bases = _BASES + tuple(range(43, 43 + 2 * reps, 2))
    for a in bases:
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
