"""Accept the reference package's own parameter and table objects at the
drop-in boundary.

A maintainer dispatching hcpdq's `compress.comp` to this package (the
snippet in INTEGRATION.md) passes hcpdq objects straight through: an
`hcpdq.heiface.HeParams`, an `hcpdq.compress.CompressionParams` and, for
comp_masked, the `VandermondeTable` that `precompute_masked_matrix` returned
(compress.py:103-157).  These helpers turn them into this package's
equivalents by their public attributes only (duck typing: n / p / max_level,
N / s / he, and `VandermondeTable.block`), so neither side reads the
other's private fields.
"""

from __future__ import annotations

import numpy as np

from .params import CompressionParams, HeParams


def he_params(obj) -> HeParams:
    """HeParams (heiface.py:50-70) from any object with n, p, max_level."""
    if isinstance(obj, HeParams):
        return obj
    return HeParams(int(obj.n), int(obj.p), int(obj.max_level))


def compression_params(obj) -> CompressionParams:
    """CompressionParams (compress.py:39-73) from any object with N, s, he."""
    if isinstance(obj, CompressionParams):
        return obj
    return CompressionParams(int(obj.N), int(obj.s), he_params(obj.he))


def db_mod_p_from_table(table, params: CompressionParams) -> np.ndarray:
    """The cleartext database (mod p) behind a reference comp_masked table.

    `VandermondeTable.block(k)` row 0 holds col * DB[col-1] mod p for the
    block's columns col = k*m+1 .. (compress.py:118-139, first power of the
    column scaled by the database); p > N >= col makes col invertible mod p,
    so DB[col-1] mod p = row0 * col^-1."""
    p = params.he.p
    m = params.block_width
    out = np.zeros(params.N, dtype=np.uint64)
    for k in range(params.num_blocks):
        row0 = np.asarray(table.block(k)[0], dtype=object)
        c0 = k * m
        cnt = min(m, params.N - c0)
        for i in range(cnt):
            col = c0 + i + 1
            out[c0 + i] = int(row0[i]) * pow(col, -1, p) % p
    return out
