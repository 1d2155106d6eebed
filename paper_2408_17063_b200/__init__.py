"""B200-native Comp for arXiv 2408.17063 (homomorphic compression for PDQ).

Drop-in surface of the reference package `hcpdq` for the Comp hot path:
`make_backend("bgv-b200", params, seed)` returns a BGV backend whose ring
operations and fused Comp run as hand-written sm_100a CUDA (libhcomp.so);
`comp(cd, params, backend, keys, index_hint=cv)` is the reference's
compress.comp on it.  See DESIGN.md and INTEGRATION.md.
"""

from .backend import (
    B200BgvBackend,
    Ciphertext,
    KeySet,
    OpCounters,
    RnsPayload,
    SlotMatrix,
)
from .compress import (
    CompressedAnswer,
    DeviceComp,
    MaskedMatrix,
    answer_from_match,
    comp,
    comp_masked,
    encode_vector,
    encrypt_vector,
    mask,
    precompute_masked_matrix,
)
from .params import (
    BackendMismatch,
    CompressionParams,
    HeParams,
    LevelExhausted,
    MissingRotationKey,
    NoiseOverflow,
    bsgs_shape,
    find_chain_primes,
    plan_rotation_amounts,
)

__version__ = "0.1.0"


def make_backend(backend_name: str, params: HeParams, seed: int | None = None, **kw):
    """Backend registry (net.py:103-110) with the B200 BGV backend registered."""
    if backend_name in ("bgv-b200", "b200", "bgv"):
        return B200BgvBackend(params, seed=seed, **kw)
    raise ValueError(f"unknown backend {backend_name!r}")


__all__ = [n for n in dir() if not n.startswith("_")]
