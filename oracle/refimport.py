"""TEST INFRASTRUCTURE ONLY -- import the read-only Python reference
(`hcpdq`, /root/reference/pkg/src) in THIS container, with the gmpy2
stand-in from `oracle/_shim`.

The reference does not exist on the GPU box; only golden-fixture generation
(`oracle/make_golden.py`) and the CPU tests that pin the oracle use this
module, and they skip cleanly when the reference is absent.
"""

from __future__ import annotations

import contextlib
import os
import sys

REF_SRC = "/root/reference/pkg/src"
_SHIM = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_shim")


def available() -> bool:
    return os.path.isdir(os.path.join(REF_SRC, "hcpdq"))


def load():
    """Return the reference `hcpdq` package (raises ImportError if absent)."""
    if not available():
        raise ImportError("reference package not present (only in the build container)")
    try:
        import gmpy2  # noqa: F401  (a real gmpy2 works too)
    except ImportError:
        if _SHIM not in sys.path:
            sys.path.insert(0, _SHIM)
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import hcpdq  # noqa: F401
    import hcpdq.bgv  # noqa: F401
    import hcpdq.compress  # noqa: F401

    return sys.modules["hcpdq"]


@contextlib.contextmanager
def noise_guard_disabled():
    """No-op the reference's heuristic noise guard:
    `BgvBackend._check_noise` (bgv.py:424-429) only raises; it never changes
    ciphertext values, so disabling it leaves every output bit unchanged."""
    hc = load()
    cls = hc.bgv.BgvBackend
    orig = cls._check_noise
    cls._check_noise = lambda self, bits, level: bits
    try:
        yield
    finally:
        cls._check_noise = orig
