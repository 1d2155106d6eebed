"""The drop-in boundary takes the reference's own objects (INTEGRATION.md
section 1): hcpdq HeParams / CompressionParams and the VandermondeTable of
hcpdq's precompute_masked_matrix convert to this package's equivalents by
their public attributes.  CPU test against the real reference package
(imported in the build container, skipped where it is absent)."""

import random

import numpy as np
import pytest

import paper_2408_17063_b200 as P
from paper_2408_17063_b200 import refcompat


@pytest.fixture(scope="module")
def hcpdq():
    from oracle import refimport

    if not refimport.available():
        pytest.skip("reference package not present")
    return refimport.load()


def test_params_from_reference_objects(hcpdq):
    from hcpdq.compress import CompressionParams as RefCP
    from hcpdq.heiface import HeParams as RefHe

    rhe = RefHe(8192, 65537, 3)
    rcp = RefCP(10000, 5, rhe)
    he = refcompat.he_params(rhe)
    cp = refcompat.compression_params(rcp)
    assert (he.n, he.p, he.max_level) == (8192, 65537, 3)
    assert he == P.HeParams(8192, 65537, 3)
    assert (cp.N, cp.s, cp.num_blocks, cp.num_ciphertexts, cp.s_pad) == (
        rcp.N, rcp.s, rcp.num_blocks, rcp.num_ciphertexts, rcp.s_pad)
    # the backend constructor and make_backend accept the reference HeParams
    be = P.make_backend("bgv-b200", rhe, seed=0)
    assert be.params == he


@pytest.mark.parametrize("n,p,N,s", [(64, 257, 200, 5), (8192, 65537, 10000, 5)])
def test_masked_table_from_reference(hcpdq, n, p, N, s):
    from hcpdq.compress import CompressionParams as RefCP
    from hcpdq.compress import precompute_masked_matrix as ref_pmm
    from hcpdq.heiface import HeParams as RefHe

    rng = random.Random(7)
    db = [rng.randrange(0, 10 * p) for _ in range(N)]
    rcp = RefCP(N, s, RefHe(n, p, 3))
    table = ref_pmm(db, rcp)
    got = refcompat.db_mod_p_from_table(table, refcompat.compression_params(rcp))
    assert np.array_equal(got, np.array([v % p for v in db], dtype=np.uint64))
    mm = P.MaskedMatrix.from_db_mod_p(refcompat.compression_params(rcp), got)
    assert np.array_equal(mm.db_mod_p, P.precompute_masked_matrix(db, refcompat.compression_params(rcp)).db_mod_p)
