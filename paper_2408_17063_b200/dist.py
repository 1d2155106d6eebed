"""Block-sharded Comp over torch.distributed.

The BSGS matvec is a sum over width-4096 blocks (compress.py:286-297): every
block's pack, baby rotations and diagonal products are independent until
they are added into the giant-step accumulators acc[g] at level 1.  Each
rank runs those for a contiguous block range (libhcomp hc_comp_partial) and
leaves partial accumulators whose words are all < 2^54 (< 2^56 when its
last chunk ran as concurrent baby-step lanes, which add with atomics); one
uint64 SUM reduce to the root (NCCL over NVLink on GPUs; < 2^59 for <= 8
ranks, no overflow) combines them, and the root alone runs the giant-step and fold
key switches and the output mask (hc_comp_finish), which do not shard:
key switching is not additive bit-for-bit.

This is the only collective on the path.  Batched independent queries
(config 5) need none: one query per rank.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .compress import CompressedAnswer, _check_inputs, comp_noise, live_diagonals
from .backend import Ciphertext, RnsPayload


def shard_blocks(B: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced block range [b0, b1) of `rank` (first B % world
    ranks take one extra block).  Ranges tile [0, B) exactly."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    base, extra = divmod(B, world)
    b0 = rank * base + min(rank, extra)
    return b0, b0 + base + (1 if rank < extra else 0)


def reduce_partials(t, dist, group=None, root: int = 0):
    """Sum the ranks' partial accumulators on `root` (int64 view of uint64 words,
    each < 2^56: the sum over <= 255 ranks stays exact).  NCCL reduces device
    tensors in place; a CPU backend (gloo) goes through a host copy."""
    if t.is_cuda and dist.get_backend(group) != "nccl":
        h = t.cpu()
        dist.reduce(h, dst=root, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
        return t
    dist.reduce(t, dst=root, op=dist.ReduceOp.SUM, group=group)
    return t


def comp_sharded(cd, params, backend, keys, index_hint, dist, group=None, root: int = 0):
    """compress.comp (hint path, packed) with the blocks sharded over the ranks
    of `group`.  Every rank holds the full standard-layout inputs; the
    CompressedAnswer is returned on `root` (None elsewhere).

    A rank whose block range is empty (world > num_blocks) uploads nothing and
    contributes a zero partial, so every rank still joins the reduce.  All
    device work runs on torch's current stream of the backend's device, the
    stream the reduce is ordered on."""
    import torch

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cv = list(index_hint)
    cd = list(cd)
    if _check_inputs(cd, cv, params, backend, keys):
        raise NotImplementedError("sharded Comp takes level-3 inputs (mixed-level answer() inputs run unsharded)")
    live = live_diagonals(params)
    bits, sim = comp_noise(backend, params, [c.payload.noise_bits for c in cv], [c.payload.noise_bits for c in cd], live)
    b0, b1 = shard_blocks(params.num_blocks, world, rank)
    # this rank's plan: only its blocks' diagonals and input ciphertexts
    backend.plan(params.N, params.s, keys, block_range=(b0, b1))
    L = _lib.lib(backend.params.max_level)
    h = backend._ctx()
    dev = torch.device("cuda", backend.device)
    stream = torch.cuda.current_stream(dev)
    sh = ctypes.c_void_p(stream.cuda_stream)
    c0, c1 = b0 // 2, (b1 + 1) // 2  # the input ciphertexts this rank's blocks read
    if c1 > c0:
        cd_arr = np.ascontiguousarray(np.stack([c.payload.res for c in cd[c0:c1]]), dtype=np.uint64)
        cv_arr = np.ascontiguousarray(np.stack([c.payload.res for c in cv[c0:c1]]), dtype=np.uint64)
        _lib.check(L.hc_comp_set_inputs_range(h, _lib.ptr(cd_arr), _lib.ptr(cv_arr), c0, c1, sh))
        stream.synchronize()  # pageable host buffers: the copies have landed
    words = L.hc_partial_words(h)
    part = torch.zeros(words, dtype=torch.int64, device=dev)
    _lib.check(L.hc_comp_partial(h, b0, b1, ctypes.c_void_p(part.data_ptr()), sh))
    with torch.cuda.device(dev):
        reduce_partials(part, dist, group, root)
    if rank != root:
        stream.synchronize()
        return None
    _lib.check(L.hc_comp_finish(h, ctypes.c_void_p(part.data_ptr()), sh))
    out = np.empty((2, 1, backend.params.n), dtype=np.uint64)
    stream.synchronize()
    _lib.check(L.hc_comp_get_output(h, _lib.ptr(out)))
    backend.counters.keyswitches += sim.ks
    backend.counters.pt_mults += sim.pt
    backend.counters.adds += sim.adds
    ct = Ciphertext(backend.backend_id, keys.key_id, 0, RnsPayload(out, bits, (backend.q[0],)))
    return CompressedAnswer((ct,), params.s, True)
