"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded Comp host
logic: the block partition and the uint64 partial-sum reduction.

The GPU computes each rank's partial accumulators (hc_comp_partial); here
the CPU oracle stands in for that compute so the partition and reduction
code of paper_2408_17063_b200.dist is exercised end to end: each rank's
partial acc[g] (sum over its blocks of mul_plain(rot(u_t, b), diag), the
reference's accumulation, compress.py:286-297) is reduced with the same
reduce_partials() call as on GPUs, and the root's modular fold must equal
the single-process accumulators."""

import os
import socket

import numpy as np
import pytest

from paper_2408_17063_b200.dist import shard_blocks


def test_shard_blocks_tiles_exactly():
    for B in (1, 2, 3, 4, 7, 16, 128, 1024):
        for world in (1, 2, 3, 4, 8):
            ranges = [shard_blocks(B, world, r) for r in range(world)]
            covered = [b for b0, b1 in ranges for b in range(b0, b1)]
            assert covered == list(range(B))
            sizes = [b1 - b0 for b0, b1 in ranges]
            assert max(sizes) - min(sizes) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _partial_accs(O, be, keys, u, plan, blocks):
    """Oracle partial accumulators (uint64 [giant][2][2][n], level 1) over `blocks`."""
    acc = np.zeros((plan.giant, 2, 2, be.n), dtype=np.uint64)
    for t in blocks:
        rotated = [u[t]] + [be.rot_row(u[t], b, keys) for b in range(1, plan.baby)]
        for g in range(plan.giant):
            for b in range(plan.baby):
                d = plan.diagonals[t][g * plan.baby + b]
                if d is None:
                    continue
                prod = be.mul_plain(rotated[b], d)
                acc[g] = be.pointwise(acc[g], prod.c, 1, "add")
    return acc


def _worker(rank, world, port, result_q, N=200):
    import torch
    import torch.distributed as dist

    from oracle import bgv_oracle as O
    from paper_2408_17063_b200.dist import reduce_partials, shard_blocks

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, p, s = 64, 257, 5  # N=200: 7 blocks of 32 slots, odd count; N=64: 2 blocks
        be = O.OracleBgv(n, p, 3, seed=21, check_noise=False)
        keys = be.keygen(*O.plan_rotation_amounts(s, n))
        dense = O.plant_sparse(__import__("random").Random(21), N, s, p)
        cd = O.encrypt_vector(dense, N, be, keys)
        cv = O.encrypt_vector([1 if x else 0 for x in dense], N, be, keys)
        u = O.pack_pair(cv, cd, N, be, keys)
        plan = O.build_plan(N, s, n, p)
        B = len(u)
        b0, b1 = shard_blocks(B, world, rank)
        part = _partial_accs(O, be, keys, u, plan, range(b0, b1))
        t = torch.from_numpy(part.view(np.int64).copy())
        reduce_partials(t, dist, root=0)
        if rank == 0:
            total = t.numpy().view(np.uint64)
            qv = np.array(be.q[:2], dtype=np.uint64).reshape(1, 1, 2, 1)
            folded = total % qv
            full = _partial_accs(O, be, keys, u, plan, range(B))
            result_q.put(bool(np.array_equal(folded, full)) and b1 - b0 >= 1)
        elif b1 == b0:  # world > blocks: an empty range contributes a zero partial
            result_q.put(bool(not part.any()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,world", [(200, 2), (64, 3)])
def test_sharded_partials_reduce_to_full_accumulators(N, world):
    """world 2 over 7 blocks, and world 3 over 2 blocks (one rank empty)."""
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, N)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=300)
        assert pr.exitcode == 0
    n_results = 1 + sum(1 for r in range(1, world) if shard_blocks(-(-N // 32), world, r)[0] == shard_blocks(-(-N // 32), world, r)[1])
    assert all(q.get(timeout=5) is True for _ in range(n_results))
