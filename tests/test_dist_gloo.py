"""N>1 plumbing on CPU: world_size-2 gloo ranks over 127.0.0.1 exercise the
same reductions bench.py runs over NCCL (max of step time, sum of work), the
bit-row gather, and the shard partitions."""
import os
import socket

import pytest

from paper_2501_02747_b200.dist import pair_row_blocks, shard


def test_shard_partitions_cover_exactly():
    for total in (0, 1, 7, 100, 788140):
        for world in (1, 2, 3, 8):
            ranges = [shard(total, r, world) for r in range(world)]
            assert ranges[0][0] == 0 and ranges[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))


def test_pair_row_blocks_balanced():
    n = 1256
    blocks = pair_row_blocks(n, 4)
    counts = [sum(n - 1 - i for i in range(a, b)) for a, b in blocks]
    assert sum(counts) == n * (n - 1) // 2
    assert max(counts) - min(counts) < n


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2501_02747_b200.dist import gather_bit_rows, reduce_step_metrics
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ms, units = reduce_step_metrics(10.0 + rank, 1000.0 * (rank + 1))
    rows = torch.full((2, 3), rank, dtype=torch.int64)
    got = gather_bit_rows(rows)
    # row-block merge: each rank's matrix carries its own (disjoint) bits, top bit included
    import numpy as np
    from paper_2501_02747_b200.dist import merge_bit_blocks
    mine = np.zeros((4, 2), np.uint64)
    mine[rank, 0] = np.uint64(1) << np.uint64(63 if rank == 0 else 5)
    mine[3, 1] = np.uint64(0xF0 if rank == 0 else 0x0F)
    merged = merge_bit_blocks(mine)
    expect = np.zeros((4, 2), np.uint64)
    expect[0, 0] = np.uint64(1) << np.uint64(63)
    expect[1, 0] = np.uint64(1) << np.uint64(5)
    expect[3, 1] = np.uint64(0xFF)
    assert (merged == expect).all()
    q.put((rank, ms, units, [int(t[0, 0]) for t in got]))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_reductions():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ms, units, gathered in res:
        assert ms == 11.0            # max over ranks
        assert units == 3000.0       # sum over ranks
        assert gathered == [0, 1]
