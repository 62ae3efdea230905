"""Host-side logic of the multi-GPU batch path on CPU with gloo, world size 2.

The batch of C5 instances is partitioned contiguously over the ranks; each rank generates only
its block; the final gather reassembles the batch in instance order.  Checked here: the blocks
are disjoint and cover the batch, every rank's block equals the matching slice of the full
batch bitwise, and an all_gather of per-rank results reproduces the single-process order.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from synth.generator import make_config, partition


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, total, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench  # the bench's own partition/workload code
    a, b = partition(total, world, rank)
    inst = bench.workload("C5", rank, 0, world) if total == bench.C5_TOTAL else \
        make_config("C5", instance=a, batch=b - a)
    # stand-in for x: a deterministic per-instance digest of the generated values
    dig = torch.tensor(np.stack([inst.Sigma_x[k][:8] for k in range(b - a)]))
    out = [torch.zeros_like(dig) for _ in range(world)]
    dist.all_gather(out, dig)
    if rank == 0:
        q.put((a, b, torch.cat(out).numpy()))
    else:
        q.put((a, b, None))
    dist.destroy_process_group()


@pytest.mark.parametrize("total", [8, 512])
def test_partition_and_gather_gloo(total):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, total, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = sorted((a, b) for a, b, _ in res)
    assert ranges[0][0] == 0 and ranges[-1][1] == total and ranges[0][1] == ranges[1][0]
    gathered = next(g for _, _, g in res if g is not None)
    full = make_config("C5", batch=total)
    assert np.array_equal(gathered, np.stack([full.Sigma_x[k][:8] for k in range(total)]))


def test_partition_blocks_cover_exactly():
    for total in (1, 7, 512):
        for world in (1, 2, 3, 4, 8):
            blocks = [partition(total, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == total
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))


def test_rank_block_equals_full_batch_slice():
    full = make_config("C5", batch=16)
    for world in (2, 4):
        for r in range(world):
            a, b = partition(16, world, r)
            blk = make_config("C5", instance=a, batch=b - a)
            for k in range(b - a):
                one = blk.instance(k) if blk.batch > 1 else blk
                assert np.array_equal(one.W_vals, full.W_vals[a + k])
                assert np.array_equal(one.J_vals, full.J_vals[a + k])
                assert np.array_equal(one.b, full.b[a + k])
