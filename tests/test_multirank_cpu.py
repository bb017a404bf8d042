"""The N>1 path's host logic on CPU with gloo, world_size 2: each rank bins its
contiguous index shard (oracle histogram standing in for the per-rank kernel,
which needs a GPU) and the product's own ``allreduce_bins`` sums the counters.
The result must equal the unsharded histogram bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

N = 20_000


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import synth
        import paper_2312_02756_b200 as gvx
        a, b = synth.shard_range(N, rank, world)
        v1, v2 = synth.muon_pairs(np.arange(a, b), dtype=np.float32)
        h, _ = oracle.mass_histogram(v1, v2, 0.25, 300.0, 1000)
        bins = torch.from_numpy(h.astype(np.int64))
        gvx.allreduce_bins(bins)
        q.put((rank, bins.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_histogram_gloo(world, oracle_lib):
    import synth
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    v1, v2 = synth.muon_pairs(np.arange(N), dtype=np.float32)
    full, _ = oracle_lib.mass_histogram(v1, v2, 0.25, 300.0, 1000)
    for r in range(world):
        assert np.array_equal(res[r], full.astype(np.int64))


def test_shard_ranges_partition():
    import synth
    for n in (0, 1, 7, 1000, 10 ** 9 + 3):
        for g in (1, 2, 3, 4, 8):
            rs = [synth.shard_range(n, r, g) for r in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(g - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
