"""World-size-2 gloo test of the batch partition + gather path (CPU; the solver is an
injected deterministic stand-in, since the product solver runs only on a GPU)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2008_08825_b200.batch import max_shard, run_batch, shard_seeds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _stub(n):
    def solve(seed):
        lam = torch.arange(n, dtype=torch.float64) + 1000.0 * seed
        v = torch.full((n, 2 * n), complex(seed, -seed), dtype=torch.complex128)
        return lam, v
    return solve


def _worker(rank, world, port, batch, n, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = run_batch(_stub(n), batch, n, rank, world, torch.device("cpu"),
                        gather_vectors=True, dist=dist)
        out = {"rank": rank, "lam": res.lam, "seeds": res.local_seeds,
               "vkeys": sorted(res.v.keys()) if res.v is not None else None}
        if rank == 0:
            out["vlast"] = res.v[batch - 1][0, 0]
        q.put(out)
    finally:
        dist.destroy_process_group()


def test_shard_partition():
    for world in (1, 2, 4, 8):
        allseeds = sorted(s for r in range(world) for s in shard_seeds(64, r, world))
        assert allseeds == list(range(64))
        assert all(len(shard_seeds(64, r, world)) == 64 // world for r in range(world))
    assert max_shard(10, 4) == 3
    with pytest.raises(ValueError):
        shard_seeds(8, 2, 2)


@pytest.mark.parametrize("batch", [8, 7])
def test_gloo_world2_gather(batch):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 5
    procs = [ctx.Process(target=_worker, args=(r, 2, port, batch, n, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o["rank"])
    expect = np.stack([np.arange(n) + 1000.0 * s for s in range(batch)])
    for o in outs:
        assert np.array_equal(o["lam"], expect)
    assert outs[0]["seeds"] == [s for s in range(batch) if s % 2 == 0]
    assert outs[0]["vkeys"] == list(range(batch))
    assert outs[0]["vlast"] == complex(batch - 1, -(batch - 1))
    assert outs[1]["vkeys"] is None
