"""Multi-GPU batch driver (BASELINE.json config 5).

A batch of independent BSE matrices (distinct seeds, standing in for momentum-transfer
points) is partitioned across ranks — one process per GPU — with NO collective on the data
path: every rank solves its own seeds on its own device. The only communication is the
result gather: eigenvalues to every rank (all_gather) and, optionally, eigenvectors to rank
0 (point-to-point send/recv). Over NCCL on NVLink/NVSwitch in production; the same code
runs over gloo on CPU tensors in tests/test_dist.py (with an injected stand-in solver).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Dict, List, Optional

import numpy as np


def shard_seeds(batch: int, rank: int, world: int) -> List[int]:
    """Static round-robin partition: rank r owns seeds r, r+N, ... (balanced when N | batch)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    return [s for s in range(batch) if s % world == rank]


def max_shard(batch: int, world: int) -> int:
    return (batch + world - 1) // world


@dataclass
class BatchResult:
    lam: Optional[np.ndarray]           # (batch, n) on every rank, seed order
    v: Optional[Dict[int, np.ndarray]]  # seed -> 2n x n eigenvectors (rank 0, if gathered)
    local_seeds: List[int]


def run_batch(solve: Callable[[int], tuple], batch: int, n: int, rank: int, world: int,
              device, gather_vectors: bool = False, dist=None) -> BatchResult:
    """solve(seed) -> (lam (n,) float64 tensor on `device`, V (2n x n) complex128 tensor on
    `device`, column-major bytes). Returns the gathered results."""
    import torch
    seeds = shard_seeds(batch, rank, world)
    per = max_shard(batch, world)
    lam_local = torch.zeros((per, n), dtype=torch.float64, device=device)
    vs = {}
    for i, s in enumerate(seeds):
        lam, v = solve(s)
        lam_local[i].copy_(lam)
        if gather_vectors:
            vs[s] = v
    if world == 1 or dist is None:
        lam_all = lam_local[: len(seeds)].cpu().numpy()
        return BatchResult(lam_all, {k: v.cpu().numpy() for k, v in vs.items()}
                           if gather_vectors else None, seeds)
    gathered = torch.zeros((world * per, n), dtype=torch.float64, device=device)
    dist.all_gather_into_tensor(gathered, lam_local)
    lam_all = np.zeros((batch, n))
    g = gathered.cpu().numpy()
    for r in range(world):
        for i, s in enumerate(shard_seeds(batch, r, world)):
            lam_all[s] = g[r * per + i]
    vout = None
    if gather_vectors:
        # rank 0 receives every remote eigenvector block (P2P; NVLink under NCCL)
        if rank == 0:
            vout = {s: v.cpu().numpy() for s, v in vs.items()}
            for r in range(1, world):
                for s in shard_seeds(batch, r, world):
                    buf = torch.empty((n, 2 * n), dtype=torch.complex128, device=device)
                    dist.recv(buf, src=r)
                    vout[s] = buf.cpu().numpy()
        else:
            for s in seeds:
                dist.send(vs[s].contiguous(), dst=0)
    return BatchResult(lam_all, vout, seeds)
