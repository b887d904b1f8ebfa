"""Multi-GPU partitioning of a search batch (one process per GPU).

SURVEY.md §8(e): the searches are independent, so a batch is split into
contiguous search ranges, one per rank, with no data-path collective.  The
only exchange is the final gather of per-search counts (fixed size, one
`all_gather`) and, when a caller needs one contiguous list, the variable-size
pair records (size exchange + padded `all_gather`).  Canonical order is kept
because rank r holds searches [lo_r, hi_r) and ranks concatenate in order --
the multi-GPU analogue of the reference's ordered slice concatenation
(src/search.cpp:433-455).

The collectives go through torch.distributed: NCCL over NVLink on the B200
box, gloo in the CPU tests (tests/test_distributed.py).
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable

import numpy as np


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [lo, hi) share of n items for `rank` (balanced to +-1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return n * rank // world, n * (rank + 1) // world


@dataclass
class ShardResult:
    lo: int                 # first global search index of this rank
    hi: int
    counts: np.ndarray      # (n_searches,) global per-search pair counts (all ranks)
    offsets: np.ndarray     # (n_searches + 1,) global exclusive prefix
    idx: np.ndarray         # this rank's pair indices (k * n_angles + m)
    codes: np.ndarray       # this rank's pair codes (n, 6)

    @property
    def global_pair_offset(self) -> int:
        """Position of this rank's first pair in the global canonical list."""
        return int(self.offsets[self.lo])


def _device(group):
    import torch.distributed as dist

    return "cuda" if dist.get_backend(group) == "nccl" else "cpu"


def search_sharded(workload, local_search: Callable, group=None) -> ShardResult:
    """Runs this rank's share of `workload` with `local_search(shard)` (a
    callable returning a dict with "counts", "idx", "codes", e.g. a bound
    Context.search) and gathers the per-search counts of all ranks."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = workload.n_searches
    lo, hi = shard_range(n, rank, world)
    res = local_search(workload.shard(rank, world))
    local_counts = np.asarray(res["counts"], dtype=np.int64)
    dev = _device(group)
    width = max(shard_range(n, r, world)[1] - shard_range(n, r, world)[0] for r in range(world))
    buf = torch.zeros(width, dtype=torch.int64, device=dev)
    buf[: hi - lo] = torch.from_numpy(local_counts)
    gathered = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(gathered, buf, group=group)
    counts = np.concatenate([
        gathered[r][: shard_range(n, r, world)[1] - shard_range(n, r, world)[0]].cpu().numpy()
        for r in range(world)])
    offsets = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    return ShardResult(lo, hi, counts, offsets, np.asarray(res["idx"]), np.asarray(res["codes"]))


def gather_pairs(shard: ShardResult, group=None, dst: int = 0):
    """Variable-size gather of every rank's records onto `dst` in canonical
    order (size exchange, then a padded all_gather).  Returns (idx, codes) on
    dst, None elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device(group)
    n_local = len(shard.idx)
    sizes = [int(shard.offsets[shard_range(len(shard.counts), r, world)[1]] -
                 shard.offsets[shard_range(len(shard.counts), r, world)[0]]) for r in range(world)]
    assert sizes[rank] == n_local, (sizes, n_local)
    width = max(sizes) if sizes else 0
    rec = torch.zeros((max(width, 1), 10), dtype=torch.uint8, device=dev)
    if n_local:
        packed = np.zeros((n_local, 10), np.uint8)
        packed[:, :4] = np.ascontiguousarray(shard.idx, np.uint32).view(np.uint8).reshape(-1, 4)
        packed[:, 4:] = shard.codes
        rec[:n_local] = torch.from_numpy(packed)
    out = [torch.empty_like(rec) for _ in range(world)]
    dist.all_gather(out, rec, group=group)
    if rank != dst:
        return None
    parts = [out[r][: sizes[r]].cpu().numpy() for r in range(world)]
    allrec = np.concatenate(parts) if parts else np.zeros((0, 10), np.uint8)
    idx = np.ascontiguousarray(allrec[:, :4]).view(np.uint32).reshape(-1)
    codes = np.ascontiguousarray(allrec[:, 4:])
    return idx, codes
