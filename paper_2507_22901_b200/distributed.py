"""Multi-GPU partitioning of a search batch (one process per GPU).

SURVEY.md §8(e): the searches are independent, so a batch is split into
contiguous search ranges, one per rank, with no data-path collective.  A batch
with fewer searches than ~4 per rank (cfg0: 1 target, cfg2: 9 targets) is
split by radius rows instead: rank r evaluates rows [k_lo, k_hi) of every
search, as the reference's threads do (src/search.cpp:433-455), and a
search's list is the rank-order concatenation of its row slices.  The
only exchange is the final gather of per-search counts (fixed size, one
`all_gather`) and, when a caller needs one contiguous list, the variable-size
pair records (size exchange, then exact-size send/recv into offset slices
on the destination rank only).  Canonical order is kept
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


def partition(n_searches: int, n_radii: int, world: int) -> str:
    """"searches" (contiguous search ranges) unless there are fewer than 4
    searches per rank and at least one radius row per rank: then "rows"."""
    if world > 1 and n_searches < 4 * world and n_radii >= world:
        return "rows"
    return "searches"


def shard_rows(workload, rank: int, world: int):
    """(sub-workload with radius rows [k_lo, k_hi) of every search, k_lo)."""
    k_lo, k_hi = shard_range(len(workload.radii), rank, world)
    sub = type(workload)(workload.name, workload.targets, workload.patterns, workload.v_th, workload.r_novib,
                         workload.radii[k_lo:k_hi], workload.angles, workload.output, workload.note)
    return sub, k_lo


@dataclass
class ShardResult:
    lo: int                 # first global search index of this rank (rows: 0)
    hi: int                 # (rows: n_searches)
    counts: np.ndarray      # (n_searches,) global per-search pair counts (all ranks)
    offsets: np.ndarray     # (n_searches + 1,) global exclusive prefix
    idx: np.ndarray         # this rank's pair indices (global k * n_angles + m)
    codes: np.ndarray       # this rank's pair codes (n, 6)
    by: str = "searches"    # partition: "searches" or "rows"
    rank_counts: np.ndarray | None = None  # (world, n_searches) per-rank counts

    @property
    def global_pair_offset(self) -> int:
        """Position of this rank's first pair in the global canonical list
        (search partition only: a row slice is not contiguous globally)."""
        if self.by != "searches":
            raise ValueError("row-partitioned pairs are interleaved per search; use gather_pairs")
        return int(self.offsets[self.lo])


def _device(group):
    import torch.distributed as dist

    return "cuda" if dist.get_backend(group) == "nccl" else "cpu"


def search_sharded(workload, local_search: Callable, group=None, by: str = "auto") -> ShardResult:
    """Runs this rank's share of `workload` with `local_search(shard)` (a
    callable returning a dict with "counts", "idx", "codes", e.g. a bound
    Context.search) and gathers the per-search counts of all ranks.
    `by`: "searches", "rows" or "auto" (`partition`)."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n = workload.n_searches
    if by == "auto":
        by = partition(n, len(workload.radii), world)
    dev = _device(group)
    if by == "rows":
        sub, k_lo = shard_rows(workload, rank, world)
        res = local_search(sub)
        local_counts = np.asarray(res["counts"], dtype=np.int64).reshape(n)
        buf = torch.from_numpy(local_counts).to(dev)
        gathered = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(gathered, buf, group=group)
        rank_counts = np.stack([g.cpu().numpy() for g in gathered])
        counts = rank_counts.sum(axis=0)
        offsets = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(counts, out=offsets[1:])
        idx = np.asarray(res["idx"], dtype=np.uint32) + np.uint32(k_lo * len(workload.angles))
        return ShardResult(0, n, counts, offsets, idx, np.asarray(res["codes"]), "rows", rank_counts)
    if by != "searches":
        raise ValueError("by must be 'searches', 'rows' or 'auto'")
    lo, hi = shard_range(n, rank, world)
    res = local_search(workload.shard(rank, world))
    local_counts = np.asarray(res["counts"], dtype=np.int64)
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


def _rank_sizes(shard: ShardResult, world: int) -> list:
    if shard.by == "rows":
        return [int(x) for x in shard.rank_counts.sum(axis=1)]
    n = len(shard.counts)
    return [int(shard.offsets[shard_range(n, r, world)[1]] - shard.offsets[shard_range(n, r, world)[0]])
            for r in range(world)]


def _row_destinations(shard: ShardResult, r: int) -> np.ndarray:
    """Global list positions of rank r's records (rows partition): search s's
    list is rank 0's slice, then rank 1's, ..."""
    C = shard.rank_counts
    before = np.cumsum(C, axis=0)[r] - C[r]              # pairs of s on ranks < r
    start = shard.offsets[:-1] + before                   # where rank r's block of s begins
    local = np.cumsum(C[r]) - C[r]                        # where it sits in rank r's list
    return np.repeat(start - local, C[r]) + np.arange(int(C[r].sum()))

def pack_records(idx, codes):
    """(n, 10) uint8 records: u32 LE idx, then the 6 code bytes (the wire
    layout of the pair gather)."""
    n = len(idx)
    rec = np.empty((n, 10), np.uint8)
    if n:
        rec[:, :4] = np.ascontiguousarray(idx, "<u4").view(np.uint8).reshape(-1, 4)
        rec[:, 4:] = codes
    return rec


def gather_records(rec, sizes: list, group=None, dst: int = 0):
    """Variable-size gather of every rank's (sizes[r], 10) uint8 record
    tensor into ONE (sum(sizes), 10) tensor on `dst`, rank r's records at
    offset sum(sizes[:r]) (grouped send/recv into
    offset slices).  Only dst allocates and receives; the other ranks only
    send their exact-size buffer.  `rec` lives on the backend's device (CUDA
    for NCCL, CPU for gloo).  Returns the tensor on dst, None elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    assert rec.shape[0] == sizes[rank], (rec.shape, sizes)
    to_global = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    if rank != dst:
        if sizes[rank]:
            dist.send(rec.contiguous(), to_global(dst), group=group)
        return None
    out = torch.empty((sum(sizes), 10), dtype=torch.uint8, device=rec.device)
    offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    ops = []
    for r in range(world):
        if r == dst or not sizes[r]:
            continue
        ops.append(dist.P2POp(dist.irecv, out[offs[r]:offs[r + 1]], to_global(r), group=group))
    reqs = dist.batch_isend_irecv(ops) if ops else []
    if sizes[dst]:
        out[offs[dst]:offs[dst + 1]].copy_(rec)
    for q in reqs:
        q.wait()
    return out


def gather_pairs(shard: ShardResult, group=None, dst: int = 0):
    """Gather of every rank's records onto `dst` in canonical order
    (gather_records: exact-size sends into offset slices, nothing received
    on the other ranks).  Returns (idx, codes) on dst, None elsewhere."""
    import torch
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _device(group)
    n_local = len(shard.idx)
    sizes = _rank_sizes(shard, world)
    assert sizes[rank] == n_local, (sizes, n_local)
    rec = torch.from_numpy(pack_records(shard.idx, shard.codes)).to(dev)
    out = gather_records(rec, sizes, group, dst)
    if rank != dst:
        return None
    allrec = out.cpu().numpy()
    if shard.by == "rows":
        # rank r's block of search s lands after ranks < r's blocks of s
        placed = np.empty_like(allrec)
        offs = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        for r in range(world):
            placed[_row_destinations(shard, r)] = allrec[offs[r]:offs[r + 1]]
        allrec = placed
    idx = np.ascontiguousarray(allrec[:, :4]).view(np.uint32).reshape(-1)
    codes = np.ascontiguousarray(allrec[:, 4:])
    return idx, codes
