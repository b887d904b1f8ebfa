"""Multi-rank partitioning: world_size 2 over gloo (CPU oracle, and the real
device search on one GPU under -m gpu).

Each rank evaluates its contiguous share of a batch (here with the CPU oracle
standing in for the per-GPU search -- the partition/gather logic is what is
under test), the per-search counts are all_gathered and the pair lists
gathered in canonical order.  The result must equal one process evaluating
the whole batch.
"""
import os
import socket

import numpy as np
import pytest

from paper_2507_22901_b200 import workloads as W
from paper_2507_22901_b200.distributed import shard_range


def test_shard_range_partitions_exactly():
    for n in (0, 1, 7, 756, 4096):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _small_batch(n_targets=3):
    radii, angles = W.uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    t, p, v, r = [], [], [], []
    for tg in ([170, 170, 170], [240, 100, 240], [100, 100, 240])[:n_targets]:
        for pat in (5, 7, 4):
            for vt, rn in ((50.0, 0.5), (100.0, 0.25)):
                t.append(tg); p.append(pat); v.append(vt); r.append(rn)
    return W.Workload("small", np.array(t, np.int32), np.array(p, np.int32), np.array(v), np.array(r),
                      radii, angles)


def _oracle_search(shard):
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    if root not in sys.path:
        sys.path.insert(0, root)
    from oracle.oracle import Oracle

    o = Oracle()
    counts, idx, codes = [], [], []
    for s in range(shard.n_searches):
        i, c, _ = o.search(shard.targets[s], int(shard.patterns[s]), shard.v_th[s], shard.r_novib[s], shard.radii,
                           shard.angles, method=1, want_deltas=False)
        counts.append(len(i)); idx.append(i); codes.append(c)
    return {"counts": np.array(counts), "idx": np.concatenate(idx) if idx else np.zeros(0, np.uint32),
            "codes": np.concatenate(codes) if codes else np.zeros((0, 6), np.uint8)}


def _worker(rank, world, port, q, by="auto", n_targets=3):
    import torch.distributed as dist

    from paper_2507_22901_b200.distributed import gather_pairs, search_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = _small_batch(n_targets)
        res = search_sharded(wl, _oracle_search, by=by)
        got = gather_pairs(res)
        q.put((rank, res.counts.tolist(), res.global_pair_offset if res.by == "searches" else None,
               None if got is None else (got[0].tolist(), got[1].tolist())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,by,n_targets", [(2, "auto", 3), (2, "rows", 3), (2, "auto", 1)])
def test_gloo_shards_equal_single_process(world, by, n_targets):
    """Search ranges (18 searches) and radius-row slices (forced, and auto
    for a 6-search batch: < 4 searches per rank) give the single-process
    result in canonical order."""
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, by, n_targets)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    outs.sort()
    full = _oracle_search(_small_batch(n_targets))
    for rank, counts, off, _ in outs:
        assert counts == full["counts"].tolist()
        if off is not None:
            lo, _ = shard_range(len(counts), rank, world)
            assert off == int(np.sum(full["counts"][:lo]))
    idx, codes = outs[0][3]
    assert idx == full["idx"].tolist()
    assert codes == full["codes"].tolist()


def test_partition_rule():
    from paper_2507_22901_b200.distributed import partition

    assert partition(756, 256, 8) == "searches"   # cfg1
    assert partition(9, 4096, 8) == "rows"        # cfg2
    assert partition(1, 256, 8) == "rows"         # cfg0
    assert partition(1, 256, 1) == "searches"
    assert partition(4, 3, 8) == "searches"       # fewer rows than ranks


# ---- the sharded search on the GPU ------------------------------------------

def _gpu_search(shard):
    import paper_2507_22901_b200 as cv

    ctx = _gpu_search.ctx = getattr(_gpu_search, "ctx", None) or cv.Context(0)
    return ctx.search(shard.targets, shard.patterns, shard.v_th, shard.r_novib, shard.radii, shard.angles)


def _gpu_worker(rank, world, port, q, name):
    import hashlib

    import torch.distributed as dist

    from paper_2507_22901_b200.distributed import gather_pairs, search_sharded

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        wl = W.ALL[name]()
        try:
            res = search_sharded(wl, _gpu_search)
        except Exception as e:  # noqa: BLE001 -- reported to the parent instead of hanging it
            q.put((rank, "error", repr(e), None))
            raise
        got = gather_pairs(res)
        sha = None
        if got is not None:
            m = hashlib.sha256()
            for s in range(wl.n_searches):
                a, b = int(res.offsets[s]), int(res.offsets[s + 1])
                m.update(np.ascontiguousarray(got[0][a:b], np.uint32).tobytes())
                m.update(np.ascontiguousarray(got[1][a:b], np.uint8).tobytes())
            sha = m.hexdigest()
        q.put((rank, res.by, res.counts.tolist(), sha))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["cfg0", "cfg1"])
def test_sharded_gpu_search_matches_golden(name):
    """search_sharded with the REAL device search (Context.search) in two
    processes sharing cuda:0 (gloo collectives on the host: the two ranks'
    kernels never wait on each other), gathered on rank 0: cfg1 partitions
    by search ranges, cfg0 (one search) by radius rows; counts and the
    gathered records equal the reference goldens."""
    import multiprocessing as mp

    import torch
    from cvtest_util import golden

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, q, name)) for r in range(2)]
    for p in procs:
        p.start()
    outs = sorted(q.get(timeout=300) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(o[1] != "error" for o in outs), outs
    g = golden("workloads.json")[name]
    assert outs[0][1] == ("rows" if name == "cfg0" else "searches")
    for _, _, counts, _ in outs:
        assert counts == g["counts"]
    assert outs[0][3] == g["sha256"]
