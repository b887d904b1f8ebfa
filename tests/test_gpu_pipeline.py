"""The pipelined PAIRS read-back (cvg_search.cpp search_pipelined): batches of
>= 2^25 candidates are split into search ranges whose pairs are copied back
while later ranges compute.  The result must equal the single-plan result
bit for bit, including when the pinned result has to grow (early ranges
with few pairs, late ranges with many) and when ranges are empty.
"""
import numpy as np
import pytest

from paper_2507_22901_b200 import workloads as W

pytestmark = pytest.mark.gpu


def single_plan(ctx, targets, pats, vt, rn, radii, angles, step):
    """The same batch as sub-batches below the pipelining threshold."""
    idx, codes, counts = [], [], []
    for a in range(0, len(pats), step):
        r = ctx.search(targets[a:a + step], pats[a:a + step], vt[a:a + step], rn[a:a + step], radii, angles)
        assert r["n_pairs"] == 0 or len(r["idx"]) == r["n_pairs"]
        idx.append(r["idx"].copy())
        codes.append(r["codes"].copy())
        counts.append(r["counts"].copy())
    return np.concatenate(idx), np.concatenate(codes), np.concatenate(counts)


@pytest.mark.parametrize("na", [1024, 1000])
@pytest.mark.parametrize("order", ["sparse_first", "dense_first", "mixed"])
def test_pipelined_equals_single_plan(ctx, order, na):
    """na = 1000: tiles straddle radius rows."""
    rng = np.random.default_rng({"sparse_first": 1, "dense_first": 2, "mixed": 3}[order])
    radii, angles = W.radii(256, 1.0), W.angles(na)
    n = 320  # 83.9M candidates -> 2 ranges (sizes 1:2)
    targets = rng.integers(0, 256, (n, 3)).astype(np.int32)
    pats = rng.integers(1, 8, n).astype(np.int32)
    vt = rng.choice([5.0, 20.0, 50.0], n)
    rn = np.full(n, 0.5)
    if order == "sparse_first":
        vt[: n // 2] = 254.9  # almost nothing passes in the first range
    elif order == "dense_first":
        vt[n // 2:] = 254.9
    got = ctx.search(targets, pats, vt, rn, radii, angles)
    want_idx, want_codes, want_counts = single_plan(ctx, targets, pats, vt, rn, radii, angles, 64)
    assert np.array_equal(got["counts"], want_counts)
    assert got["n_pairs"] == len(want_idx)
    assert np.array_equal(got["offsets"][1:], np.cumsum(want_counts))
    assert np.array_equal(got["idx"], want_idx)
    assert np.array_equal(got["codes"], want_codes)
    assert got["stats"]["class_mismatch"] == 0
    # a repeat of the same shape takes the hinted capacity path
    again = ctx.search(targets, pats, vt, rn, radii, angles)
    assert np.array_equal(again["idx"], want_idx) and np.array_equal(again["codes"], want_codes)


def test_hinted_repeat_and_overflow_rerun(ctx):
    """A repeat of a pipelined shape sizes the device pair buffer from the
    previous total (+25%).  A repeat with many more pairs overflows it, and
    the batch reruns at the exact size (cvg_search.cpp search_pipelined).
    Every call must equal the single-plan result."""
    rng = np.random.default_rng(5)
    radii, angles = W.radii(256, 1.0), W.angles(1024)
    n = 320
    targets = rng.integers(0, 256, (n, 3)).astype(np.int32)
    pats = rng.integers(1, 8, n).astype(np.int32)
    rn = np.full(n, 0.5)
    sparse = np.full(n, 254.9)
    sparse[:8] = 20.0
    dense = rng.choice([5.0, 20.0, 50.0], n)
    for vt in (sparse, sparse, dense, dense, dense):
        got = ctx.search(targets, pats, vt, rn, radii, angles)
        want_idx, want_codes, want_counts = single_plan(ctx, targets, pats, vt, rn, radii, angles, 64)
        assert np.array_equal(got["counts"], want_counts)
        assert np.array_equal(got["idx"], want_idx) and np.array_equal(got["codes"], want_codes)
        assert got["stats"]["class_mismatch"] == 0


def test_pipelined_no_pairs(ctx):
    radii, angles = W.radii(256, 1.0), W.angles(1024)
    n = 300  # 78.6M candidates -> 2 ranges
    targets = np.zeros((n, 3), np.int32)
    res = ctx.search(targets, np.full(n, 7, np.int32), np.full(n, 300.0), np.full(n, 0.5), radii, angles)
    assert res["n_pairs"] == 0 and len(res["idx"]) == 0 and res["counts"].sum() == 0
    assert np.all(res["offsets"] == 0)


def test_pipelined_many_ranges_audit(ctx, oracle):
    """4 ranges; sampled searches checked against the oracle on the audit path."""
    rng = np.random.default_rng(9)
    radii, angles = W.radii(128, 0.5), W.angles(1024)
    n = 12000  # 1.57G candidates -> 4 ranges
    targets = rng.integers(0, 256, (n, 3)).astype(np.int32)
    pats = rng.integers(1, 8, n).astype(np.int32)
    vt = rng.choice([60.0, 100.0, 150.0], n)
    rn = rng.choice([0.5, 0.25], n)
    res = ctx.search(targets, pats, vt, rn, radii, angles, path="audit")
    assert res["stats"]["audit_violations"] == 0
    for s in rng.choice(n, 12, replace=False):
        a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
        oi, oc, _ = oracle.search(targets[s], int(pats[s]), vt[s], rn[s], radii, angles, method=1, want_deltas=False)
        assert np.array_equal(res["idx"][a:b], oi) and np.array_equal(res["codes"][a:b], oc), s


@pytest.mark.parametrize("output", ["first", "counts"])
def test_ranged_counts_first_equal_single_plans(ctx, output):
    """Per-pixel-size COUNTS / FIRST batches (>= 2^20 searches) run as 4
    search ranges whose prep and read-back overlap the kernels
    (cvg_search.cpp search_ranges_fixed); results equal sub-batch single plans."""
    rng = np.random.default_rng(31)
    n = (1 << 20) + 12345
    radii, angles = W.radii(8, 6.0), W.angles(64)
    targets = rng.integers(0, 256, (n, 3)).astype(np.int32)
    pats = rng.integers(1, 8, n).astype(np.int32)
    vt = rng.choice([20.0, 50.0], n)
    rn = np.full(n, 0.5)
    got = ctx.search(targets, pats, vt, rn, radii, angles, output=output)
    step = 1 << 18
    for a in range(0, n, step):
        want = ctx.search(targets[a:a + step], pats[a:a + step], vt[a:a + step], rn[a:a + step], radii, angles,
                          output=output)
        assert np.array_equal(got["counts"][a:a + step], want["counts"])
        if output == "first":
            assert np.array_equal(got["first_idx"][a:a + step], want["first_idx"])
            assert np.array_equal(got["first_codes"][a:a + step], want["first_codes"])
    assert got["n_pairs"] == int(got["counts"].sum())
