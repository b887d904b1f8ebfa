"""Randomized parity: seeded random batches (targets, patterns, thresholds,
irregular explicit grids, white points, both delta bases) on the GPU vs the
CPU oracle, bit for bit, on all three evaluation paths.  Hypothesis drives
the case generation with a fixed database-free seed so runs are repeatable.
"""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, seed, settings
from hypothesis import strategies as st

from paper_2507_22901_b200 import workloads as W

pytestmark = pytest.mark.gpu


def random_grid(rng, nr, na, rmax):
    radii = np.unique(np.round(rng.uniform(0.0, rmax, nr), 6))
    angles = np.unique(rng.uniform(0.0, 2 * np.pi, na))
    angles = angles[angles < 2 * np.pi]
    return radii.astype(np.float64), angles.astype(np.float64)


def check_batch(ctx, oracle, rng, nr, na, rmax, n, basis, path, white=None):
    radii, angles = random_grid(rng, nr, na, rmax)
    targets = rng.integers(0, 256, (n, 3)).astype(np.int32)
    patterns = rng.integers(1, 8, n).astype(np.int32)
    v_th = rng.choice([0.5, 1.0, 7.0, 20.0, 50.0, 100.0, 150.0, 254.9, 255.0, 300.0], n)
    r_novib = rng.choice([1.0, 0.5, 0.25, 0.125, 0.01], n)
    res = ctx.search(targets, patterns, v_th, r_novib, radii, angles, path=path, delta_basis=basis,
                     white_point=white)
    assert res["stats"]["class_mismatch"] == 0
    if path == "audit":
        assert res["stats"]["audit_violations"] == 0
        assert res["stats"]["audit_max_ratio"] < 1.0
    for s in range(n):
        a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
        oi, oc, _ = oracle.search(targets[s], int(patterns[s]), v_th[s], r_novib[s], radii, angles,
                                  delta_basis=basis, white=white, method=1, want_deltas=False)
        assert np.array_equal(res["idx"][a:b], oi), (s, targets[s], patterns[s], v_th[s], r_novib[s])
        assert np.array_equal(res["codes"][a:b], oc), s


@seed(20260120)
@settings(max_examples=25, deadline=None, suppress_health_check=list(HealthCheck), database=None)
@given(st.integers(0, 2**31 - 1), st.sampled_from([0, 1]), st.sampled_from(["fast", "audit"]))
def test_random_batches(ctx, oracle, s, basis, path):
    rng = np.random.default_rng(s)
    nr = int(rng.integers(1, 40))
    na = int(rng.integers(1, 200))
    rmax = float(rng.choice([0.5, 5.0, 40.0, 130.0, 300.0]))
    check_batch(ctx, oracle, rng, nr, na, rmax, n=12, basis=basis, path=path)


@pytest.mark.parametrize("path", ["fast", "exact", "audit"])
def test_random_white_points(ctx, oracle, path):
    rng = np.random.default_rng(4242)
    for wp in ([0.9642, 1.0, 0.8251], [0.9505, 1.0, 1.089], [1.0985, 1.0, 0.3558]):
        check_batch(ctx, oracle, rng, 24, 96, 80.0, n=8, basis=0, path=path, white=wp)


def test_dark_targets_linear_branch(ctx, oracle):
    """Targets with L* near/below 8 put f on the linear branch of f^-1 for
    most candidates (convert_kernel.hpp:70-73)."""
    rng = np.random.default_rng(77)
    radii, angles = W.radii(48, 3.0), W.angles(160)
    targets = np.array([[0, 0, 0], [1, 1, 1], [3, 0, 7], [8, 8, 8], [12, 5, 0], [0, 20, 30]], np.int32)
    for pat in range(1, 8):
        n = len(targets)
        res = ctx.search(targets, np.full(n, pat, np.int32), np.full(n, 5.0), np.full(n, 0.5), radii, angles,
                         path="audit")
        assert res["stats"]["audit_violations"] == 0
        for s in range(n):
            a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
            oi, oc, _ = oracle.search(targets[s], pat, 5.0, 0.5, radii, angles, method=1, want_deltas=False)
            assert np.array_equal(res["idx"][a:b], oi) and np.array_equal(res["codes"][a:b], oc)
    del rng


@pytest.mark.parametrize("s", range(6))
@pytest.mark.parametrize("basis", [0, 1])
def test_random_aligned_grids_pruned(ctx, oracle, s, basis):
    """CVG_PATH_PRUNED on aligned grids (the band hot loop with row pruning;
    FrameDiff batches ignore the flag): every record equals the oracle's,
    dark and bright targets, radii from tiny to beyond the gamut."""
    rng = np.random.default_rng(1000 + s)
    nr = int(rng.integers(1, 48))
    na = int(rng.choice([32, 64, 96, 256, 512]))
    rmax = float(rng.choice([0.5, 5.0, 40.0, 130.0, 300.0]))
    check_batch(ctx, oracle, rng, nr, na, rmax, n=16, basis=basis, path="pruned")
