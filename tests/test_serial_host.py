"""colorvibe::serial_search, the reference's scalar "previous method"
(search.cpp:184-218), runs on the host in the product library: one candidate
after another, as run_benchmark's serial column times it.  It
needs no device, so its parity with the reference is checked here on CPU:
the reference-generated small-case goldens (test_search.cpp:177-204 cases,
Quantized x both bases) and the oracle's serial method in all four
SearchOptions combinations, deltas included."""
import numpy as np
import pytest

from cvtest_util import golden, sha_records
from paper_2507_22901_b200 import workloads as W

GRID = (1.0, 91.0, 10.0, 0.0, 350.0, 10.0)


def _opts(cv, mode, basis):
    o = cv.SearchOptions()
    o.delta_mode = cv.DeltaMode.QUANTIZED if mode == 0 else cv.DeltaMode.CONTINUOUS
    o.delta_basis = cv.DeltaBasis.TARGET_SWING if basis == 0 else cv.DeltaBasis.FRAME_DIFF
    return o


def _records(pairs, grid):
    na = len(grid.angles)
    ri = {r: k for k, r in enumerate(grid.radii)}
    ai = {a: m for m, a in enumerate(grid.angles)}
    idx = np.array([ri[p.radius] * na + ai[p.angle] for p in pairs], np.uint32)
    codes = np.array([[p.plus.r, p.plus.g, p.plus.b, p.minus.r, p.minus.g, p.minus.b] for p in pairs],
                     np.uint8).reshape(-1, 6)
    return idx, codes


@pytest.mark.parametrize("basis", [0, 1])
def test_serial_search_matches_reference_goldens(cv, basis):
    grid = cv.VibrationGrid.uniform(*GRID)
    for c in golden("small_cases.json"):
        if c["basis"] != basis:
            continue
        pairs = cv.serial_search_opts(cv.SrgbColor(*c["target"]), grid, cv.BitPattern(c["pattern"]),
                                      cv.Thresholds(c["v_th"], c["r_novib"]), _opts(cv, 0, basis))
        idx, codes = _records(pairs, grid)
        assert len(idx) == c["count"], c
        assert sha_records(idx, codes) == c["sha256"], c


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("basis", [0, 1])
def test_serial_search_matches_oracle_with_deltas(cv, oracle, mode, basis):
    grid = cv.VibrationGrid.uniform(*GRID)
    for t in ([170, 170, 170], [240, 240, 240], [100, 100, 240], [8, 8, 8]):
        for p in ("100", "011", "111"):
            pairs = cv.serial_search_opts(cv.SrgbColor(*t), grid, cv.BitPattern(p), cv.Thresholds(50.0, 0.5),
                                          _opts(cv, mode, basis))
            oi, oc, od = oracle.search(t, W.bits(p), 50.0, 0.5, grid.radii, grid.angles, delta_mode=mode,
                                       delta_basis=basis, method=0)
            idx, codes = _records(pairs, grid)
            assert idx.tolist() == oi.tolist()
            assert codes.tolist() == oc.tolist()
            assert [[q.deltas.dr, q.deltas.dg, q.deltas.db] for q in pairs] == od.tolist()
            assert all(q.target == cv.SrgbColor(*t) for q in pairs)


def test_serial_search_validates_like_the_reference(cv):
    grid = cv.VibrationGrid.uniform(*GRID)
    with pytest.raises(ValueError):
        cv.serial_search(cv.SrgbColor(256, 0, 0), grid, cv.BitPattern("100"), cv.Thresholds(50.0, 0.5))
    with pytest.raises(ValueError):
        cv.serial_search(cv.SrgbColor(1, 2, 3), grid, cv.BitPattern("000"), cv.Thresholds(50.0, 0.5))
    empty = cv.VibrationGrid()
    assert cv.serial_search(cv.SrgbColor(1, 2, 3), empty, cv.BitPattern("100"), cv.Thresholds(50.0, 0.5)) == []
