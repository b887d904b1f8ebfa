"""The reference's feasibility sweep over the batched device path.

Pins: tests/test_feasibility.cpp:103-154 (cells == serial oracle, golden
aggregated CSV) and SURVEY.md §6 (run_benchmark(benchmark_defaults) finds
408,364 pairs).
"""
import numpy as np
import pytest

from cvtest_util import golden
from paper_2507_22901_b200 import sweep
from paper_2507_22901_b200 import workloads as W

pytestmark = pytest.mark.gpu


def test_golden_aggregated_matrix(ctx):
    cfg = sweep.SearchConfig.defaults()
    cells = sweep.feasibility_matrix(cfg, ctx)
    assert len(cells) == 756
    assert sweep.export_aggregated_csv(cfg, cells) == golden("matrix_aggregated.csv")


def test_cells_match_oracle_select_best(ctx, oracle):
    cfg = sweep.SearchConfig.defaults()
    cfg.names, cfg.colors = [cfg.names[1], cfg.names[5]], cfg.colors[[1, 5]]  # Gray, Blue (tiny_config)
    cells = sweep.feasibility_matrix(cfg, ctx)
    for c in cells:
        vt, rn = cfg.v_th_values[c.v_th_index], cfg.r_novib_values[c.r_novib_index]
        idx, codes, d = oracle.search(cfg.colors[c.color_index], W.bits(cfg.patterns[c.pattern_index]), vt, rn,
                                      cfg.radii, cfg.angles, method=0)
        assert c.pair_count == len(idx)
        assert c.feasible == (len(idx) > 0)
        if len(idx):
            j = sweep.select_best_index(d, vt, rn)
            na = len(cfg.angles)
            assert c.best_pair["radius"] == cfg.radii[idx[j] // na]
            assert c.best_pair["angle"] == cfg.angles[idx[j] % na]
            assert c.best_pair["plus"].tolist() == codes[j, :3].tolist()
            assert c.best_pair["minus"].tolist() == codes[j, 3:].tolist()
            assert c.best_pair["deltas"].tolist() == d[j].tolist()


def test_benchmark_defaults_pair_total(ctx):
    cfg = sweep.SearchConfig.benchmark_defaults()
    cells = sweep.feasibility_matrix(cfg, ctx)
    assert sum(c.pair_count for c in cells) == 408364  # SURVEY.md §6, run_benchmark parity pass


def test_pairs_array_matches_colorpair_objects(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    radii, angles = np.array(grid.radii), np.array(grid.angles)
    res = ctx.search(np.array([[240, 100, 240]], np.int32), np.array([5], np.int32), np.array([50.0]),
                     np.array([0.5]), radii, angles)
    recs = sweep.pairs_array(res, 0, [240, 100, 240], radii, angles)
    objs = cv.batch_search(cv.SrgbColor(240, 100, 240), grid, cv.BitPattern("101"), cv.Thresholds(50.0, 0.5))
    assert len(recs) == len(objs)
    for r, o in zip(recs, objs):
        assert r["radius"] == o.radius and r["angle"] == o.angle
        assert r["plus"].tolist() == [o.plus.r, o.plus.g, o.plus.b]
        assert r["minus"].tolist() == [o.minus.r, o.minus.g, o.minus.b]
        assert r["deltas"].tolist() == [o.deltas.dr, o.deltas.dg, o.deltas.db]
