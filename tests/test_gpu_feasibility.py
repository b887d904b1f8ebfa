"""The feasibility sweep on the GPU (feasibility.hpp): every cell in one
batched launch, exports byte-identical to the reference's own
feasibility_matrix + export_matrix (oracle/_ref, run on CPU here), and the
reference's test_feasibility.cpp device cases."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

CONFIGS = [
    '{"version": 1}',
    '{"version": 1, "delta_basis": "frame_diff"}',
    '{"version": 1, "white_point": [0.9642, 1.0, 0.8251], "v_th": [20, 60.5], "r_novib": [0.3]}',
    '{"version": 1, "delta_mode": "continuous", "v_th": [50], "r_novib": [0.5]}',
    '{"version": 1, "delta_mode": "continuous", "delta_basis": "frame_diff", "v_th": [50, 100], "r_novib": [0.5]}',
    '{"version": 1, "grid": {"radius": {"min": 0, "max": 100, "step": 1}, '
    '"angle_deg": {"min": 0, "max": 359, "step": 1}}}',
]


@pytest.mark.parametrize("text", CONFIGS)
@pytest.mark.parametrize("fmt,aggregated", [("csv", True), ("json", True), ("csv", False), ("json", False)])
def test_exports_match_reference(cv, ctx, ref_codec, text, fmt, aggregated):
    m = cv.feasibility_matrix(cv.config_from_json(text))
    assert cv.export_matrix(m, fmt, aggregated) == ref_codec.export(text, fmt, aggregated)


def tiny(cv):  # test_feasibility.cpp:20-29
    cfg = cv.SearchConfig.defaults()
    cfg.colors = [cfg.colors[1], cfg.colors[5]]
    cfg.patterns = [cv.BitPattern("101"), cv.BitPattern("010")]
    cfg.v_th_values = [50.0]
    cfg.r_novib_values = [0.5]
    return cfg


def test_cells_match_serial_reference(cv, ctx):  # test_feasibility.cpp:103-123
    cfg = tiny(cv)
    m = cv.feasibility_matrix(cfg)
    assert len(m.cells) == cfg.combo_count()
    th = cv.Thresholds(50.0, 0.5)
    for ci in range(2):
        for pi in range(2):
            oracle = cv.serial_search(cfg.colors[ci].rgb, cfg.grid, cfg.patterns[pi], th)
            cell = m.cell(ci, pi, 0, 0)
            assert cell.feasible == bool(oracle) and cell.pair_count == len(oracle)
            assert (cell.best_pair is not None) == cell.feasible
            if cell.best_pair is not None:
                assert cell.best_pair == cv.select_best(oracle, th)


def test_aggregate_is_or_over_thresholds(cv, ctx):  # test_feasibility.cpp:125-141
    m = cv.feasibility_matrix(cv.SearchConfig.defaults())
    agg = cv.aggregate_any(m)
    assert len(agg.patterns) == 7 and len(agg.colors) == 9
    for pi in range(7):
        for ci in range(9):
            assert agg.at(pi, ci) == any(m.cell(ci, pi, vi, ri).feasible for vi in range(4) for ri in range(3))


def test_aggregated_export_golden_and_deterministic(cv, ctx):  # test_feasibility.cpp:143-154
    from cvtest_util import golden

    m = cv.feasibility_matrix(cv.SearchConfig.defaults())
    csv = cv.export_matrix(m, "csv", True)
    assert csv == golden("matrix_aggregated.csv")
    m2 = cv.feasibility_matrix(cv.SearchConfig.defaults())
    assert cv.export_matrix(m2, "csv", True) == csv
    assert cv.export_matrix(m2, "json", True) == cv.export_matrix(m, "json", True)


def test_full_export_rows(cv, ctx):  # test_feasibility.cpp:156-164
    cfg = tiny(cv)
    csv = cv.export_matrix(cv.feasibility_matrix(cfg), "csv", False)
    assert csv.count("\n") == cfg.combo_count() + 1
    assert csv.startswith("color,pattern,v_th,r_novib,feasible,pair_count")


def test_benchmark_defaults_total(cv, ctx):
    m = cv.feasibility_matrix(cv.SearchConfig.benchmark_defaults())
    assert sum(c.pair_count for c in m.cells) == 408364  # SURVEY §6, run_benchmark parity pass


def bench_config(cv):  # test_bench.cpp:11-20
    cfg = cv.SearchConfig.defaults()
    cfg.colors = [cfg.colors[1]]
    cfg.patterns = [cv.BitPattern("101"), cv.BitPattern("111")]
    cfg.v_th_values = [50.0]
    cfg.r_novib_values = [0.5]
    cfg.grid = cv.VibrationGrid.uniform(1.0, 61.0, 20.0, 0.0, 315.0, 45.0)
    return cfg


def test_benchmark_small_workload(cv, ctx):  # test_bench.cpp:23-49
    import json

    cfg = bench_config(cv)
    r = cv.run_benchmark(cfg, 2)
    assert r.result_parity and r.combos == cfg.combo_count() and r.candidates == cfg.grid.candidate_count()
    assert r.repetitions == 2 and r.workers >= 1
    assert r.serial_seconds > 0 and r.batch_seconds > 0 and r.batch_single_seconds > 0
    assert r.speedup == r.serial_seconds / r.batch_seconds
    assert r.config_hash == cv.config_hash(cfg)
    found = sum(len(cv.serial_search(cfg.colors[0].rgb, cfg.grid, p, cv.Thresholds(50.0, 0.5))) for p in cfg.patterns)
    assert r.pairs_found == found
    with pytest.raises(ValueError):
        cv.run_benchmark(cfg, 0)
    j = json.loads(cv.bench_report_json(r))
    assert j["version"] == 1 and j["combos"] == r.combos and j["candidates_per_combo"] == r.candidates
    assert j["result_parity"] is True and j["config_hash"] == r.config_hash


def test_benchmark_defaults_parity_pass(cv, ctx):  # run_benchmark(benchmark_defaults) = 408,364
    r = cv.run_benchmark(cv.SearchConfig.benchmark_defaults(), 1)
    assert r.result_parity and r.pairs_found == 408364


def _host_select_best(res, targets, v_th, r_novib, basis):
    """select_best (search.cpp:458-489) over each search's PAIRS records in
    double: the first maximum of classification_margin in canonical order."""
    best = []
    for s in range(len(res["counts"])):
        a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
        if a == b:
            best.append(None)
            continue
        c = res["codes"][a:b].astype(np.int64)
        t = np.asarray(targets[s], np.int64)
        if basis == 0:
            d = np.maximum(np.abs(c[:, :3] - t), np.abs(c[:, 3:] - t)).astype(np.float64)
        else:
            d = np.abs(c[:, :3] - c[:, 3:]).astype(np.float64)
        low = v_th[s] * r_novib[s]
        g = np.where(d > v_th[s], d - v_th[s], low - d)
        m = g.min(axis=1)
        j = int(np.argmax(m))  # first maximum
        best.append((int(res["idx"][a + j]), res["codes"][a + j].tolist()))
    return best


@pytest.mark.parametrize("basis", [0, 1])
def test_best_output_mode_matches_host_select_best(ctx, basis):
    """CVG_OUT_BEST (select_best on the device) on the 756-search cfg1 sweep
    against select_best's rule applied to the full pair lists."""
    from paper_2507_22901_b200 import workloads as W

    wl = W.cfg1()
    args = (wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles)
    full = ctx.search(*args, delta_basis=basis)
    best = ctx.search(*args, output="best", delta_basis=basis)
    assert np.array_equal(best["counts"], full["counts"])
    want = _host_select_best(full, wl.targets, wl.v_th, wl.r_novib, basis)
    for s, w in enumerate(want):
        if w is None:
            assert best["first_idx"][s] == 0xFFFFFFFF
        else:
            assert (int(best["first_idx"][s]), best["first_codes"][s].tolist()) == w, s


def test_best_output_rejects_continuous(ctx):
    from paper_2507_22901_b200 import workloads as W

    wl = W.cfg0()
    with pytest.raises(RuntimeError):
        ctx.search(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, output="best", delta_mode=1)
