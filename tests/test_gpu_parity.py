"""GPU parity: the fused sm_100a search vs the CPU oracle / reference goldens.

Bar: bit-exact (integer/byte work).  Per-search counts and every emitted
(idx = k*na+m, plus rgb, minus rgb) record must equal the oracle's on the same
inputs; full-size configs are checked against reference-generated golden
counts/hashes and size-independent properties.
"""
import threading

import numpy as np
import pytest

from cvtest_util import golden, records10_sha, sha_records
from paper_2507_22901_b200 import workloads as W
from paper_2507_22901_b200.workloads import uniform_grid

pytestmark = pytest.mark.gpu


def run(ctx, wl, output="pairs", path="fast", basis=0, white=None, mode=0):
    return ctx.search(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles, output=output,
                      path=path, delta_basis=basis, white_point=white, delta_mode=mode)


def split(res, s):
    a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
    return res["idx"][a:b], res["codes"][a:b]


def oracle_records(oracle, wl, s, basis=0, white=None, workers=4, mode=0):
    idx, codes, _ = oracle.search(wl.targets[s], int(wl.patterns[s]), wl.v_th[s], wl.r_novib[s], wl.radii,
                                  wl.angles, delta_basis=basis, white=white, method=1, workers=workers,
                                  want_deltas=False, delta_mode=mode)
    return idx, codes


def sha_by_search(res):
    """Hash in the fixture's layout: per search, its idx bytes then its codes bytes."""
    import hashlib

    m = hashlib.sha256()
    for s in range(len(res["counts"])):
        idx, codes = split(res, s)
        m.update(np.ascontiguousarray(idx, np.uint32).tobytes())
        m.update(np.ascontiguousarray(codes, np.uint8).tobytes())
    return m.hexdigest()


def assert_clean(res, path):
    st = res["stats"]
    assert st["class_mismatch"] == 0
    if path == "audit":
        assert st["audit_violations"] == 0
        assert st["audit_max_ratio"] < 1.0, st


@pytest.mark.parametrize("path", ["fast", "exact", "audit", "pruned"])
def test_cfg0_bit_exact(ctx, oracle, path):
    wl = W.cfg0()
    res = run(ctx, wl, path=path)
    g = golden("workloads.json")["cfg0"]
    assert res["n_pairs"] == g["total"] == 4802
    idx, codes = split(res, 0)
    oi, oc = oracle_records(oracle, wl, 0)
    assert np.array_equal(idx, oi)
    assert np.array_equal(codes, oc)
    assert sha_records(idx, codes) == g["sha256"]
    assert_clean(res, path)


@pytest.mark.parametrize("basis", [0, 1])
@pytest.mark.parametrize("path", ["fast", "exact", "audit"])
def test_reference_small_grid_cases(ctx, path, basis):
    """tests/test_search.cpp:177-204 cases, one launch for all of them."""
    radii, angles = uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    cases = [c for c in golden("small_cases.json") if c["basis"] == basis]
    res = ctx.search(np.array([c["target"] for c in cases], np.int32),
                     np.array([W.bits(c["pattern"]) for c in cases], np.int32),
                     np.array([c["v_th"] for c in cases]), np.array([c["r_novib"] for c in cases]),
                     radii, angles, path=path, delta_basis=basis)
    for s, c in enumerate(cases):
        idx, codes = split(res, s)
        assert len(idx) == c["count"], c
        assert sha_records(idx, codes) == c["sha256"], c
    assert_clean(res, path)


@pytest.mark.parametrize("path", ["fast", "audit", "pruned"])
def test_cfg1_full_sweep(ctx, path):
    wl = W.cfg1()
    res = run(ctx, wl, path=path)
    g = golden("workloads.json")["cfg1"]
    assert res["counts"].tolist() == g["counts"]
    assert res["n_pairs"] == g["total"] == 3785016
    assert sha_by_search(res) == g["sha256"]
    assert_clean(res, path)


def test_cfg1_counts_mode_matches_pairs(ctx):
    wl = W.cfg1()
    res = run(ctx, wl, output="counts")
    assert res["counts"].tolist() == golden("workloads.json")["cfg1"]["counts"]


@pytest.mark.parametrize("path", ["fast", "pruned"])
def test_cfg3_dense_targets(ctx, path):
    wl = W.cfg3()
    res = run(ctx, wl, path=path)
    g = golden("workloads.json")["cfg3"]
    assert res["counts"].tolist() == g["counts"]
    assert sha_by_search(res) == g["sha256"]
    assert_clean(res, "fast")


@pytest.mark.parametrize("path", ["fast", "pruned"])
def test_cfg4_first_pair_mode_crop(ctx, path):
    g = golden("workloads.json")["cfg4_256x144"]
    wl = W.cfg4(g["width"], g["height"])
    res = run(ctx, wl, output="first", path=path)
    import hashlib

    m = hashlib.sha256()
    m.update(res["counts"].astype(np.uint64).tobytes())
    m.update(np.ascontiguousarray(res["first_idx"], np.uint32).tobytes())
    m.update(np.ascontiguousarray(res["first_codes"], np.uint8).tobytes())
    assert int(res["counts"].sum()) == g["total"]
    assert m.hexdigest() == g["sha256"]


def test_duplicate_searches_share_constants(ctx):
    """Repeated (target, pattern, thresholds) share one constant record
    (hash dedup path); every search still gets its own full result."""
    wl = W.cfg1()
    rep = W.Workload("rep", np.concatenate([wl.targets, wl.targets[::-1]]),
                     np.concatenate([wl.patterns, wl.patterns[::-1]]), np.concatenate([wl.v_th, wl.v_th[::-1]]),
                     np.concatenate([wl.r_novib, wl.r_novib[::-1]]), wl.radii, wl.angles)
    res = run(ctx, rep)
    g = golden("workloads.json")["cfg1"]["counts"]
    assert res["counts"].tolist() == g + g[::-1]
    n = wl.n_searches
    for s in (0, 100, 755):
        a_idx, a_codes = split(res, s)
        b_idx, b_codes = split(res, 2 * n - 1 - s)
        assert np.array_equal(a_idx, b_idx) and np.array_equal(a_codes, b_codes)


@pytest.mark.slow
def test_cfg4_full_image_first_pair(ctx):
    g = golden("workloads.json").get("cfg4")
    if not g:
        pytest.skip("cfg4 golden not generated")
    wl = W.cfg4()
    res = run(ctx, wl, output="first")
    import hashlib

    m = hashlib.sha256()
    m.update(res["counts"].astype(np.uint64).tobytes())
    m.update(np.ascontiguousarray(res["first_idx"], np.uint32).tobytes())
    m.update(np.ascontiguousarray(res["first_codes"], np.uint8).tobytes())
    assert int(res["counts"].sum()) == g["total"]
    assert m.hexdigest() == g["sha256"]


@pytest.mark.slow
def test_cfg2_fine_grid_full_pair_set(ctx, oracle):
    """cfg2 (2.4G candidates, 444M pairs): per-target counts AND the full
    ordered record set of every target against the reference's own
    batch_search (tests/golden/make_golden.py --cfg2: 10-byte-record sha256
    per target), plus a few rows against the oracle directly."""
    wl = W.cfg2()
    res = run(ctx, wl)
    g = golden("workloads.json")["cfg2"]
    assert res["counts"].tolist() == g["counts"]
    assert res["n_pairs"] == g["total"] == 444092662
    assert_clean(res, "fast")
    for s in range(wl.n_searches):
        idx, codes = split(res, s)
        assert records10_sha(idx, codes) == g["sha256_records10"][s], f"cfg2 target {s} pair set differs"
    na = len(wl.angles)
    rows = [0, 1, 777, 2048, 4095]
    for s in (0, 3, 8):
        idx, codes = split(res, s)
        sub = W.Workload("sub", wl.targets[s:s + 1], wl.patterns[s:s + 1], wl.v_th[s:s + 1],
                         wl.r_novib[s:s + 1], wl.radii[rows], wl.angles)
        oi, oc = oracle_records(oracle, sub, 0, workers=8)
        k = idx // na
        sel = np.isin(k, rows)
        kk = np.searchsorted(np.array(rows), k[sel])
        assert np.array_equal(kk * na + idx[sel] % na, oi)
        assert np.array_equal(codes[sel], oc)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg2", "cfg3", "cfg4"])
def test_audit_bound_holds_on_large_configs(ctx, name):
    """AUDIT path (every candidate in FP32 and FP64) on the grids that stress
    the error bound most: cfg2 (r <= 128 on a 65536-angle grid), cfg3 (4096
    lattice targets incl. near-black), cfg4 (8.3M pixels, r <= 126, the
    linear branch of f^-1).  No FP32 decision claimed certain may be wrong,
    and every |lin32 - lin64| must stay inside its proven bound."""
    wl = W.ALL[name]()
    out = {"cfg2": "counts", "cfg3": "pairs", "cfg4": "first"}[name]
    res = run(ctx, wl, output=out, path="audit")
    g = golden("workloads.json")[name]
    assert int(res["counts"].sum()) == g["total"]
    if name != "cfg4":
        assert res["counts"].tolist() == g["counts"]
    st = res["stats"]
    assert st["audit_violations"] == 0, st
    assert 0.0 < st["audit_max_ratio"] < 1.0, st
    assert st["class_mismatch"] == 0, st


# ---- reference API through the Python binding (test_search.cpp pins) -------

def test_python_api_serial_equals_batch_and_oracle(cv, ctx, oracle):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    for t in ([170, 170, 170], [240, 240, 240], [100, 100, 240], [240, 100, 240], [8, 8, 8]):
        for p in ("100", "001", "101", "110", "111"):
            th = cv.Thresholds(50.0, 0.5)
            s = cv.serial_search(cv.SrgbColor(*t), grid, cv.BitPattern(p), th)
            b = cv.batch_search(cv.SrgbColor(*t), grid, cv.BitPattern(p), th)
            assert s == b
            oi, oc, od = oracle.search(t, W.bits(p), 50.0, 0.5, grid.radii, grid.angles, method=0)
            assert len(b) == len(oi)
            for pair, i, c, d in zip(b, oi, oc, od):
                assert pair.radius == grid.radii[i // len(grid.angles)]
                assert pair.angle == grid.angles[i % len(grid.angles)]
                assert [pair.plus.r, pair.plus.g, pair.plus.b, pair.minus.r, pair.minus.g, pair.minus.b] == c.tolist()
                assert [pair.deltas.dr, pair.deltas.dg, pair.deltas.db] == d.tolist()
                assert (pair.target.r, pair.target.g, pair.target.b) == tuple(t)


def test_worker_count_independence(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    args = (cv.SrgbColor(170, 170, 170), grid, cv.BitPattern("101"), cv.Thresholds(50.0, 0.5))
    base = cv.batch_search(*args, workers=1)
    assert base
    for w in (2, 3, 5, 16, 64):
        assert cv.batch_search(*args, workers=w) == base


def test_canonical_order_and_reverification(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    th = cv.Thresholds(50.0, 0.5)
    pairs = cv.batch_search(cv.SrgbColor(240, 240, 240), grid, cv.BitPattern("110"), th)
    assert len(pairs) > 1
    for a, b in zip(pairs, pairs[1:]):
        assert a.radius < b.radius or (a.radius == b.radius and a.angle < b.angle)
    lab = cv.srgb_to_lab(cv.SrgbColor(240, 240, 240))
    for p in pairs:
        lp, lm = cv.displaced_pair(lab, p.radius, p.angle)
        assert cv.lab_to_srgb_clipped(lp) == p.plus
        assert cv.lab_to_srgb_clipped(lm) == p.minus
        assert cv.channel_deltas(p.target, p.plus, p.minus) == p.deltas
        assert cv.classify_pair(p.deltas, cv.BitPattern("110"), th)
        assert lp.l == lab.l and lm.l == lab.l


def test_zero_radius_never_pairs(cv, ctx):
    grid = cv.VibrationGrid()
    grid.radii = [0.0]
    grid.angles = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0).angles
    for p in ("100", "010", "001", "110", "101", "011", "111"):
        args = (cv.SrgbColor(170, 170, 170), grid, cv.BitPattern(p), cv.Thresholds(50.0, 0.5))
        assert cv.serial_search(*args) == []
        assert cv.batch_search(*args) == []


def test_relaxing_r_novib_only_adds_pairs(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    for t in ((170, 170, 170), (100, 100, 240)):
        for p in ("100", "101", "111"):
            for v in (50.0, 100.0):
                sets = []
                for rn in (0.125, 0.25, 0.5):
                    pairs = cv.batch_search(cv.SrgbColor(*t), grid, cv.BitPattern(p), cv.Thresholds(v, rn))
                    sets.append({(x.radius, x.angle) for x in pairs})
                assert sets[0] <= sets[1] <= sets[2]


def test_frame_diff_basis(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    opts = cv.SearchOptions()
    opts.delta_basis = cv.DeltaBasis.FRAME_DIFF
    args = (cv.SrgbColor(170, 170, 170), grid, cv.BitPattern("101"), cv.Thresholds(50.0, 0.5))
    fd = cv.batch_search_opts(*args, opts)
    assert fd
    for p in fd:
        assert p.deltas == cv.frame_deltas(p.plus, p.minus)
    assert fd == cv.serial_search_opts(*args, opts)
    assert len(fd) != len(cv.batch_search(*args))


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("out", ["pairs", "counts", "first"])
def test_frame_diff_aligned_grid_outputs(ctx, oracle, mode, out):
    """FrameDiff on an aligned grid (na % 32 == 0): the FAST path's own row
    loops -- code bounds (Quantized, frame_tile) and FP32 signal bounds
    (Continuous) -- in every output mode, against the oracle search by search."""
    radii, angles = W.radii(48, 2.5), W.angles(256)
    rng = np.random.default_rng(17 + mode)
    n = 40
    t = rng.integers(0, 256, (n, 3)).astype(np.int32)
    t[:4] = [[0, 0, 0], [255, 255, 255], [8, 8, 8], [255, 0, 128]]
    p = rng.integers(1, 8, n).astype(np.int32)
    v = rng.choice([20.0, 50.0, 100.0, 150.5], n)
    r = rng.choice([0.125, 0.25, 0.5, 1.0], n)
    wl = W.Workload("fd", t, p, v, r, radii, angles)
    res = run(ctx, wl, basis=1, mode=mode, output=out)
    assert res["stats"]["class_mismatch"] == 0
    total = 0
    for s in range(n):
        oi, oc = oracle_records(oracle, wl, s, basis=1, workers=1, mode=mode)
        total += len(oi)
        assert res["counts"][s] == len(oi), s
        if out == "pairs":
            idx, codes = split(res, s)
            assert np.array_equal(idx, oi) and np.array_equal(codes, oc), s
        elif out == "first" and len(oi):
            assert res["first_idx"][s] == oi[0] and np.array_equal(res["first_codes"][s], oc[0]), s
    assert total > 1000


@pytest.mark.parametrize("path", ["fast", "audit", "exact"])
def test_continuous_target_swing_bit_exact(ctx, oracle, path):
    """DeltaMode::Continuous x TargetSwing (search.cpp:161-180): signal-space
    bands from the host bisection, decided on the device."""
    radii, angles = uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    t, p, v, r = [], [], [], []
    for tg in ([170, 170, 170], [240, 240, 240], [100, 100, 240], [240, 100, 240], [8, 8, 8], [0, 255, 30]):
        for pat in (1, 4, 5, 6, 7):
            for vt, rn in ((50.0, 0.5), (100.0, 0.25), (20.5, 0.333)):
                t.append(tg); p.append(pat); v.append(vt); r.append(rn)
    wl = W.Workload("cont", np.array(t, np.int32), np.array(p, np.int32), np.array(v), np.array(r), radii, angles)
    res = run(ctx, wl, path=path, mode=1)
    assert res["stats"]["audit_violations"] == 0
    for s in range(wl.n_searches):
        a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
        oi, oc, _ = oracle.search(wl.targets[s], int(wl.patterns[s]), wl.v_th[s], wl.r_novib[s], radii, angles,
                                  delta_mode=1, method=0, want_deltas=False)
        assert np.array_equal(res["idx"][a:b], oi), s
        assert np.array_equal(res["codes"][a:b], oc), s


def test_continuous_api_deltas_match_oracle(cv, ctx, oracle):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 5.0, 0.0, 355.0, 5.0)
    opts = cv.SearchOptions()
    opts.delta_mode = cv.DeltaMode.CONTINUOUS
    for t, p in (([170, 170, 170], "101"), ([100, 100, 240], "111"), ([240, 100, 100], "100")):
        got = cv.batch_search_opts(cv.SrgbColor(*t), grid, cv.BitPattern(p), cv.Thresholds(50.0, 0.5), opts)
        assert got == cv.serial_search_opts(cv.SrgbColor(*t), grid, cv.BitPattern(p), cv.Thresholds(50.0, 0.5),
                                            opts)
        oi, oc, od = oracle.search(t, W.bits(p), 50.0, 0.5, grid.radii, grid.angles, delta_mode=1, method=0)
        assert len(got) == len(oi)
        for pair, c, d in zip(got, oc, od):
            assert [pair.plus.r, pair.plus.g, pair.plus.b, pair.minus.r, pair.minus.g, pair.minus.b] == c.tolist()
            assert [pair.deltas.dr, pair.deltas.dg, pair.deltas.db] == d.tolist()


@pytest.mark.parametrize("path", ["fast", "exact", "audit"])
@pytest.mark.parametrize("out", ["pairs", "counts", "first"])
def test_continuous_frame_diff_bit_exact(ctx, oracle, path, out):
    """DeltaMode::Continuous x FrameDiff (search.cpp:146-173): |s(p) - s(m)|
    of device-pow signal values, decided with the glibc-pow margin."""
    radii, angles = uniform_grid(0.0, 128.0, 2.5, 0.0, 359.0, 1.0)
    t, p, v, r = [], [], [], []
    for tg in ([170, 170, 170], [240, 240, 240], [100, 100, 240], [240, 100, 240], [8, 8, 8], [0, 255, 30],
               [255, 255, 255], [0, 0, 0]):
        for pat in (1, 2, 4, 5, 6, 7):
            for vt, rn in ((50.0, 0.5), (100.0, 0.25), (20.5, 0.333), (3.0, 1.0)):
                t.append(tg); p.append(pat); v.append(vt); r.append(rn)
    wl = W.Workload("cfd", np.array(t, np.int32), np.array(p, np.int32), np.array(v), np.array(r), radii, angles)
    res = run(ctx, wl, path=path, mode=1, basis=1, output=out)
    # the FP32 signal-bound prefilter never decides against the FP64 path
    assert res["stats"]["audit_violations"] == 0
    if path == "fast":
        assert res["stats"]["band_repairs"] < wl.candidates // 20  # the prefilter decides most candidates
    total = 0
    for s in range(wl.n_searches):
        oi, oc, _ = oracle.search(wl.targets[s], int(wl.patterns[s]), wl.v_th[s], wl.r_novib[s], radii, angles,
                                  delta_mode=1, delta_basis=1, method=0, want_deltas=False)
        total += len(oi)
        assert res["counts"][s] == len(oi), s
        if out == "pairs":
            a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
            assert np.array_equal(res["idx"][a:b], oi), s
            assert np.array_equal(res["codes"][a:b], oc), s
        elif out == "first" and len(oi):
            assert res["first_idx"][s] == oi[0], s
            assert np.array_equal(res["first_codes"][s], oc[0]), s
    assert total > 1000


def test_continuous_frame_diff_api(cv, ctx, oracle):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 5.0, 0.0, 355.0, 5.0)
    opts = cv.SearchOptions()
    opts.delta_mode = cv.DeltaMode.CONTINUOUS
    opts.delta_basis = cv.DeltaBasis.FRAME_DIFF
    n = 0
    for t, p in (([170, 170, 170], "101"), ([100, 100, 240], "111"), ([240, 100, 100], "100"), ([8, 8, 8], "010")):
        args = (cv.SrgbColor(*t), grid, cv.BitPattern(p), cv.Thresholds(50.0, 0.5))
        got = cv.batch_search_opts(*args, opts)
        assert got == cv.serial_search_opts(*args, opts)
        oi, oc, od = oracle.search(t, W.bits(p), 50.0, 0.5, grid.radii, grid.angles, delta_mode=1, delta_basis=1,
                                   method=0)
        assert len(got) == len(oi)
        n += len(got)
        for pair, c, d in zip(got, oc, od):
            assert [pair.plus.r, pair.plus.g, pair.plus.b, pair.minus.r, pair.minus.g, pair.minus.b] == c.tolist()
            assert [pair.deltas.dr, pair.deltas.dg, pair.deltas.db] == d.tolist()
    assert n > 0


def test_batch_many_equals_single(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 60.0, 3.0, 0.0, 357.0, 3.0)
    specs = [cv.SearchSpec(cv.SrgbColor(*t), cv.BitPattern(p), cv.Thresholds(v, r))
             for t in ((100, 100, 100), (240, 100, 240)) for p in ("101", "111") for v, r in ((50, .5), (100, .25))]
    many = cv.batch_search_many(specs, grid)
    counts = cv.batch_count_many(specs, grid)
    for sp, got, n in zip(specs, many, counts):
        assert got == cv.batch_search(sp.target, grid, sp.pattern, sp.thresholds)
        assert n == len(got)


def test_concurrent_callers(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 5.0, 0.0, 355.0, 5.0)
    args = (cv.SrgbColor(170, 170, 170), grid, cv.BitPattern("101"), cv.Thresholds(50.0, 0.5))
    want = cv.batch_search(*args)
    out = [None] * 6

    def work(i):
        out[i] = cv.batch_search(*args)

    th = [threading.Thread(target=work, args=(i,)) for i in range(6)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert all(o == want for o in out)


# ---- edge cases -------------------------------------------------------------

EDGE_GRIDS = {
    "na1": (W.radii(50, 2.0), np.array([0.3])),
    "na7": (W.radii(33, 3.0), W.angles(7)),
    "na33": (W.radii(70, 1.5), W.angles(33)),
    "nr1": (np.array([40.0]), W.angles(4096)),
    "huge_r": (W.radii(16, 70.0), W.angles(512)),
    "tiny_r": (W.radii(64, 1e-3), W.angles(96)),
}
EDGE_TARGETS = [[0, 0, 0], [255, 255, 255], [8, 8, 8], [255, 0, 0], [0, 255, 255], [1, 254, 128], [128, 128, 128]]


@pytest.mark.parametrize("gname", sorted(EDGE_GRIDS))
@pytest.mark.parametrize("path", ["fast", "audit", "pruned"])
def test_edge_grids_vs_oracle(ctx, oracle, gname, path):
    radii, angles = EDGE_GRIDS[gname]
    t, p, v, r = [], [], [], []
    for tg in EDGE_TARGETS:
        for pat, vt, rn in ((7, 50.0, 0.5), (5, 100.0, 0.25), (2, 20.0, 1.0), (1, 300.0, 0.5), (6, 0.5, 1.0)):
            t.append(tg); p.append(pat); v.append(vt); r.append(rn)
    wl = W.Workload("edge", np.array(t, np.int32), np.array(p, np.int32), np.array(v), np.array(r), radii, angles)
    # Quantized x {TargetSwing, FrameDiff}, Continuous x FrameDiff (its FP32 prefilter)
    for mode, basis in ((0, 0), (0, 1), (1, 1)):
        res = run(ctx, wl, path=path, basis=basis, mode=mode)
        for s in range(wl.n_searches):
            idx, codes = split(res, s)
            oi, oc = oracle_records(oracle, wl, s, basis=basis, workers=1, mode=mode)
            assert np.array_equal(idx, oi), (gname, s, mode, basis)
            assert np.array_equal(codes, oc), (gname, s, mode, basis)
        assert_clean(res, path)


def test_custom_white_point(ctx, oracle):
    wp = [0.9642, 1.0, 0.8251]
    wl = W.Workload("wp", np.array([[120, 60, 200], [30, 200, 90]], np.int32), np.array([5, 7], np.int32),
                    np.array([50.0, 40.0]), np.array([0.5, 0.5]), W.radii(80, 1.25), W.angles(360))
    res = run(ctx, wl, white=wp, path="audit")
    for s in range(2):
        idx, codes = split(res, s)
        oi, oc = oracle_records(oracle, wl, s, white=wp)
        assert np.array_equal(idx, oi) and np.array_equal(codes, oc)
    assert_clean(res, "audit")


def test_empty_grid_and_empty_batch(ctx):
    wl = W.cfg0()
    res = ctx.search(wl.targets, wl.patterns, wl.v_th, wl.r_novib, np.zeros(0), wl.angles)
    assert res["n_pairs"] == 0 and res["counts"].tolist() == [0]
    res = ctx.search(np.zeros((0, 3), np.int32), np.zeros(0, np.int32), np.zeros(0), np.zeros(0), wl.radii,
                     wl.angles)
    assert res["n_pairs"] == 0


def test_plan_overflow_then_reserve(ctx):
    wl = W.cfg1()
    plan = ctx.plan(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles)
    plan.reserve(1000)  # far too small: counts stay valid, the pairs overflow
    plan.run()
    with pytest.raises(RuntimeError, match="too small"):
        plan.sync()
    plan.reserve(3785016)
    plan.run()
    assert plan.sync() == 3785016
    res = plan.fetch()
    assert sha_by_search(res) == golden("workloads.json")["cfg1"]["sha256"]
    for _ in range(3):  # repeated runs reuse the device buffers
        plan.run()
    assert plan.sync() == 3785016
    assert plan.launches == 4  # phase 1, tile lists (strip tiles), offset scan, emit
    # kernels chained by programmatic dependent launch: no per-kernel split
    # unless phase marks are requested (events between the kernels)
    with pytest.raises(ValueError, match="phase marks"):
        plan.last_phase_ms()
    plan.set_phase_marks(True)
    plan.run()
    assert plan.sync() == 3785016
    p1, sc, em = plan.last_phase_ms()
    assert p1 > 0 and sc > 0 and em > 0
    assert abs((p1 + sc + em) - plan.last_kernel_ms()) < 0.05 * plan.last_kernel_ms()
    plan.set_phase_marks(False)
    plan.run()
    assert plan.sync() == 3785016
    assert sha_by_search(plan.fetch()) == golden("workloads.json")["cfg1"]["sha256"]


def test_huge_single_search_linearity(ctx):
    """One search of 2^31 candidates (4096 radii x 524288 angles: candidate
    indices k*na + m up to 2^31, 524288 tiles): COUNTS and FIRST over the full
    grid equal the sum / first over four radius slices run as separate
    searches (the pair set of a search is a disjoint union over its rows)."""
    radii, angles = W.radii(4096, 0.03125), W.angles(524288)
    t = np.array([[200, 60, 90]], np.int32)
    p, v, r = np.array([5], np.int32), np.array([40.0]), np.array([0.5])
    full = ctx.search(t, p, v, r, radii, angles, output="first")
    total, first = 0, None
    for q in range(4):
        sl = radii[q * 1024:(q + 1) * 1024]
        part = ctx.search(t, p, v, r, sl, angles, output="first")
        c = int(part["counts"][0])
        if c and first is None:
            first = int(part["first_idx"][0]) + q * 1024 * len(angles)
            first_codes = part["first_codes"][0].tolist()
        total += c
    assert int(full["counts"][0]) == total > 0
    assert int(full["first_idx"][0]) == first
    assert full["first_codes"][0].tolist() == first_codes


# ---- CVG_PATH_MEMO (distinct searches only, scattered on the device) --------

@pytest.mark.parametrize("out", ["first", "counts"])
def test_memo_path_crop_matches_golden(ctx, out):
    g = golden("workloads.json")["cfg4_256x144"]
    wl = W.cfg4(g["width"], g["height"])
    res = run(ctx, wl, output=out, path="memo")
    full = run(ctx, wl, output=out)
    assert np.array_equal(res["counts"], full["counts"])
    assert int(res["counts"].sum()) == g["total"]
    if out == "first":
        import hashlib

        m = hashlib.sha256()
        m.update(res["counts"].astype(np.uint64).tobytes())
        m.update(np.ascontiguousarray(res["first_idx"], np.uint32).tobytes())
        m.update(np.ascontiguousarray(res["first_codes"], np.uint8).tobytes())
        assert m.hexdigest() == g["sha256"]


def test_memo_path_mixed_classifiers(ctx, oracle):
    """Repeated searches with different patterns / thresholds: the record key
    is (color, pattern, v_th, r_novib), not the color alone."""
    radii, angles = W.radii(40, 2.5), W.angles(128)
    rng = np.random.default_rng(5)
    base_t = rng.integers(0, 256, (12, 3)).astype(np.int32)
    n = 300
    pick = rng.integers(0, 12, n)
    t = base_t[pick]
    p = np.where(pick % 2 == 0, 7, 5).astype(np.int32)
    v = np.where(pick % 3 == 0, 50.0, 100.0)
    r = np.full(n, 0.5)
    wl = W.Workload("memo", t, p, v, r, radii, angles, output="first")
    res = run(ctx, wl, output="first", path="memo")
    full = run(ctx, wl, output="first")
    assert np.array_equal(res["counts"], full["counts"])
    assert np.array_equal(res["first_idx"], full["first_idx"])
    assert np.array_equal(res["first_codes"], full["first_codes"])
    for s in range(0, n, 37):
        oi, oc = oracle_records(oracle, wl, s, workers=1)
        assert res["counts"][s] == len(oi)
        if len(oi):
            assert res["first_idx"][s] == oi[0] and np.array_equal(res["first_codes"][s], oc[0])


def test_memo_path_rejects_pairs(ctx):
    wl = W.cfg0()
    with pytest.raises(ValueError):
        run(ctx, wl, output="pairs", path="memo")


def test_result_outlives_its_context(cv):
    """Result arrays view the context's pinned pool; dropping the context
    first must not free them (use-after-free)."""
    import gc

    wl = W.cfg0()
    c = cv.Context(0)
    res = c.search(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles)
    idx, codes = res["idx"], res["codes"]
    del c, res
    gc.collect()
    c2 = cv.Context(0)  # reuses the freed pinned memory if the result did not keep it
    junk = c2.search(wl.targets, wl.patterns, wl.v_th + 7.0, wl.r_novib, wl.radii, wl.angles)
    assert sha_records(idx, codes) == golden("workloads.json")["cfg0"]["sha256"]
    del junk, c2


# ---- PairView (lazy ColorPair materialization, module.cpp:121-131) ----------

def test_pair_view_equals_list(cv, ctx):
    grid = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    fd = cv.SearchOptions()
    fd.delta_basis = cv.DeltaBasis.FRAME_DIFF
    co = cv.SearchOptions()
    co.delta_mode = cv.DeltaMode.CONTINUOUS
    for t in ([170, 170, 170], [240, 100, 240], [8, 8, 8]):
        for p in ("101", "111", "010"):
            args = (cv.SrgbColor(*t), grid, cv.BitPattern(p), cv.Thresholds(50.0, 0.5))
            lst = cv.batch_search(*args)
            v = cv.batch_search_view(*args)
            assert len(v) == len(lst) and v == lst and v.to_list() == lst and list(v) == lst
            assert bool(v) == bool(lst)
            if lst:
                assert v[0] == lst[0] and v[-1] == lst[-1] and v[1:4] == lst[1:4]
                assert v.idx.dtype == np.uint32 and v.codes.shape == (len(lst), 6)
            for opts in (fd, co):
                assert cv.batch_search_view(*args, options=opts) == cv.batch_search_opts(*args, opts)
    with pytest.raises(IndexError):
        cv.batch_search_view(cv.SrgbColor(170, 170, 170), grid, cv.BitPattern("111"), cv.Thresholds(50.0, 0.5))[10 ** 6]
    with pytest.raises(ValueError):
        cv.batch_search_view(cv.SrgbColor(300, 0, 0), grid, cv.BitPattern("111"), cv.Thresholds(50.0, 0.5))


@pytest.mark.slow
def test_pair_view_cfg2_target_not_list_bound(cv, ctx):
    """A cfg2 target through the Python API (46M pairs): the view holds the
    10-byte records (reference-pinned sha), no 80-byte objects are built."""
    import time

    wl = W.cfg2()
    grid = cv.VibrationGrid()
    grid.radii = wl.radii.tolist()
    grid.angles = wl.angles.tolist()
    t0 = time.perf_counter()
    v = cv.batch_search_view(cv.SrgbColor(*wl.targets[0].tolist()), grid, cv.BitPattern("111"),
                             cv.Thresholds(50.0, 0.5))
    dt = time.perf_counter() - t0
    g = golden("workloads.json")["cfg2"]
    assert len(v) == g["counts"][0]
    assert records10_sha(v.idx, v.codes) == g["sha256_records10"][0]
    p = v[len(v) // 2]
    assert p.radius == wl.radii[v.idx[len(v) // 2] // len(wl.angles)]
    assert dt < 10.0, dt  # list materialization of 46M ColorPair objects takes minutes


# ---- strip tiles (COUNTS / FIRST, band FAST path: lane per angle) ----------

@pytest.mark.parametrize("nr,na", [(24, 7), (40, 100), (33, 130), (64, 256), (70, 384), (100, 33)])
@pytest.mark.parametrize("out", ["counts", "first"])
def test_strip_tiles_edge_shapes(ctx, oracle, nr, na, out):
    """Partial row blocks (nr % 32), partial angle blocks (na % 128), odd na,
    against the oracle search by search; same answer with row-major tiles
    (path 'pruned' keeps row-major tiles)."""
    radii, angles = W.radii(nr, 126.0 / max(nr - 1, 1)), W.angles(na)
    rng = np.random.default_rng(nr * 1000 + na)
    n = 24
    t = rng.integers(0, 256, (n, 3)).astype(np.int32)
    t[:3] = [[0, 0, 0], [255, 255, 255], [8, 8, 8]]
    p = rng.integers(1, 8, n).astype(np.int32)
    v = rng.choice([30.0, 50.0, 100.0], n)
    r = rng.choice([0.25, 0.5, 1.0], n)
    wl = W.Workload("cols", t, p, v, r, radii, angles, output=out)
    res = run(ctx, wl, output=out)
    rowm = run(ctx, wl, output=out, path="pruned")
    assert np.array_equal(res["counts"], rowm["counts"])
    for s in range(n):
        oi, oc = oracle_records(oracle, wl, s, workers=1)
        assert res["counts"][s] == len(oi), s
        if out == "first":
            if len(oi):
                assert res["first_idx"][s] == oi[0] and np.array_equal(res["first_codes"][s], oc[0]), s
            else:
                assert res["first_idx"][s] == 0xFFFFFFFF


# ---- twin tiles (PAIRS, rows of whole tiles, grid symmetric under +pi) -----

def _twin_workload(na, angles=None, nr=36, n=6, seed=7):
    rng = np.random.default_rng(seed)
    t = rng.integers(60, 250, (n, 3)).astype(np.int32)
    t[0] = [170, 170, 170]
    t[1] = [8, 8, 8]  # near black: the linear branch of f^-1
    p = rng.integers(1, 8, n).astype(np.int32)
    p[0] = 7
    v = rng.choice([50.0, 100.0], n)
    r = rng.choice([0.25, 0.5], n)
    return W.Workload("twin", t, p, v, r, W.radii(nr, 128.0 / (nr - 1)),
                      W.angles(na) if angles is None else angles)


@pytest.mark.parametrize("na", [8192, 16384])
def test_twin_tiles_match_oracle(ctx, oracle, na, monkeypatch):
    """Twin tiles on: every search's records equal the oracle's; the same
    with both lists built for every odd row (the split path a differing twin
    row takes) and with twins off."""
    wl = _twin_workload(na)
    plan = ctx.plan(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles)
    assert plan.twin_tiles
    res = run(ctx, wl)
    assert_clean(res, "fast")
    assert res["n_pairs"] > 0
    for s in range(wl.n_searches):
        oi, oc = oracle_records(oracle, wl, s, workers=8)
        idx, codes = split(res, s)
        assert np.array_equal(idx, oi), s
        assert np.array_equal(codes, oc), s
    want = sha_by_search(res)
    monkeypatch.setenv("CVG_TWIN_SPLIT_TEST", "1")
    assert sha_by_search(run(ctx, wl)) == want
    monkeypatch.delenv("CVG_TWIN_SPLIT_TEST")
    monkeypatch.setenv("CVG_TWIN", "0")
    plan0 = ctx.plan(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles)
    assert not plan0.twin_tiles
    assert sha_by_search(run(ctx, wl)) == want


def test_twin_tiles_off_on_asymmetric_grid(ctx, oracle):
    """Angles over half a circle: no twin tiles; results still exact."""
    na = 8192
    angles = np.pi * np.arange(na) / na
    wl = _twin_workload(na, angles=angles, nr=20)
    plan = ctx.plan(wl.targets, wl.patterns, wl.v_th, wl.r_novib, wl.radii, wl.angles)
    assert not plan.twin_tiles
    res = run(ctx, wl)
    for s in range(wl.n_searches):
        oi, oc = oracle_records(oracle, wl, s, workers=8)
        idx, codes = split(res, s)
        assert np.array_equal(idx, oi) and np.array_equal(codes, oc), s


def test_ranged_batch_validates_range_by_range(ctx):
    """A COUNTS batch of >= 2^20 searches runs as search ranges, each
    validated just before its plan: a bad search in a late range still fails
    the call with the message the whole-batch check gives, and the context
    keeps working."""
    n = (1 << 20) + 7
    rng = np.random.default_rng(5)
    t = rng.integers(0, 256, (n, 3)).astype(np.int32)
    p = rng.integers(1, 8, n).astype(np.int32)
    v = np.full(n, 100.0)
    r = np.full(n, 0.25)
    radii, angles = W.radii(4, 20.0), W.angles(32)
    ok = ctx.search(t, p, v, r, radii, angles, output="counts")
    assert len(ok["counts"]) == n
    for field, idx, val in (("patterns", n - 3, 0), ("v_th", n - 1, -1.0), ("targets", 5, 300)):
        tt, pp, vv = t.copy(), p.copy(), v.copy()
        {"patterns": pp, "v_th": vv, "targets": tt}[field][idx] = val
        with pytest.raises(ValueError) as big:
            ctx.search(tt, pp, vv, r, radii, angles, output="counts")
        one = slice(idx, idx + 1)
        with pytest.raises(ValueError) as small:
            ctx.search(tt[one], pp[one], vv[one], r[one], radii, angles, output="counts")
        assert str(big.value) == str(small.value), field
    again = ctx.search(t, p, v, r, radii, angles, output="counts")
    assert np.array_equal(again["counts"], ok["counts"])


@pytest.mark.parametrize("out", ["counts", "first"])
def test_strip_bulk_skip_random_grids_vs_exact(ctx, out):
    """The strip tiles' bulk skip of the inner rows (a bound on the strip
    form, bisection over row groups) on random targets, patterns, thresholds
    and irregular radius grids up to r = 150 (deep into the linear branch of
    f^-1): FAST (strip tiles + skip) equals EXACT (FP64 op-for-op, row-major
    tiles) search by search."""
    rng = np.random.default_rng(11)
    for trial in range(3):
        nr = int(rng.integers(20, 140))
        radii = np.sort(rng.uniform(0.0, 150.0, nr))
        radii = np.unique(radii)
        na = int(rng.choice([64, 96, 128, 256]))
        n = 96
        t = rng.integers(0, 256, (n, 3)).astype(np.int32)
        p = rng.integers(1, 8, n).astype(np.int32)
        v = rng.uniform(20.0, 200.0, n)
        r = rng.uniform(0.1, 1.0, n)
        wl = W.Workload("skip", t, p, v, r, radii, W.angles(na), output=out)
        fast = run(ctx, wl, output=out)
        exact = run(ctx, wl, output=out, path="exact")
        assert np.array_equal(fast["counts"], exact["counts"]), trial
        if out == "first":
            assert np.array_equal(fast["first_idx"], exact["first_idx"]), trial
            assert np.array_equal(fast["first_codes"], exact["first_codes"]), trial
