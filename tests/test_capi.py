"""C-ABI and host-side API checks that need no GPU.

* libcolorvibe_gpu.so loads and exports every function include/cvg.h declares;
* validation mirrors the reference (messages and exception types,
  reference src/color.cpp:27-39, src/search.cpp:22-30, 49-56, 92-111) and
  runs before any device work;
* the host scalar helpers equal the oracle bit for bit;
* the reference API types behave like the reference's unit tests
  (tests/test_search.cpp:42-175, test_color.cpp:103-200).
"""
import ctypes as C
import math
import re
import os

import numpy as np
import pytest

import paper_2507_22901_b200 as cv
from cvtest_util import golden
from paper_2507_22901_b200 import workloads as W

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "cvg.h")


@pytest.fixture(scope="module")
def lib():
    return C.CDLL(cv.LIBRARY_PATH)


class Desc(C.Structure):
    _fields_ = [("n_searches", C.c_int32), ("target_rgb", C.POINTER(C.c_int32)),
                ("pattern_bits", C.POINTER(C.c_int32)), ("v_th", C.POINTER(C.c_double)),
                ("r_novib", C.POINTER(C.c_double)), ("n_radii", C.c_int32), ("radii", C.POINTER(C.c_double)),
                ("n_angles", C.c_int32), ("angles", C.POINTER(C.c_double)), ("delta_mode", C.c_int32),
                ("delta_basis", C.c_int32), ("white_point", C.POINTER(C.c_double)), ("output", C.c_int32),
                ("path", C.c_int32), ("workers", C.c_int32)]


def declared_functions():
    txt = open(HEADER).read()
    return re.findall(r"CVG_API\s+[\w\s\*]+?\b(cvg_\w+)\s*\(", txt)


def test_every_declared_symbol_is_exported(lib):
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n


def _desc(targets, patterns, vth, rn, radii, angles, mode=0, basis=0):
    keep = [np.ascontiguousarray(targets, np.int32), np.ascontiguousarray(patterns, np.int32),
            np.ascontiguousarray(vth, np.float64), np.ascontiguousarray(rn, np.float64),
            np.ascontiguousarray(radii, np.float64), np.ascontiguousarray(angles, np.float64)]
    d = Desc()
    d.n_searches = len(keep[1])
    d.target_rgb = keep[0].ctypes.data_as(C.POINTER(C.c_int32))
    d.pattern_bits = keep[1].ctypes.data_as(C.POINTER(C.c_int32))
    d.v_th = keep[2].ctypes.data_as(C.POINTER(C.c_double))
    d.r_novib = keep[3].ctypes.data_as(C.POINTER(C.c_double))
    d.n_radii = len(keep[4])
    d.radii = keep[4].ctypes.data_as(C.POINTER(C.c_double))
    d.n_angles = len(keep[5])
    d.angles = keep[5].ctypes.data_as(C.POINTER(C.c_double))
    d.delta_mode, d.delta_basis = mode, basis
    return d, keep


def _validate(lib, *a, **k):
    d, keep = _desc(*a, **k)
    lib.cvg_validate.restype = C.c_int
    lib.cvg_last_error.restype = C.c_char_p
    st = lib.cvg_validate(C.byref(d))
    return st, lib.cvg_last_error().decode()


GRID = W.uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)


@pytest.mark.parametrize("case,status,msg", [
    (dict(targets=[[170, 170, 300]]), 1, "sRGB channel code outside [0, 255]: (170, 170, 300)"),
    (dict(targets=[[-1, 0, 0]]), 1, "sRGB channel code outside [0, 255]: (-1, 0, 0)"),
    (dict(radii=[1.0, -2.0]), 1, "grid radii must be non-negative"),
    (dict(radii=[-1.0]), 1, "grid radii must be non-negative"),
    (dict(radii=[3.0, 2.0]), 1, "grid radii must be strictly increasing"),
    (dict(angles=[0.0, 7.0]), 1, "grid angles must lie in [0, 2pi)"),
    (dict(angles=[1.0, 0.5]), 1, "grid angles must be strictly increasing"),
    (dict(vth=[0.0]), 1, "v_th must be positive"),
    (dict(vth=[float("nan")]), 1, "v_th must be positive"),
    (dict(rn=[0.0]), 1, "r_novib must be in (0, 1]"),
    (dict(rn=[1.5]), 1, "r_novib must be in (0, 1]"),
    (dict(patterns=[0]), 1, "bit pattern has no set bits"),
    (dict(mode=2), 1, "unknown delta_mode"),
])
def test_validation_mirrors_reference(lib, case, status, msg):
    args = dict(targets=[[170, 170, 170]], patterns=[5], vth=[50.0], rn=[0.5], radii=GRID[0], angles=GRID[1])
    args.update(case)
    st, err = _validate(lib, args["targets"], args["patterns"], args["vth"], args["rn"], args["radii"],
                        args["angles"], mode=args.get("mode", 0), basis=args.get("basis", 0))
    assert st == status
    assert msg in err


def test_validation_accepts_reference_inputs(lib):
    st, _ = _validate(lib, [[170, 170, 170]], [5], [50.0], [0.5], GRID[0], GRID[1])
    assert st == 0
    st, _ = _validate(lib, [[170, 170, 170]], [5], [50.0], [0.5], [], [])  # empty grid is valid
    assert st == 0
    st, _ = _validate(lib, [[170, 170, 170]], [5], [50.0], [0.5], GRID[0], GRID[1], mode=1)  # continuous swing
    assert st == 0
    st, _ = _validate(lib, [[170, 170, 170]], [5], [50.0], [0.5], GRID[0], GRID[1], mode=1, basis=1)
    assert st == 0  # continuous frame diff: runs on the device


def test_create_without_device_fails_loudly(lib):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    ctx = C.c_void_p()
    lib.cvg_create.restype = C.c_int
    assert lib.cvg_create(0, C.byref(ctx)) == 2  # CVG_ECUDA, never a CPU fallback
    with pytest.raises(RuntimeError):
        cv.batch_search(cv.SrgbColor(170, 170, 170), cv.VibrationGrid.uniform(1, 91, 10, 0, 350, 10),
                        cv.BitPattern("101"), cv.Thresholds(50, 0.5))


# ---- host scalar helpers vs the oracle ------------------------------------

def test_thresholds_and_white_point_match_golden():
    ka = golden("known_answers.json")
    assert np.array_equal(cv.quant_thresholds(), [float.fromhex(x) for x in ka["thresholds"]])
    w = cv.d65_white()
    assert [w.x, w.y, w.z] == [float.fromhex(x) for x in ka["white"]]
    assert w.y == 1.0


def test_srgb_to_lab_bit_exact_vs_oracle(oracle):
    rng = np.random.default_rng(7)
    for rgb in rng.integers(0, 256, (2000, 3)):
        lab = cv.srgb_to_lab(cv.SrgbColor(*map(int, rgb)))
        assert [lab.l, lab.a, lab.b] == oracle.srgb_to_lab(rgb).tolist()


def test_lab_to_srgb_clipped_vs_oracle(oracle):
    rng = np.random.default_rng(99)
    for _ in range(2000):
        lab = [rng.uniform(0, 100), rng.uniform(-150, 150), rng.uniform(-150, 150)]
        got = cv.lab_to_srgb_clipped(cv.LabColor(*lab))
        lin = oracle.lab_to_linear(lab)
        assert [got.r, got.g, got.b] == [oracle.quantize(x) for x in lin]


def test_palette_round_trip_and_gamut():
    for t in W.TABLE1:
        c = cv.SrgbColor(*map(int, t))
        assert cv.lab_to_srgb(cv.srgb_to_lab(c)) == c
        assert cv.lab_to_srgb_clipped(cv.srgb_to_lab(c)) == c
    assert cv.lab_to_srgb(cv.LabColor(50.0, 200.0, 0.0)) is None
    assert cv.lab_to_srgb(cv.LabColor(5.0, 0.0, -100.0)) is None
    assert 0 <= cv.lab_to_srgb_clipped(cv.LabColor(50.0, 200.0, 0.0)).r <= 255
    with pytest.raises(ValueError):
        cv.lab_to_srgb(cv.LabColor(100.5, 0, 0))
    with pytest.raises(ValueError):
        cv.srgb_to_lab(cv.SrgbColor(0, 256, 0))


# ---- reference API types (test_search.cpp pins) ----------------------------

def test_bit_pattern_parsing():
    p = cv.BitPattern.parse("101")
    assert p.r and not p.g and p.b and str(p) == "101"
    for bad in ("000", "10", "1011", "1a0"):
        with pytest.raises(ValueError):
            cv.BitPattern.parse(bad)


def test_thresholds_validation_and_low_band():
    for v, r in ((0.0, 0.5), (-1.0, 0.5), (50.0, 0.0), (50.0, 1.5)):
        with pytest.raises(ValueError):
            cv.Thresholds(v, r).validate()
    cv.Thresholds(50.0, 1.0).validate()
    assert cv.Thresholds(50.0, 0.5).low_band() == 25.0


def test_uniform_grid():
    g = cv.VibrationGrid.uniform(1, 100, 1, 0, 359, 1)
    assert len(g.radii) == 100 and len(g.angles) == 360
    assert g.radii[0] == 1.0 and g.radii[-1] == 100.0 and g.angles[0] == 0.0
    assert math.isclose(g.angles[-1], 359.0 * math.pi / 180.0)
    assert g.candidate_count() == 36000
    assert cv.VibrationGrid.standard().candidate_count() == 36000
    for args in ((10, 1, 1, 0, 359, 1), (1, 10, 0, 0, 359, 1), (1, 10, 1, 0, 360, 1)):
        with pytest.raises(ValueError):
            cv.VibrationGrid.uniform(*args)
    bad = cv.VibrationGrid()
    bad.radii = [3.0, 2.0]
    bad.angles = [0.0]
    with pytest.raises(ValueError):
        bad.validate()
    r, a = W.uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    g = cv.VibrationGrid.uniform(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    assert g.radii == r.tolist() and g.angles == a.tolist()


def test_displaced_pair_geometry():
    t = cv.LabColor(50.0, 4.0, -3.0)
    p, m = cv.displaced_pair(t, 0.0, 1.234)
    assert (p.l, p.a, p.b) == (t.l, t.a, t.b) and (m.a, m.b) == (t.a, t.b)
    p, m = cv.displaced_pair(t, 10.0, 0.0)
    assert p.a == t.a and p.b == t.b + 10.0 and m.b == t.b - 10.0
    p, m = cv.displaced_pair(t, 77.0, 2.1)
    assert p.l == t.l and m.l == t.l
    rng = np.random.default_rng(5)
    for r, j in zip(rng.uniform(0, 100, 200), rng.uniform(0, math.pi, 200)):
        p1, m1 = cv.displaced_pair(t, r, j)
        p2, m2 = cv.displaced_pair(t, r, j + math.pi)
        assert abs(p2.a - m1.a) < 1e-9 and abs(p2.b - m1.b) < 1e-9
        assert abs(m2.a - p1.a) < 1e-9 and abs(m2.b - p1.b) < 1e-9
    with pytest.raises(ValueError):
        cv.displaced_pair(t, -1.0, 0.0)


def test_channel_and_frame_deltas():
    t, p, m = cv.SrgbColor(100, 100, 100), cv.SrgbColor(150, 90, 100), cv.SrgbColor(60, 100, 100)
    ts = cv.channel_deltas(t, p, m)
    assert (ts.dr, ts.dg, ts.db) == (50.0, 10.0, 0.0)
    fd = cv.frame_deltas(p, m)
    assert (fd.dr, fd.dg, fd.db) == (90.0, 10.0, 0.0)
    rng = np.random.default_rng(11)
    for a, b, c in rng.integers(0, 256, (500, 3, 3)):
        A, B, Cc = (cv.SrgbColor(*map(int, x)) for x in (a, b, c))
        assert cv.channel_deltas(A, B, Cc) == cv.channel_deltas(A, Cc, B)
        assert cv.frame_deltas(B, Cc) == cv.frame_deltas(Cc, B)


def test_classify_pair_band_semantics():
    th = cv.Thresholds(50.0, 0.5)
    D, P = cv.ChannelDeltas, cv.BitPattern.parse
    assert cv.classify_pair(D(51.0, 25.0, 25.0), P("100"), th)
    assert not cv.classify_pair(D(50.0, 0.0, 0.0), P("100"), th)
    assert cv.classify_pair(D(0.0, 0.0, 51.0), P("001"), th)
    assert cv.classify_pair(D(25.0, 25.0, 51.0), P("001"), th)
    assert not cv.classify_pair(D(26.0, 0.0, 51.0), P("001"), th)
    assert not cv.classify_pair(D(40.0, 0.0, 0.0), P("100"), th)
    assert not cv.classify_pair(D(0.0, 40.0, 51.0), P("001"), th)
    assert cv.classify_pair(D(51.0, 51.0, 51.0), P("111"), th)


def test_select_best_margin_and_ties():
    """tests/test_search.cpp:316-351."""
    th = cv.Thresholds(50.0, 0.5)
    D = cv.ChannelDeltas
    a = cv.ColorPair(radius=10.0, angle=0.1, deltas=D(60.0, 20.0, 60.0))  # margin 5
    b = cv.ColorPair(radius=20.0, angle=0.2, deltas=D(70.0, 5.0, 80.0))   # margin 20
    c = cv.ColorPair(radius=15.0, angle=0.3, deltas=D(70.0, 5.0, 80.0))   # same margin, smaller radius
    assert cv.classification_margin(a, th) == 5.0
    assert cv.classification_margin(b, th) == 20.0
    assert cv.select_best([a, b, c], th).radius == 15.0
    d = cv.ColorPair(radius=15.0, angle=0.05, deltas=D(70.0, 5.0, 80.0))
    assert cv.select_best([a, b, c, d], th).angle == 0.05
    with pytest.raises(ValueError):
        cv.select_best([], th)


def _code64(x, thr):
    """QuantTable::code (convert_kernel.hpp:143-154) as 'thresholds at or below x'."""
    c = np.searchsorted(thr[1:], x, side="right")
    return np.where(x <= 0.0, 0, np.where(x >= 1.0, 255, c))


@pytest.mark.parametrize("E", [2.0 ** -22, 1e-6, 2.0 ** -16])
def test_code_table_proof(lib, E):
    """The kernels' FP32 code lookup (cvg_kernels.cu code_fast) restated in
    numpy over the exported table: wherever it claims a verified code
    (|xs - t| > E), every FP64 value within eps = E - 2^-23 of the FP32 value
    has that code (QuantTable::code, convert_kernel.hpp:143-154).  Probes: every
    float threshold +- 64 ulps and 2M uniform values in [-0.1, 1.1]."""
    tab = np.zeros(8194, np.float32)
    lib.cvg_code_table(tab.ctypes.data_as(C.POINTER(C.c_float)))
    lib.cvg_code_slack.restype = C.c_float
    assert E <= lib.cvg_code_slack() + 1e-12
    thr = np.zeros(256, np.float64)
    lib.cvg_quant_thresholds(thr.ctypes.data_as(C.POINTER(C.c_double)))
    t_tab = tab[0::2]
    c_tab = tab[1::2].view(np.int32)
    assert np.all(np.diff(c_tab) >= 0) and c_tab[0] == 0 and c_tab[-1] == 255
    tf = thr[1:].astype(np.float32)
    near = (tf[:, None].view(np.int32) + np.arange(-64, 65, dtype=np.int32)[None, :]).view(np.float32).ravel()
    rng = np.random.default_rng(5)
    x = np.concatenate([near, rng.uniform(-0.1, 1.1, 2_000_000).astype(np.float32),
                        np.float32([0.0, 1.0, -1e-9, 1.0 + 1e-7])])
    xs = np.clip(x, np.float32(0), np.float32(1))
    b = np.rint(xs.astype(np.float64) * 4096).astype(np.int64)  # fmaf(xs, 4096, 2^23): round half even
    t = t_tab[b]
    with np.errstate(invalid="ignore"):
        ok = np.abs(xs - t) > np.float32(E)
        code = c_tab[b] + (xs >= t)
    eps = E - 2.0 ** -23
    x64 = x.astype(np.float64)
    lo, hi = _code64(x64 - eps, thr), _code64(x64 + eps, thr)
    assert np.array_equal(code[ok], lo[ok]) and np.array_equal(code[ok], hi[ok])
    # the unverified share is the +-E windows around the 255 thresholds
    assert ok[len(near):].mean() > 1.0 - 600 * E


def test_signal_table_bounds(lib):
    """The Continuous x FrameDiff prefilter's table (cvg_kernels.cu
    signal_bounds): for every double x in bucket i = [(i - 1/2), (i + 1/2)] / 4096,
    L[i] <= signal_value(x) <= U[i] (convert_kernel.hpp:109-112), and the
    bounds are tight enough to decide almost every candidate."""
    tab = np.zeros(8194, np.float32)
    lib.cvg_signal_table(tab.ctypes.data_as(C.POINTER(C.c_float)))
    L, U = tab[0::2].astype(np.float64), tab[1::2].astype(np.float64)

    def signal(x):
        x = np.clip(x, 0.0, 1.0)
        return 255.0 * np.where(x <= 0.0031308, 12.92 * x, 1.055 * np.power(x, 1.0 / 2.4) - 0.055)

    rng = np.random.default_rng(11)
    i = np.arange(4097)
    edges = np.concatenate([(i - 0.5) / 4096, (i + 0.5) / 4096])
    x = np.concatenate([rng.uniform(-0.05, 1.05, 1_000_000), edges, np.nextafter(edges, 2), np.nextafter(edges, -2)])
    b = np.clip(np.rint(np.clip(x, 0, 1) * 4096), 0, 4096).astype(np.int64)
    inside = (np.clip(x, 0, 1) >= (b - 0.5) / 4096) & (np.clip(x, 0, 1) <= (b + 0.5) / 4096)
    s = signal(x)
    assert np.all(L[b][inside] <= s[inside]) and np.all(s[inside] <= U[b][inside])
    assert np.all(np.diff(L) >= 0) and np.all(np.diff(U) >= 0) and L[0] <= 0.0 and U[-1] >= 255.0
    assert (U - L).max() < 1.0 and np.median(U - L) < 0.05


def test_frame_diff_linear_bounds(lib):
    """The Quantized x FrameDiff linear-space prefilter (cvg_host.h
    Tables::fd_loud / fd_quiet, cvg_kernels.cu frame_surely_fails): with
    D_loud(k1) = min_c thr[c+k1-1] - thr[c] and D_quiet(q0) = max_c
    thr[min(c+q0+1, 256)] - thr[c] (thr[256] = 1), clamped values with
    |x_p - x_m| <= D_loud(k1) never have |code_p - code_m| >= k1, and values with
    |x_p - x_m| > D_quiet(q0) never have |code_p - code_m| <= q0 (frame_deltas,
    search.cpp:138-144, on QuantTable codes)."""
    thr = np.zeros(256, np.float64)
    lib.cvg_quant_thresholds(thr.ctypes.data_as(C.POINTER(C.c_double)))
    ext = np.concatenate([thr, [1.0]])
    rng = np.random.default_rng(23)
    xp = np.clip(rng.uniform(-0.05, 1.05, 400_000), 0, 1)
    # differences concentrated near the bounds as well as spread out
    xm = np.clip(xp + rng.normal(0, 0.2, xp.size) * rng.choice([1e-3, 1e-2, 1e-1, 1.0], xp.size), 0, 1)
    d = np.abs(xp - xm)
    code = lambda x: _code64(x, thr)  # noqa: E731
    dc = np.abs(code(xp) - code(xm))
    for k1 in (1, 2, 11, 51, 101, 151, 201, 255):
        dl = min(thr[c + k1 - 1] - thr[c] for c in range(1, 257 - k1))
        assert not np.any((d <= dl) & (dc >= k1)), k1
    for q0 in (0, 1, 6, 12, 25, 50, 100, 200, 254):
        dq = max(ext[min(c + q0 + 1, 256)] - thr[c] for c in range(256))
        assert not np.any((d > dq) & (dc <= q0)), q0


def test_continuous_frame_diff_linear_bounds():
    """The Continuous x FrameDiff linear-space prefilter (cvg_prep.cpp
    frame_signal_bounds): signal_value s is increasing and concave on [0, 1],
    so |x_p - x_m| <= a with s(a) <= T - 1e-6 gives |s_p - s_m| < T, and
    |x_p - x_m| >= 1 - b with s(b) <= 255 - T - 1e-6 gives |s_p - s_m| > T
    (convert_kernel.hpp:109-112, search.cpp:161-173).  Checked on clamped
    random pairs, concentrated near each bound."""
    def s(x):
        x = np.clip(x, 0.0, 1.0)
        return 255.0 * np.where(x <= 0.0031308, 12.92 * x, 1.055 * np.power(x, 1.0 / 2.4) - 0.055)

    def largest_below(v):
        lo, hi = 0.0, 1.0
        for _ in range(80):
            mid = 0.5 * (lo + hi)
            if s(mid) <= v:
                lo = mid
            else:
                hi = mid
        return lo

    rng = np.random.default_rng(29)
    for T in (3.0, 6.25, 12.5, 25.0, 50.0, 100.0, 150.0, 200.0, 250.0):
        a = largest_below(T - 1e-6)
        q = 1.0 - largest_below(255.0 - T - 1e-6)
        x = rng.uniform(0, 1, 300_000)
        for dx, want in ((a, "below"), (q, "above")):
            d = dx * (1 + rng.choice([-1e-3, -1e-9, 0.0], x.size)) if want == "below" else \
                dx * (1 + rng.choice([1e-3, 1e-9, 0.0], x.size))
            y = np.clip(x + d * rng.choice([-1, 1], x.size), 0, 1)
            real = np.abs(np.clip(x, 0, 1) - y)
            ds = np.abs(s(x) - s(y))
            if want == "below":
                sel = real <= a
                assert np.all(ds[sel] < T), T
            else:
                sel = real >= q
                assert np.all(ds[sel] > T), T
