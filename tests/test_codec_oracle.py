"""The codec oracle and the host side of the codec API, on CPU.

* oracle/codec_oracle.py (NumPy restatement of codec.cpp) is pinned against
  the reference's own codec (oracle/_ref/libcolorvibe_ref_codec.so): frames of
  embed_blocks, decode_blocks results bit for bit.
* The sidecar JSON text of our C++ API equals the reference's nlohmann
  ordered_json dump(2) text byte for byte; layout_from_json round-trips and
  rejects what the reference rejects (test_codec.cpp:226-250).
* Validation messages of BlockLayout / DisplayParams equal the reference's
  (test_codec.cpp:33-65).
"""
import numpy as np
import pytest

from oracle import codec_oracle as CO
from paper_2507_22901_b200 import workloads as W

KTH = (50.0, 0.5)


def matrix_grid():
    return W.uniform_grid(1.0, 76.0, 15.0, 9.0, 359.0, 12.0)


def random_layout(rng, w, h, bw, bh, n_max):
    """Non-overlapping blocks by rejection on a coarse occupancy grid."""
    taken = np.zeros((h, w), bool)
    xy = []
    for _ in range(n_max * 4):
        x, y = int(rng.integers(0, w - bw + 1)), int(rng.integers(0, h - bh + 1))
        if not taken[y:y + bh, x:x + bw].any():
            taken[y:y + bh, x:x + bw] = True
            xy.append((x, y))
        if len(xy) == n_max:
            break
    return np.array(xy, np.int32).reshape(-1, 2)


def oracle_embed(oracle, base, bw, bh, xy, rgb, bits, v_th, r_novib, radii, angles):
    plus, minus = [], []
    for t, b in zip(rgb, bits):
        idx, codes, _ = oracle.search(t, int(b), v_th, r_novib, radii, angles, method=1, want_deltas=False)
        assert len(idx), "infeasible block in test layout"
        j = CO.select_best(codes, t, v_th, r_novib)
        plus.append(codes[j, :3])
        minus.append(codes[j, 3:])
    return CO.paint(base, bw, bh, xy, plus, minus)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_oracle_embed_matches_reference(oracle, ref_codec, seed):
    rng = np.random.default_rng(seed)
    radii, angles = matrix_grid()
    h, w, bw, bh = 40, 56, 8, 6
    base = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    xy = random_layout(rng, w, h, bw, bh, 12)
    # feasible (color, pattern) cells of the default sweep (test_codec.cpp:160-195)
    cells = [(c, p) for c in W.TABLE1 for p in (W.bits(s) for s in W.PATTERNS)]
    rng.shuffle(cells)
    rgb, bits = [], []
    for c, p in cells:
        idx, _, _ = oracle.search(c, p, *KTH, radii, angles, method=1, want_deltas=False)
        if len(idx):
            rgb.append(c)
            bits.append(p)
        if len(rgb) == len(xy):
            break
    rgb, bits = np.array(rgb, np.int32), np.array(bits, np.int32)
    fa, fb = ref_codec.embed(base, bw, bh, xy, rgb, bits, *KTH, radii, angles)
    oa, ob = oracle_embed(oracle, base, bw, bh, xy, rgb, bits, *KTH, radii, angles)
    assert np.array_equal(fa, oa) and np.array_equal(fb, ob)


@pytest.mark.parametrize("seed", [4, 5])
def test_oracle_decode_matches_reference(ref_codec, seed):
    rng = np.random.default_rng(seed)
    h, w, bw, bh = 30, 50, 7, 5
    xy = random_layout(rng, w, h, bw, bh, 16)
    rgb = rng.integers(0, 256, (len(xy), 3)).astype(np.int32)
    bits = rng.integers(1, 8, len(xy)).astype(np.int32)
    fa = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    fb = np.clip(fa.astype(int) + rng.integers(-40, 41, fa.shape), 0, 255).astype(np.uint8)
    for th in ((50.0, 0.5), (100.0, 0.25), (7.0, 1.0)):
        st, pat, md = ref_codec.decode(fa, fb, bw, bh, xy, rgb, bits, *th)
        got = CO.classify(CO.block_sums(fa, fb, bw, bh, xy), bw, bh, rgb, *th)
        assert [g[0] for g in got] == st.tolist()
        assert [g[1] for g in got] == pat.tolist()
        assert np.array_equal(np.array([g[2] for g in got]), md)  # bit-exact doubles


def _layout(cv, bw, bh, specs):
    L = cv.BlockLayout()
    L.block_width, L.block_height = bw, bh
    L.blocks = [cv.BlockSpec(x, y, name, cv.SrgbColor(*rgb), cv.BitPattern(p)) for x, y, name, rgb, p in specs]
    return L


SPECS = [(2, 3, "gray", (170, 170, 170), "110"), (20, 3, "blue", (100, 100, 240), "001"),
         (40, 9, "we\"ird\\name\té", (0, 255, 7), "111")]


def test_layout_json_matches_reference_text(cv, ref_codec):
    for th in ((50.0, 0.5), (100.0, 0.25), (0.1, 1e-05), (123456789012345680.0, 0.3333333333333333)):
        L = _layout(cv, 12, 10, SPECS)
        ours = cv.layout_to_json(L, cv.Thresholds(*th))
        ref = ref_codec.layout_json(12, 10, [s[:2] for s in SPECS], [s[3] for s in SPECS],
                                    [W.bits(s[4]) for s in SPECS], [s[2] for s in SPECS], *th)
        assert ours == ref


def test_report_json_matches_reference_text(cv, ref_codec):
    L = _layout(cv, 12, 10, SPECS)
    fp = cv.FramePair()
    fp.layout = L
    st = [0, 1, 2]
    pat = [6, 0, 0]
    md = np.array([[116.0, 4.0, 120.0], [0.0, 12.333333333333334, 1e-7], [70.0, 1e20, 0.5]])
    ref = ref_codec.report_json(12, 10, [s[:2] for s in SPECS], [s[3] for s in SPECS],
                                [W.bits(s[4]) for s in SPECS], [s[2] for s in SPECS], 50.0, 0.5, st, pat, md)
    assert '"embedded_pattern": "110"' in ref
    ours_results = _results(cv, st, pat, md)
    assert cv.decode_report_json(L, cv.Thresholds(50.0, 0.5), ours_results) == ref


def _results(cv, st, pat, md):
    status = [cv.BlockStatus.PATTERN, cv.BlockStatus.NO_SIGNAL, cv.BlockStatus.AMBIGUOUS]
    pattern = lambda b: cv.BitPattern(format(b, "03b")) if b else cv.BitPattern("001")  # noqa: E731
    out = []
    for s, p, d in zip(st, pat, md):
        r = cv.BlockResult(status[s], pattern(p), [float(x) for x in d])
        if not p:  # a default (all-zero) pattern for non-Pattern results
            r = cv.BlockResult(status[s], cv.BlockResult().pattern, [float(x) for x in d])
        out.append(r)
    return out


def test_layout_from_json_round_trip_and_errors(cv):
    L = _layout(cv, 12, 10, SPECS[:2])
    th = cv.Thresholds(50.0, 0.5)
    text = cv.layout_to_json(L, th)
    sc = cv.layout_from_json(text)
    assert sc.thresholds.v_th == 50.0 and sc.thresholds.r_novib == 0.5
    assert len(sc.layout.blocks) == 2 and sc.layout.block_width == 12
    assert sc.layout.blocks[0].color_name == "gray"
    assert sc.layout.blocks[0].color == cv.SrgbColor(170, 170, 170)
    assert sc.layout.blocks[0].pattern == cv.BitPattern("110")
    assert sc.layout.blocks[1].x == 20
    assert cv.layout_to_json(sc.layout, sc.thresholds) == text
    for bad in ('{"version": 3}', "nope", "[1, 2]", '{"version": 1}', '{"version": "1"}',
                '{"version": 1, "block_width": 1, "block_height": 1, "v_th": 5, "r_novib": 2, "blocks": []}',
                '{"version": 1, "block_width": 1, "block_height": 1, "v_th": 5, "r_novib": 0.5,'
                ' "blocks": [{"x": 0, "y": 0, "rgb": [1, 2], "pattern": "101"}]}',
                '{"version": 1, "block_width": 1, "block_height": 1, "v_th": 5, "r_novib": 0.5,'
                ' "blocks": [{"x": 0, "y": 0, "rgb": [1, 2, 3], "pattern": "000"}]}'):
        with pytest.raises(ValueError):
            cv.layout_from_json(bad)


def test_validation_messages_match_reference(cv, ref_codec):
    radii, angles = matrix_grid()
    base = np.full((64, 64, 3), 170, np.uint8)
    cases = [
        (16, 16, [(0, 0), (50, 0)]),    # out of bounds
        (16, 16, [(0, 0), (15, 0)]),    # overlap
        (0, 16, [(0, 0)]),              # degenerate
        (16, 16, [(0, 0), (30, 30), (20, 20), (40, 0)]),  # overlap not between neighbours in list order
    ]
    for bw, bh, xy in cases:
        rgb = [(170, 170, 170)] * len(xy)
        bits = [5] * len(xy)
        names = [f"b{i}" for i in range(len(xy))]
        with pytest.raises(ValueError) as ref_err:
            ref_codec.embed(base, bw, bh, xy, rgb, bits, *KTH, radii, angles, names=names)
        L = _layout(cv, bw, bh, [(x, y, nm, c, "101") for (x, y), nm, c in zip(xy, names, rgb)])
        with pytest.raises(ValueError) as our_err:
            L.validate(64, 64)
        assert str(our_err.value) == str(ref_err.value)
    for hz in (50.0, 24.0, 0.0):
        with pytest.raises(ValueError) as ref_err:
            ref_codec.embed(base, 16, 16, [(0, 0)], [(170, 170, 170)], [5], *KTH, radii, angles, refresh_hz=hz)
        with pytest.raises(ValueError) as our_err:
            cv.DisplayParams(hz).validate()
        assert str(our_err.value) == str(ref_err.value)
    cv.DisplayParams(60.0).validate()
    cv.DisplayParams(50.2).validate()
