"""The codec on the GPU: embed_blocks / decode_blocks /
make_testcard through the device passes, bit-exact against the reference's
own codec (oracle/_ref/libcolorvibe_ref_codec.so) and the NumPy oracle.

The first group restates the reference's tests/test_codec.cpp cases.
"""
import numpy as np
import pytest

from oracle import codec_oracle as CO
from paper_2507_22901_b200 import workloads as W

pytestmark = pytest.mark.gpu

KTH = (50.0, 0.5)


def grid(cv):
    g = cv.VibrationGrid()
    g.radii, g.angles = [list(a) for a in W.uniform_grid(1.0, 76.0, 15.0, 9.0, 359.0, 12.0)]
    return g


def layout(cv, bw, bh, specs):
    L = cv.BlockLayout()
    L.block_width, L.block_height = bw, bh
    L.blocks = [cv.BlockSpec(x, y, name, cv.SrgbColor(*rgb), cv.BitPattern(p)) for x, y, name, rgb, p in specs]
    return L


# ---- tests/test_codec.cpp restated ---------------------------------------------


def test_testcard_embeds_best_pair_and_decodes(cv, ctx):  # test_codec.cpp:67-92
    gray, pat, th = cv.SrgbColor(170, 170, 170), cv.BitPattern("101"), cv.Thresholds(*KTH)
    fp = cv.make_testcard(gray, pat, th, grid(cv), cv.DisplayParams(), 48, 32)
    assert fp.frame_a.width == 48 and fp.frame_a.height == 32
    pairs = cv.batch_search(gray, grid(cv), pat, th)
    best = cv.select_best(pairs, th)
    assert fp.frame_a.get(0, 0) == best.plus
    assert fp.frame_b.get(0, 0) == best.minus
    assert fp.frame_a.get(47, 31) == best.plus
    res = cv.decode_blocks(fp, th)
    assert len(res) == 1 and res[0].status == cv.BlockStatus.PATTERN and res[0].pattern == pat
    assert res[0].mean_deltas[0] > 50.0 and res[0].mean_deltas[1] <= 25.0 and res[0].mean_deltas[2] > 50.0


def test_identical_frames_decode_no_signal(cv, ctx):  # :94-107
    fp = cv.FramePair()
    fp.frame_a = cv.Image.solid(32, 32, cv.SrgbColor(170, 170, 170))
    fp.frame_b = cv.Image.solid(32, 32, cv.SrgbColor(170, 170, 170))
    fp.layout = layout(cv, 32, 32, [(0, 0, "x", (170, 170, 170), "101")])
    res = cv.decode_blocks(fp, cv.Thresholds(*KTH))
    assert res[0].status == cv.BlockStatus.NO_SIGNAL and res[0].mean_deltas[0] == 0.0


def test_dead_zone_decodes_ambiguous(cv, ctx):  # :109-125
    fp = cv.FramePair()
    fp.frame_a = cv.Image.solid(8, 8, cv.SrgbColor(240, 175, 170))
    fp.frame_b = cv.Image.solid(8, 8, cv.SrgbColor(100, 165, 170))
    fp.layout = layout(cv, 8, 8, [(0, 0, "x", (170, 170, 170), "100")])
    res = cv.decode_blocks(fp, cv.Thresholds(100.0, 0.25))
    assert res[0].status == cv.BlockStatus.AMBIGUOUS
    assert list(res[0].mean_deltas) == [70.0, 5.0, 0.0]


def test_embedding_is_local_to_blocks(cv, ctx):  # :127-158
    base = cv.Image.solid(64, 48, cv.SrgbColor(30, 60, 90))
    L = layout(cv, 16, 16, [(4, 4, "gray", (170, 170, 170), "101"), (40, 24, "white", (240, 240, 240), "001")])
    fp = cv.embed_blocks(base, L, cv.Thresholds(*KTH), grid(cv), cv.DisplayParams())
    a, b, base_px = fp.frame_a.pixels, fp.frame_b.pixels, base.pixels
    inside = np.zeros((48, 64), bool)
    inside[4:20, 4:20] = True
    inside[24:40, 40:56] = True
    assert np.array_equal(a[~inside], base_px[~inside]) and np.array_equal(b[~inside], base_px[~inside])
    assert (a[inside] != base_px[inside]).any()
    res = cv.decode_blocks(fp, cv.Thresholds(*KTH))
    assert [r.pattern for r in res] == [cv.BitPattern("101"), cv.BitPattern("001")]


def test_multi_block_round_trip(cv, ctx):  # :160-195
    th, g = cv.Thresholds(*KTH), grid(cv)
    specs, x, y = [], 0, 0
    for name, rgb in zip(W.TABLE1_NAMES, W.TABLE1):
        for p in W.PATTERNS:
            if not cv.batch_search(cv.SrgbColor(*map(int, rgb)), g, cv.BitPattern(p), th):
                continue
            specs.append((x, y, name, tuple(map(int, rgb)), p))
            x += 8
            if x + 8 > 160:
                x, y = 0, y + 8
    assert len(specs) >= 20 and y + 8 <= 80
    fp = cv.embed_blocks(cv.Image.solid(160, 80, cv.SrgbColor(128, 128, 128)), layout(cv, 8, 8, specs), th, g,
                         cv.DisplayParams())
    res = cv.decode_blocks(fp, th)
    assert all(r.status == cv.BlockStatus.PATTERN for r in res)
    assert [str(r.pattern) for r in res] == [s[4] for s in specs]


def test_infeasible_block_fails_loudly(cv, ctx):  # :197-208
    L = layout(cv, 8, 8, [(0, 0, "red", (240, 100, 100), "100")])
    with pytest.raises(RuntimeError, match="no pair satisfies"):
        cv.embed_blocks(cv.Image.solid(16, 16, cv.SrgbColor(240, 100, 100)), L, cv.Thresholds(*KTH), grid(cv),
                        cv.DisplayParams())


def test_decode_validates_geometry(cv, ctx):  # :252-261
    fp = cv.FramePair()
    fp.frame_a = cv.Image.solid(16, 16, cv.SrgbColor(170, 170, 170))
    fp.frame_b = cv.Image.solid(16, 8, cv.SrgbColor(170, 170, 170))
    fp.layout = layout(cv, 8, 8, [(0, 0, "x", (170, 170, 170), "100")])
    with pytest.raises(ValueError, match="frame dimensions differ"):
        cv.decode_blocks(fp, cv.Thresholds(*KTH))


def test_decode_report(cv, ctx):  # :263-276
    th = cv.Thresholds(*KTH)
    fp = cv.make_testcard(cv.SrgbColor(170, 170, 170), cv.BitPattern("101"), th, grid(cv), cv.DisplayParams(), 16, 16)
    rep = cv.decode_report_json(fp.layout, th, cv.decode_blocks(fp, th))
    assert '"embedded_pattern": "101"' in rep and '"result": "pattern"' in rep and '"pattern": "101"' in rep
    with pytest.raises(ValueError):
        cv.decode_report_json(fp.layout, th, [])


# ---- bit-exact parity with the reference codec -----------------------------------


def random_layout(rng, w, h, bw, bh, n_max):
    taken = np.zeros((h, w), bool)
    xy = []
    for _ in range(n_max * 6):
        x, y = int(rng.integers(0, w - bw + 1)), int(rng.integers(0, h - bh + 1))
        if not taken[y:y + bh, x:x + bw].any():
            taken[y:y + bh, x:x + bw] = True
            xy.append((x, y))
        if len(xy) == n_max:
            break
    return xy


# feasible at (50, 0.5) on the matrix grid (pair counts 28, 10, 14, 10, 4, 8 by the oracle)
FEASIBLE = [((170, 170, 170), "101"), ((240, 240, 240), "001"), ((100, 100, 240), "110"),
            ((240, 100, 240), "101"), ((170, 170, 170), "111"), ((240, 240, 100), "100")]


@pytest.mark.parametrize("w,h,bw,bh,n,seed", [(64, 48, 8, 8, 12, 1), (61, 37, 5, 7, 10, 2), (130, 66, 13, 3, 40, 3),
                                               (33, 20, 33, 20, 1, 4), (256, 128, 1, 1, 300, 5),
                                               (100, 40, 9, 5, 20, 6), (96, 64, 2, 17, 30, 7)])
def test_embed_decode_match_reference(cv, ctx, ref_codec, w, h, bw, bh, n, seed):
    """Random base images and layouts: widths with 3W mod 16 / mod 12 != 0
    (the per-row geometry paths), unaligned block x, 1x1 and 2-pixel-wide
    blocks, a full-image block."""
    rng = np.random.default_rng(seed)
    base = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    xy = random_layout(rng, w, h, bw, bh, n)
    picks = [FEASIBLE[int(i)] for i in rng.integers(0, len(FEASIBLE), len(xy))]
    specs = [(x, y, f"b{i}", rgb, p) for i, ((x, y), (rgb, p)) in enumerate(zip(xy, picks))]
    th, g = cv.Thresholds(*KTH), grid(cv)
    fp = cv.embed_blocks(cv.Image.from_array(base), layout(cv, bw, bh, specs), th, g, cv.DisplayParams())
    rgb = [s[3] for s in specs]
    bits = [W.bits(s[4]) for s in specs]
    fa, fb = ref_codec.embed(base, bw, bh, xy, rgb, bits, *KTH, g.radii, g.angles)
    assert np.array_equal(fp.frame_a.pixels, fa) and np.array_equal(fp.frame_b.pixels, fb)
    # decode of noisy frames (not just the clean embed) against the reference
    na = np.clip(fa.astype(int) + rng.integers(-30, 31, fa.shape), 0, 255).astype(np.uint8)
    nb = np.clip(fb.astype(int) + rng.integers(-30, 31, fb.shape), 0, 255).astype(np.uint8)
    noisy = cv.FramePair()
    noisy.frame_a, noisy.frame_b, noisy.layout = cv.Image.from_array(na), cv.Image.from_array(nb), fp.layout
    for t in ((50.0, 0.5), (20.0, 0.25)):
        res = cv.decode_blocks(noisy, cv.Thresholds(*t))
        st, pat, md = ref_codec.decode(na, nb, bw, bh, xy, rgb, bits, *t)
        status = {cv.BlockStatus.PATTERN: 0, cv.BlockStatus.NO_SIGNAL: 1, cv.BlockStatus.AMBIGUOUS: 2}
        assert [status[r.status] for r in res] == st.tolist()
        assert [W.bits(str(r.pattern)) if str(r.pattern) != "000" else 0 for r in res] == pat.tolist()
        assert np.array_equal(np.array([list(r.mean_deltas) for r in res]).reshape(-1, 3), md)


def test_embed_frame_diff_matches_reference(cv, ctx, ref_codec):
    rng = np.random.default_rng(11)
    base = rng.integers(0, 256, (40, 40, 3)).astype(np.uint8)
    # feasible under FrameDiff at (50, 0.5) (oracle pair counts 26, 6, 14)
    specs = [(0, 0, "a", (170, 170, 170), "101"), (20, 0, "b", (240, 240, 240), "001"),
             (0, 20, "c", (240, 100, 100), "110")]
    opts = cv.SearchOptions()
    opts.delta_basis = cv.DeltaBasis.FRAME_DIFF
    g = grid(cv)
    fp = cv.embed_blocks_opts(cv.Image.from_array(base), layout(cv, 20, 20, specs), cv.Thresholds(*KTH), g,
                              cv.DisplayParams(), opts)
    fa, fb = ref_codec.embed(base, 20, 20, [s[:2] for s in specs], [s[3] for s in specs],
                             [W.bits(s[4]) for s in specs], *KTH, g.radii, g.angles, basis=1)
    assert np.array_equal(fp.frame_a.pixels, fa) and np.array_equal(fp.frame_b.pixels, fb)


def test_pattern_000_after_infeasible_block_reports_infeasible_first(cv, ctx, ref_codec):
    """The reference searches block by block (codec.cpp:78-87): an infeasible
    block before a "000" block raises the infeasible error."""
    g = grid(cv)
    base = np.full((16, 32, 3), 100, np.uint8)
    specs = [(0, 0, "red", (240, 100, 100), "100"), (16, 0, "z", (170, 170, 170), "000")]
    with pytest.raises(RuntimeError) as ours:
        cv.embed_blocks(cv.Image.from_array(base), _raw_layout(cv, specs), cv.Thresholds(*KTH), g,
                        cv.DisplayParams())
    with pytest.raises(RuntimeError) as ref:
        ref_codec.embed(base, 16, 16, [(0, 0), (16, 0)], [(240, 100, 100), (170, 170, 170)], [4, 0], *KTH, g.radii,
                        g.angles, names=["red", "z"])
    assert str(ours.value) == str(ref.value)


def _raw_layout(cv, specs):
    L = cv.BlockLayout()
    L.block_width = L.block_height = 16
    blocks = []
    for x, y, name, rgb, p in specs:
        b = cv.BlockSpec()
        b.x, b.y, b.color_name, b.color = x, y, name, cv.SrgbColor(*rgb)
        if p != "000":
            b.pattern = cv.BitPattern(p)
        blocks.append(b)
    L.blocks = blocks
    return L


# ---- device passes at full size ---------------------------------------------------


def test_device_passes_4k_many_blocks(cv, ctx):
    """3840x2160 frames resident in HBM (torch tensors), 16x16 blocks on a
    grid plus stragglers at unaligned x: paint and block sums through the
    C-ABI device mode against the NumPy oracle."""
    import torch

    rng = np.random.default_rng(21)
    h, w, bw, bh = 2160, 3840, 16, 16
    base = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    xy = [(x, y) for y in range(0, h - bh + 1, 64) for x in range(0, w - bw + 1, 48)]
    xy += [(3, 20), (23, 20), (2001, 2139)]  # unaligned x, between grid rows
    xy = np.array(xy, np.int32)
    plus = rng.integers(0, 256, (len(xy), 3)).astype(np.uint8)
    minus = rng.integers(0, 256, (len(xy), 3)).astype(np.uint8)
    d_base = torch.from_numpy(base).cuda()
    d_a, d_b = torch.empty_like(d_base), torch.empty_like(d_base)
    d_sums = torch.zeros((len(xy), 6), dtype=torch.int64, device="cuda")
    s = torch.cuda.current_stream()
    cv.paint_blocks_device(ctx, d_base.data_ptr(), d_a.data_ptr(), d_b.data_ptr(), w, h, bw, bh, xy, plus, minus,
                           s.cuda_stream)
    cv.block_sums_device(ctx, d_a.data_ptr(), d_b.data_ptr(), w, h, bw, bh, xy, d_sums.data_ptr(), s.cuda_stream)
    torch.cuda.synchronize()
    oa, ob = CO.paint(base, bw, bh, xy, plus, minus)
    assert torch.equal(d_a.cpu(), torch.from_numpy(oa)) and torch.equal(d_b.cpu(), torch.from_numpy(ob))
    assert np.array_equal(d_sums.cpu().numpy().astype(np.uint64), CO.block_sums(oa, ob, bw, bh, xy))


def test_host_passes_full_image_block(cv, ctx):
    rng = np.random.default_rng(22)
    base = rng.integers(0, 256, (1080, 1918, 3)).astype(np.uint8)  # width % 4 != 0: per-pixel kernel
    xy = np.array([[0, 0]], np.int32)
    a, b = cv.paint_blocks_host(ctx, base, 1918, 1080, xy, [[1, 2, 3]], [[250, 251, 252]])
    assert (a == [1, 2, 3]).all() and (b == [250, 251, 252]).all()
    sums = cv.block_sums_host(ctx, base, base[::-1].copy(), 1918, 1080, xy)
    assert np.array_equal(sums, CO.block_sums(base, base[::-1].copy(), 1918, 1080, xy))


def test_prepared_layout_repaints_and_sums(cv, ctx):
    """A prepared Layout reused with new colors, then the same colors again
    (the upload is skipped), and its block sums, against the NumPy oracle."""
    import torch

    rng = np.random.default_rng(23)
    h, w, bw, bh = 120, 200, 12, 7
    base = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    xy = np.array(random_layout(rng, w, h, bw, bh, 40), np.int32)
    lay = cv.Layout(ctx, w, h, bw, bh, xy)
    d_base = torch.from_numpy(base).cuda()
    d_a, d_b = torch.empty_like(d_base), torch.empty_like(d_base)
    d_sums = torch.zeros((len(xy), 6), dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    for colors_seed in (1, 2, 2, 3):
        crng = np.random.default_rng(colors_seed)
        plus = crng.integers(0, 256, (len(xy), 3)).astype(np.uint8)
        minus = crng.integers(0, 256, (len(xy), 3)).astype(np.uint8)
        lay.paint_device(d_base.data_ptr(), d_a.data_ptr(), d_b.data_ptr(), plus, minus, st)
        lay.block_sums_device(d_a.data_ptr(), d_b.data_ptr(), d_sums.data_ptr(), st)
        torch.cuda.synchronize()
        oa, ob = CO.paint(base, bw, bh, xy, plus, minus)
        assert np.array_equal(d_a.cpu().numpy(), oa) and np.array_equal(d_b.cpu().numpy(), ob)
        assert np.array_equal(d_sums.cpu().numpy().astype(np.uint64), CO.block_sums(oa, ob, bw, bh, xy))
