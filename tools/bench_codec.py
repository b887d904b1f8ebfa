"""Measurement of the codec passes, one JSON line.

Workload: a 3840x2160 RGB8 carrier (cfg4's image size) with a 64 x 36 grid of
32x32 blocks (2,304 blocks, 28% of the pixels), synthetic seeded data.

* ``paint``: cvg_paint_blocks on device-resident frames (CVG_MEM_DEVICE).
  Algorithmic bytes per launch = read base + write both frames = 9 B/pixel.
* ``sums``: cvg_block_sums on device-resident frames.  Algorithmic bytes =
  read both frames over the blocks = 6 B per block pixel.
* ``e2e``: embed_blocks + decode_blocks through the reference-shaped C++ API
  (host Images; one batched search for all blocks, H2D/D2H inside).
* ``cpu_baseline``: the reference's own codec (oracle/_ref) on the same
  layout, embed + decode, 1 thread per batch_search call as the reference runs.

Both device passes are HBM-bound: roofline peak = MEASURED_PEAKS.json hbm_gbs.
Timing: CUDA events on the launching stream, L2 (126 MB) flushed between
iterations with a 256 MiB write.
"""
from __future__ import annotations

import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.environ.get("CVG_PKG_ROOT") or ROOT)  # CVG_PKG_ROOT: A/B another build


def main():
    import torch

    import paper_2507_22901_b200 as cv
    from paper_2507_22901_b200 import workloads as W

    steps = int(os.environ.get("STEPS", "30"))
    h, w, bw, bh = 2160, 3840, 32, 32
    rng = np.random.default_rng(0)
    base = rng.integers(0, 256, (h, w, 3)).astype(np.uint8)
    xy = np.array([(x, y) for y in range(0, h - bh + 1, 60) for x in range(0, w - bw + 1, 60)], np.int32)
    n = len(xy)
    plus = rng.integers(0, 256, (n, 3)).astype(np.uint8)
    minus = rng.integers(0, 256, (n, 3)).astype(np.uint8)
    ctx = cv.Context(0)
    st = torch.cuda.current_stream()
    d_base = torch.from_numpy(base).cuda()
    d_a, d_b = torch.empty_like(d_base), torch.empty_like(d_base)
    d_sums = torch.zeros((n, 6), dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn):
        for _ in range(3):
            fn()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        for a, b in ev:
            flush.zero_()
            a.record(st)
            fn()
            b.record(st)
        torch.cuda.synchronize()
        return statistics.median(a.elapsed_time(b) for a, b in ev)

    # prepared layout (positions uploaded once): a paint = colors copy + copy and fill kernels
    lay = cv.Layout(ctx, w, h, bw, bh, xy)
    paint = lambda: lay.paint_device(d_base.data_ptr(), d_a.data_ptr(), d_b.data_ptr(), plus, minus,  # noqa
                                     st.cuda_stream)
    sums = lambda: lay.block_sums_device(d_a.data_ptr(), d_b.data_ptr(), d_sums.data_ptr(), st.cuda_stream)  # noqa
    paint_ms = timed(paint)
    sums_ms = timed(sums)
    # one-shot calls (span table rebuilt and uploaded every call)
    oneshot_ms = timed(lambda: cv.paint_blocks_device(ctx, d_base.data_ptr(), d_a.data_ptr(), d_b.data_ptr(), w, h,
                                                      bw, bh, xy, plus, minus, st.cuda_stream))
    paint_bytes = 9 * w * h
    sums_bytes = 6 * bw * bh * n
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]

    # e2e through the C++ API: feasible (color, pattern) blocks on the matrix grid
    feas = [((170, 170, 170), "101"), ((240, 240, 240), "001"), ((100, 100, 240), "110"),
            ((240, 100, 240), "101"), ((170, 170, 170), "111"), ((240, 240, 100), "100")]
    L = cv.BlockLayout()
    L.block_width, L.block_height = bw, bh
    picks = [feas[int(i)] for i in rng.integers(0, len(feas), n)]
    L.blocks = [cv.BlockSpec(int(x), int(y), f"b{i}", cv.SrgbColor(*c), cv.BitPattern(p))
                for i, ((x, y), (c, p)) in enumerate(zip(xy, picks))]
    g = cv.VibrationGrid()
    g.radii, g.angles = [list(a) for a in W.uniform_grid(1.0, 76.0, 15.0, 9.0, 359.0, 12.0)]
    th, disp, img = cv.Thresholds(50.0, 0.5), cv.DisplayParams(), cv.Image.from_array(base)
    cv.decode_blocks(cv.embed_blocks(img, L, th, g, disp), th)
    e2e = []
    for _ in range(max(3, steps // 3)):
        t0 = time.perf_counter()
        fp = cv.embed_blocks(img, L, th, g, disp)
        res = cv.decode_blocks(fp, th)
        e2e.append(time.perf_counter() - t0)
    assert all(r.status == cv.BlockStatus.PATTERN for r in res)
    e2e_s = statistics.median(e2e)

    cpu = None
    try:
        from oracle.oracle import RefCodec

        ref = RefCodec()
        rgb = [c for c, _ in picks]
        bits = [W.bits(p) for _, p in picks]
        t0 = time.perf_counter()
        fa, fb = ref.embed(base, bw, bh, xy, rgb, bits, 50.0, 0.5, g.radii, g.angles)
        ref.decode(fa, fb, bw, bh, xy, rgb, bits, 50.0, 0.5)
        cpu_s = time.perf_counter() - t0
        assert np.array_equal(fa, fp.frame_a.pixels) and np.array_equal(fb, fp.frame_b.pixels)
        cpu = {"value": round(3 * w * h / cpu_s / 1e9, 4), "unit": "GB/s (carrier bytes)", "cores": os.cpu_count(),
               "kind": "reference", "sample": "full workload, embed_blocks + decode_blocks, reference codec "
                                               "(oracle/_ref), batch_search workers=0 (all host threads)",
               "s_per_step": round(cpu_s, 4)}
    except FileNotFoundError:
        pass

    out = {
        "metric": "codec image-pass bandwidth", "unit": "GB/s", "n_gpus": 1, "steps": steps, "warmup": 3,
        "value": round(paint_bytes / (paint_ms * 1e-3) / 1e9, 1), "ms_per_step": round(paint_ms, 4),
        "higher_is_better": True, "dtype": "u8", "data": "synthetic (seeded)",
        "config": {"workload": "codec 3840x2160, 2304 blocks of 32x32", "l2": "flushed between steps (256 MiB write)"},
        "passes": {
            "paint": {"ms": round(paint_ms, 4), "algorithmic_bytes": paint_bytes,
                      "gbs": round(paint_bytes / (paint_ms * 1e-3) / 1e9, 1)},
            "block_sums": {"ms": round(sums_ms, 4), "algorithmic_bytes": sums_bytes,
                           "gbs": round(sums_bytes / (sums_ms * 1e-3) / 1e9, 1)},
            "paint_one_shot": {"ms": round(oneshot_ms, 4), "note": "cvg_paint_blocks: layout validated, span "
                                                                     "table built and uploaded inside the call"},
        },
        "gpu_launches": {"paint": 2, "block_sums": 1},
        "roofline": {"bound": "hbm", "achieved": round(paint_bytes / (paint_ms * 1e-3) / 1e9, 1), "peak": peak,
                     "unit": "GB/s", "frac": round(paint_bytes / (paint_ms * 1e-3) / 1e9 / peak, 4),
                     "kernel": "copy2_kernel + fill_kernel", "peak_source": "MEASURED_PEAKS.json hbm_gbs (copy, burst)"},
        "e2e": {"value": round(3 * w * h / e2e_s / 1e9, 4), "unit": "GB/s (carrier bytes)", "s_per_step": round(e2e_s, 5),
                "api": "embed_blocks + decode_blocks (C++ API, host Images)",
                "h2d_bytes_per_step": 3 * 3 * w * h, "d2h_bytes_per_step": 2 * 3 * w * h + 48 * n},
        "cpu_baseline": cpu,
    }
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
