"""Generates the golden fixtures in tests/golden/ from the REFERENCE ITSELF.

Every value here comes from oracle/_ref/libcolorvibe_ref_*.so -- the
reference's own src/color.cpp + src/search.cpp compiled where they lie under
/root/reference by oracle/Makefile -- through oracle/ref_shim.cpp.  Run in the
build container (where /root/reference exists):

    python tests/golden/make_golden.py            # everything but cfg2
    python tests/golden/make_golden.py --cfg2     # + cfg2 per-target counts and record sha256 (minutes)
    python tests/golden/make_golden.py --cfg4     # + full-size cfg4 per-pixel count/first hash

Outputs (all small, committed):
  known_answers.json    thresholds, kXyzToRgb, d65 white, target Lab, code probes
  small_cases.json      reference test_search.cpp grid cases: count + sha256 per case
  workloads.json        cfg0 / cfg1 / cfg3 per-search counts + record sha256,
                        cfg2 per-target counts + 10-byte-record sha256, cfg4 (256x144 crop) count/first sha256
  matrix_aggregated.csv feasibility aggregate over SearchConfig::defaults()
                        (same bytes as the reference's tests/golden file)
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Reference  # noqa: E402
from paper_2507_22901_b200 import workloads as W  # noqa: E402
from paper_2507_22901_b200.workloads import uniform_grid  # noqa: E402


def h(x: float) -> str:
    return float(x).hex()


def records_sha(idx: np.ndarray, codes: np.ndarray) -> str:
    m = hashlib.sha256()
    m.update(np.ascontiguousarray(idx, np.uint32).tobytes())
    m.update(np.ascontiguousarray(codes, np.uint8).tobytes())
    return m.hexdigest()


SMALL_TARGETS = [[170, 170, 170], [240, 240, 240], [100, 100, 240], [240, 100, 240]]
SMALL_PATTERNS = ["100", "001", "101", "110", "111"]
SMALL_TH = [(50.0, 0.5), (100.0, 0.25), (150.0, 0.125)]


def known_answers(ref: Reference) -> dict:
    labs = {}
    probes = [[0, 0, 0], [255, 255, 255], [8, 8, 8], [1, 2, 3], [254, 0, 128]] + W.TABLE1.tolist()
    for t in probes:
        labs[",".join(map(str, t))] = [h(v) for v in ref.srgb_to_lab(t)]
    thr = ref.thresholds()
    code_probes = []
    for c in range(1, 256, 7):
        x = thr[c]
        for y in (np.nextafter(x, -1.0), x, np.nextafter(x, 2.0)):
            code_probes.append([h(y), ref.table_code(y), ref.quantize(y)])
    return {
        "thresholds": [h(v) for v in thr],
        "xyz_to_rgb": [h(v) for v in ref.xyz_to_rgb().ravel()],
        "white": [h(v) for v in ref.white()],
        "lab": labs,
        "code_probes": code_probes,
    }


def small_cases(ref: Reference) -> list:
    radii, angles = uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    out = []
    for t in SMALL_TARGETS:
        for p in SMALL_PATTERNS:
            for vt, rn in SMALL_TH:
                for basis in (0, 1):
                    idx, codes, _ = ref.search(t, W.bits(p), vt, rn, radii, angles, delta_basis=basis,
                                               method=0)
                    out.append({"target": t, "pattern": p, "v_th": vt, "r_novib": rn, "basis": basis,
                                "count": int(len(idx)), "sha256": records_sha(idx, codes)})
    return out


def workload_records(ref: Reference, wl: W.Workload, workers: int) -> dict:
    counts, shas = [], hashlib.sha256()
    for s in range(wl.n_searches):
        idx, codes, _ = ref.search(wl.targets[s], int(wl.patterns[s]), wl.v_th[s], wl.r_novib[s], wl.radii,
                                   wl.angles, method=1, workers=workers, want_deltas=False)
        counts.append(int(len(idx)))
        shas.update(np.ascontiguousarray(idx, np.uint32).tobytes())
        shas.update(np.ascontiguousarray(codes, np.uint8).tobytes())
    return {"counts": counts, "total": int(sum(counts)), "sha256": shas.hexdigest()}


def records10_sha_update(m, idx: np.ndarray, codes: np.ndarray) -> None:
    """Feeds records in the 10-byte wire layout (u32 LE idx, then the 6 code
    bytes) to hash m -- streamable, so cfg2's 444M pairs hash row chunk by
    row chunk."""
    rec = np.empty((len(idx), 10), np.uint8)
    rec[:, :4] = np.ascontiguousarray(idx, "<u4").view(np.uint8).reshape(-1, 4)
    rec[:, 4:] = codes
    m.update(rec.tobytes())


def cfg2_records(ref: Reference, workers: int, chunk: int = 256) -> dict:
    """cfg2 per-target counts and per-target record sha256 (10-byte layout),
    from the reference batch_search run on row chunks [k_lo, k_lo+chunk) of
    the grid: rows are independent (search.cpp:230-278) and a search's list
    is the concatenation of its row slices in row order (search.cpp:433-455),
    so idx = (k_lo + k) * na + m of the chunk's record k * na + m."""
    wl = W.cfg2()
    na = len(wl.angles)
    counts, shas = [], []
    for s in range(wl.n_searches):
        m, n = hashlib.sha256(), 0
        for k_lo in range(0, len(wl.radii), chunk):
            idx, codes, _ = ref.search(wl.targets[s], int(wl.patterns[s]), wl.v_th[s], wl.r_novib[s],
                                       wl.radii[k_lo:k_lo + chunk], wl.angles, method=1, workers=workers,
                                       want_deltas=False)
            records10_sha_update(m, idx.astype(np.uint64) + np.uint64(k_lo * na), codes)
            n += len(idx)
        counts.append(n)
        shas.append(m.hexdigest())
        print(f"cfg2 target {s}: {n} pairs", flush=True)
    return {"counts": counts, "total": int(sum(counts)), "sha256_records10": shas,
            "layout": "per target: sha256 over 10-byte records (u32 LE idx = k*na+m, plus rgb, minus rgb) "
                      "in canonical order; reference batch_search on 256-row chunks"}


def cfg4_small(ref: Reference, width=256, height=144) -> dict:
    """cfg4 pipeline (same generator, any size): per-pixel count and first
    canonical pair, memoized by color (results depend only on it)."""
    img = W.voronoi_image(width, height)
    wl = W.cfg4(width, height)
    flat = img.reshape(-1, 3).astype(np.int32)
    uniq, inv = np.unique(flat, axis=0, return_inverse=True)
    cnt = np.zeros(len(uniq), np.uint64)
    first = np.full(len(uniq), 0xFFFFFFFF, np.uint32)
    fcodes = np.zeros((len(uniq), 6), np.uint8)
    for u, t in enumerate(uniq):
        idx, codes, _ = ref.search(t, 7, 50.0, 0.5, wl.radii, wl.angles, method=1, workers=1,
                                   want_deltas=False)
        cnt[u] = len(idx)
        if len(idx):
            first[u] = idx[0]
            fcodes[u] = codes[0]
    inv = inv.ravel()
    m = hashlib.sha256()
    m.update(cnt[inv].tobytes()); m.update(first[inv].tobytes()); m.update(fcodes[inv].tobytes())
    return {"width": width, "height": height, "unique_colors": int(len(uniq)),
            "total": int(cnt[inv].sum()), "sha256": m.hexdigest()}


def aggregated_matrix(ref: Reference) -> str:
    """feasibility_matrix(SearchConfig::defaults()) -> export_matrix(csv, aggregated)
    (feasibility.cpp:16-36, 261-306, 349-363) restated over the reference search."""
    radii, angles = uniform_grid(1.0, 76.0, 15.0, 9.0, 359.0, 12.0)
    lines = ["pattern," + ",".join(W.TABLE1_NAMES)]
    for p in W.PATTERNS:
        row = [p]
        for ci in range(9):
            any_ = 0
            for vt in W.V_TH:
                for rn in W.R_NOVIB:
                    idx, _, _ = ref.search(W.TABLE1[ci], W.bits(p), vt, rn, radii, angles, method=1,
                                           workers=1, want_deltas=False)
                    any_ |= len(idx) > 0
            row.append("1" if any_ else "0")
        lines.append(",".join(row))
    return "\n".join(lines) + "\n"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cfg2", action="store_true")
    ap.add_argument("--cfg2-only", action="store_true", help="regenerate only the cfg2 entry")
    ap.add_argument("--cfg4", action="store_true", help="full 3840x2160 per-pixel config (memoized by color)")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    ref = Reference()
    t0 = time.time()
    with open(os.path.join(HERE, "known_answers.json"), "w") as f:
        json.dump(known_answers(ref), f, indent=1)
    with open(os.path.join(HERE, "small_cases.json"), "w") as f:
        json.dump(small_cases(ref), f, indent=1)
    with open(os.path.join(HERE, "matrix_aggregated.csv"), "w") as f:
        f.write(aggregated_matrix(ref))
    path = os.path.join(HERE, "workloads.json")
    wj = json.load(open(path)) if os.path.exists(path) else {}
    if args.cfg2_only:
        wj["cfg2"] = cfg2_records(ref, args.workers)
        with open(path, "w") as f:
            json.dump(wj, f, indent=1)
        print(f"cfg2 fixture written in {time.time() - t0:.1f}s")
        return
    wj["cfg0"] = workload_records(ref, W.cfg0(), args.workers)
    wj["cfg1"] = workload_records(ref, W.cfg1(), args.workers)
    wj["cfg3"] = workload_records(ref, W.cfg3(), args.workers)
    wj["cfg4_256x144"] = cfg4_small(ref)
    if args.cfg4:
        wj["cfg4"] = cfg4_small(ref, 3840, 2160)
    if args.cfg2:
        wj["cfg2"] = cfg2_records(ref, args.workers)
    with open(path, "w") as f:
        json.dump(wj, f, indent=1)
    print(f"golden fixtures written in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
