"""The five BASELINE.json workloads as explicit, seeded arrays.

Grids are built once, in double, left to right as SURVEY.md §8(d) pins them:
radii[k] = k * dr, angles[m] = (2.0 * pi * m) / N -- and fed identically to
the GPU path and to the CPU oracle.  The reference measures on synthetic
inputs only (no public dataset); these generators are the stand-ins.

Pattern bits are r<<2 | g<<1 | b ("101" == 5).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

# Table-1 colors in reference order (feasibility.cpp:18-24).
TABLE1_NAMES = ["Black", "Gray", "White", "Red", "Green", "Blue", "Yellow", "Cyan", "Magenta"]
TABLE1 = np.array(
    [[100, 100, 100], [170, 170, 170], [240, 240, 240], [240, 100, 100], [100, 240, 100],
     [100, 100, 240], [240, 240, 100], [100, 240, 240], [240, 100, 240]], dtype=np.int32)
# Pattern order of the reference sweep (feasibility.cpp:25-27).
PATTERNS = ["100", "010", "001", "110", "101", "011", "111"]
V_TH = [50.0, 100.0, 150.0, 200.0]
R_NOVIB = [0.5, 0.25, 0.125]


def bits(p: str) -> int:
    return (p[0] == "1") << 2 | (p[1] == "1") << 1 | (p[2] == "1")


def uniform_grid(r0: float, r1: float, rs: float, a0: float, a1: float, as_: float):
    """VibrationGrid::uniform (reference search.cpp:58-90): inclusive ranges,
    angles given in degrees, converted with deg * (pi / 180)."""
    rr, aa = [], []
    k = 0
    while r0 + k * rs <= r1 + 1e-9:
        rr.append(r0 + k * rs)
        k += 1
    k = 0
    d2r = math.pi / 180.0
    while a0 + k * as_ <= a1 + 1e-9:
        aa.append((a0 + k * as_) * d2r)
        k += 1
    return np.array(rr, np.float64), np.array(aa, np.float64)


def radii(n: int, dr: float) -> np.ndarray:
    return np.array([k * dr for k in range(n)], dtype=np.float64)


def angles(n: int) -> np.ndarray:
    return np.array([(2.0 * math.pi * m) / n for m in range(n)], dtype=np.float64)


@dataclass
class Workload:
    name: str
    targets: np.ndarray   # (n, 3) int32
    patterns: np.ndarray  # (n,) int32
    v_th: np.ndarray      # (n,) f64
    r_novib: np.ndarray   # (n,) f64
    radii: np.ndarray
    angles: np.ndarray
    output: str = "pairs"
    note: str = ""

    @property
    def n_searches(self) -> int:
        return len(self.patterns)

    @property
    def candidates(self) -> int:
        return self.n_searches * len(self.radii) * len(self.angles)

    def shard(self, rank: int, world: int) -> "Workload":
        """Contiguous search range for `rank`."""
        n = self.n_searches
        lo, hi = n * rank // world, n * (rank + 1) // world
        return Workload(self.name, self.targets[lo:hi], self.patterns[lo:hi], self.v_th[lo:hi],
                        self.r_novib[lo:hi], self.radii, self.angles, self.output, self.note)


def cfg0() -> Workload:
    """Single Gray target, 111, V_th 100, R 0.25, 256 x 1024."""
    return Workload("cfg0", TABLE1[1:2].copy(), np.array([7], np.int32), np.array([100.0]),
                    np.array([0.25]), radii(256, 0.5), angles(1024))


def cfg1() -> Workload:
    """756-search sweep on the cfg0 grid (feasibility.cpp:261-292 loop order)."""
    t, p, v, r = [], [], [], []
    for ci in range(9):
        for pat in PATTERNS:
            for vt in V_TH:
                for rn in R_NOVIB:
                    t.append(TABLE1[ci]); p.append(bits(pat)); v.append(vt); r.append(rn)
    return Workload("cfg1", np.array(t, np.int32), np.array(p, np.int32), np.array(v), np.array(r),
                    radii(256, 0.5), angles(1024))


def cfg2(n_radii: int = 4096, n_angles: int = 65536) -> Workload:
    """Fine grid, 9 targets, 111, V_th 50, R 0.5; r = k * 128/4096."""
    n = 9
    return Workload("cfg2", TABLE1.copy(), np.full(n, 7, np.int32), np.full(n, 50.0), np.full(n, 0.5),
                    radii(n_radii, 128.0 / 4096), angles(n_angles))


def cfg3() -> Workload:
    """4096 lattice targets (8+16i, 8+16j, 8+16k), i outer; pattern per target
    drawn from the 7 codes with numpy.random.default_rng(0) (BASELINE leaves
    the generator open; SURVEY.md §8(d) pins this one)."""
    lat = 8 + 16 * np.arange(16)
    t = np.array([[a, b, c] for a in lat for b in lat for c in lat], np.int32)
    codes = np.array([bits(p) for p in PATTERNS], np.int32)
    pat = codes[np.random.default_rng(0).integers(0, 7, len(t))]
    return Workload("cfg3", t, pat.astype(np.int32), np.full(len(t), 100.0), np.full(len(t), 0.25),
                    radii(256, 0.5), angles(1024), note="patterns: numpy default_rng(0).integers(0,7,4096)")


def voronoi_image(width: int = 3840, height: int = 2160, seeds: int = 64, seed: int = 0) -> np.ndarray:
    """cfg4 image: 64 Voronoi cells (nearest seed, ties -> lowest index), cell
    color uniform in [60, 250]^3, per-pixel per-channel integer noise in
    [-3, 3]; numpy default_rng(seed).  Returns (height, width, 3) uint8."""
    rng = np.random.default_rng(seed)
    sx = rng.integers(0, width, seeds)
    sy = rng.integers(0, height, seeds)
    colors = rng.integers(60, 251, (seeds, 3))
    yy, xx = np.mgrid[0:height, 0:width]
    best = np.zeros((height, width), np.int64)
    bestd = np.full((height, width), np.iinfo(np.int64).max, np.int64)
    for i in range(seeds):
        d = (xx - sx[i]).astype(np.int64) ** 2 + (yy - sy[i]).astype(np.int64) ** 2
        closer = d < bestd
        best[closer] = i
        bestd[closer] = d[closer]
    img = colors[best] + rng.integers(-3, 4, (height, width, 3))
    return np.clip(img, 0, 255).astype(np.uint8)


def cfg4(width: int = 3840, height: int = 2160) -> Workload:
    """Per-pixel batch: one search per pixel, output = count + first pair."""
    img = voronoi_image(width, height)
    t = img.reshape(-1, 3).astype(np.int32)
    n = len(t)
    return Workload("cfg4", t, np.full(n, 7, np.int32), np.full(n, 50.0), np.full(n, 0.5),
                    radii(64, 2.0), angles(256), output="first")


ALL = {"cfg0": cfg0, "cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4}
