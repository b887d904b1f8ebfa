"""Batched consumers of the search.

* `feasibility_matrix` -- the reference's Table-1 sweep
  (src/feasibility.cpp:261-292): one cell per (color, pattern, v_th,
  r_novib), color-major, with feasible / pair_count / best pair.  Here every
  cell is a search of ONE batched device launch (the reference spawns and
  joins threads for each of the 756 cells); `select_best`
  (src/search.cpp:458-489) runs vectorized over the packed records.
* `aggregate_any` / `export_aggregated_csv` -- feasibility.cpp:294-306 and
  the aggregated CSV form (byte-identical to the reference's
  tests/golden/matrix_aggregated.csv for SearchConfig::defaults()).
* `pairs_array` -- zero-copy-friendly NumPy structured records for a search
  (the ColorPair fields, search.hpp:70-79) instead of a Python list of
  objects.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import workloads as W

PAIR_DTYPE = np.dtype([("target", "i4", 3), ("plus", "i4", 3), ("minus", "i4", 3), ("radius", "f8"),
                       ("angle", "f8"), ("deltas", "f8", 3)])


@dataclass
class SearchConfig:
    """SearchConfig::defaults() (feasibility.cpp:16-36) as plain arrays."""
    names: list
    colors: np.ndarray      # (nc, 3) int32
    patterns: list          # pattern strings in sweep order
    v_th_values: list
    r_novib_values: list
    radii: np.ndarray
    angles: np.ndarray
    delta_basis: int = 0

    @staticmethod
    def defaults() -> "SearchConfig":
        radii, angles = W.uniform_grid(1.0, 76.0, 15.0, 9.0, 359.0, 12.0)
        return SearchConfig(list(W.TABLE1_NAMES), W.TABLE1.copy(), list(W.PATTERNS), list(W.V_TH), list(W.R_NOVIB),
                            radii, angles)

    @staticmethod
    def benchmark_defaults() -> "SearchConfig":
        """feasibility.cpp:38-44: the dense VibrationGrid::standard() grid."""
        cfg = SearchConfig.defaults()
        cfg.radii, cfg.angles = W.uniform_grid(1.0, 100.0, 1.0, 0.0, 359.0, 1.0)
        return cfg

    def cells(self):
        """(color, pattern, v_th, r_novib) indices in reference loop order."""
        for ci in range(len(self.colors)):
            for pi in range(len(self.patterns)):
                for vi in range(len(self.v_th_values)):
                    for ri in range(len(self.r_novib_values)):
                        yield ci, pi, vi, ri


def deltas_from_codes(targets: np.ndarray, codes: np.ndarray, basis: int) -> np.ndarray:
    """channel_deltas / frame_deltas (search.cpp:125-144) on packed codes."""
    p = codes[:, :3].astype(np.int32)
    m = codes[:, 3:].astype(np.int32)
    if basis == 0:
        return np.maximum(np.abs(p - targets), np.abs(m - targets)).astype(np.float64)
    return np.abs(p - m).astype(np.float64)


def margins(deltas: np.ndarray, v_th: float, r_novib: float) -> np.ndarray:
    """classification_margin (search.cpp:458-466), vectorized."""
    low = v_th * r_novib
    per = np.where(deltas > v_th, deltas - v_th, low - deltas)
    return per.min(axis=1)


def select_best_index(deltas: np.ndarray, v_th: float, r_novib: float) -> int:
    """select_best (search.cpp:468-489): max margin, ties to smaller radius then
    smaller angle == first maximum in canonical (radius, angle) order."""
    if len(deltas) == 0:
        raise ValueError("select_best: empty pair list")
    return int(np.argmax(margins(deltas, v_th, r_novib)))


def pairs_array(res: dict, s: int, target, radii, angles, basis: int = 0) -> np.ndarray:
    """Records of search s of a Context.search result as a structured array."""
    a, b = int(res["offsets"][s]), int(res["offsets"][s + 1])
    idx = np.asarray(res["idx"][a:b])
    codes = np.asarray(res["codes"][a:b])
    na = len(angles)
    out = np.zeros(b - a, PAIR_DTYPE)
    out["target"] = np.asarray(target, np.int32)
    out["plus"] = codes[:, :3]
    out["minus"] = codes[:, 3:]
    out["radius"] = np.asarray(radii)[idx // na]
    out["angle"] = np.asarray(angles)[idx % na]
    out["deltas"] = deltas_from_codes(np.asarray(target, np.int32), codes, basis)
    return out


@dataclass
class Cell:
    color_index: int
    pattern_index: int
    v_th_index: int
    r_novib_index: int
    feasible: bool
    pair_count: int
    best_pair: np.void | None  # PAIR_DTYPE record


def feasibility_matrix(cfg: SearchConfig, ctx=None) -> list:
    """All cells of the sweep in one device launch (feasibility.cpp:261-292)."""
    from . import Context

    ctx = ctx or Context(0)
    cells = list(cfg.cells())
    targets = np.array([cfg.colors[c] for c, _, _, _ in cells], np.int32)
    patterns = np.array([W.bits(cfg.patterns[p]) for _, p, _, _ in cells], np.int32)
    v_th = np.array([cfg.v_th_values[v] for _, _, v, _ in cells], np.float64)
    r_novib = np.array([cfg.r_novib_values[r] for _, _, _, r in cells], np.float64)
    res = ctx.search(targets, patterns, v_th, r_novib, cfg.radii, cfg.angles, delta_basis=cfg.delta_basis)
    out = []
    for s, (ci, pi, vi, ri) in enumerate(cells):
        n = int(res["counts"][s])
        best = None
        if n:
            recs = pairs_array(res, s, targets[s], cfg.radii, cfg.angles, cfg.delta_basis)
            best = recs[select_best_index(recs["deltas"], v_th[s], r_novib[s])]
        out.append(Cell(ci, pi, vi, ri, n > 0, n, best))
    return out


def aggregate_any(cfg: SearchConfig, cells: list) -> np.ndarray:
    """(patterns x colors) OR over the threshold grid (feasibility.cpp:294-306)."""
    agg = np.zeros((len(cfg.patterns), len(cfg.colors)), bool)
    for c in cells:
        agg[c.pattern_index, c.color_index] |= c.feasible
    return agg


def export_aggregated_csv(cfg: SearchConfig, cells: list) -> str:
    """export_matrix(m, Csv, aggregated=true) (feasibility.cpp:325-341)."""
    agg = aggregate_any(cfg, cells)
    lines = ["pattern," + ",".join(cfg.names)]
    for pi, p in enumerate(cfg.patterns):
        lines.append(p + "," + ",".join("1" if agg[pi, ci] else "0" for ci in range(len(cfg.colors))))
    return "\n".join(lines) + "\n"
