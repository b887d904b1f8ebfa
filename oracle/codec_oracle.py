"""CPU restatement of the reference codec passes -- TEST INFRASTRUCTURE ONLY.

NumPy restatement of src/codec.cpp (the reference's `colorvibe` codec):

* ``paint``       -- embed_blocks' painting (codec.cpp:58-64, 89-96): both
                     frames start as copies of the base, then every block is
                     filled with its pair's plus (frame a) / minus (frame b).
* ``block_sums``  -- decode_blocks' per-block channel sums (codec.cpp:124-137),
                     as exact integers (the reference's double running sums of
                     8-bit values are exact below 2^53).
* ``classify``    -- decode_blocks' per-block classification (codec.cpp:138-163)
                     in IEEE double, the same operations in the same order.
* ``select_best`` -- search.cpp:458-489 on packed records (first maximum margin
                     in canonical order).

Pinned against the reference's own codec (oracle/_ref/libcolorvibe_ref_codec.so,
``oracle.oracle.RefCodec``) by tests/test_codec_oracle.py.
"""
from __future__ import annotations

import numpy as np

PATTERN = 0
NO_SIGNAL = 1
AMBIGUOUS = 2


def paint(base: np.ndarray, bw: int, bh: int, xy, plus, minus):
    """(frame_a, frame_b) for an (H, W, 3) uint8 base (codec.cpp:58-64)."""
    fa = base.copy()
    fb = base.copy()
    for (x, y), p, m in zip(np.asarray(xy).reshape(-1, 2), np.asarray(plus).reshape(-1, 3),
                            np.asarray(minus).reshape(-1, 3)):
        fa[y:y + bh, x:x + bw] = p
        fb[y:y + bh, x:x + bw] = m
    return fa, fb


def block_sums(fa: np.ndarray, fb: np.ndarray, bw: int, bh: int, xy) -> np.ndarray:
    """(n, 6) uint64: per block (a.r, a.g, a.b, b.r, b.g, b.b) (codec.cpp:124-137)."""
    xy = np.asarray(xy).reshape(-1, 2)
    out = np.zeros((len(xy), 6), np.uint64)
    for i, (x, y) in enumerate(xy):
        out[i, :3] = fa[y:y + bh, x:x + bw].reshape(-1, 3).sum(axis=0, dtype=np.uint64)
        out[i, 3:] = fb[y:y + bh, x:x + bw].reshape(-1, 3).sum(axis=0, dtype=np.uint64)
    return out


def classify(sums: np.ndarray, bw: int, bh: int, targets, v_th: float, r_novib: float):
    """[(status, pattern_bits, (d_r, d_g, d_b))] per block (codec.cpp:138-163)."""
    low = v_th * r_novib
    n = float(bw) * float(bh)
    out = []
    for s, t in zip(np.asarray(sums, np.uint64).reshape(-1, 6), np.asarray(targets).reshape(-1, 3)):
        devs, bits, ambiguous, any_high = [], 0, False, False
        for c in range(3):
            sa, sb = float(int(s[c])), float(int(s[3 + c]))
            dev = max(abs(sa / n - int(t[c])), abs(sb / n - int(t[c])))
            devs.append(dev)
            if dev > v_th:
                bits |= 4 >> c
                any_high = True
            elif not dev <= low:
                ambiguous = True
        if ambiguous:
            out.append((AMBIGUOUS, 0, tuple(devs)))
        elif not any_high:
            out.append((NO_SIGNAL, 0, tuple(devs)))
        else:
            out.append((PATTERN, bits, tuple(devs)))
    return out


def margins(codes: np.ndarray, target, v_th: float, r_novib: float, basis: int = 0) -> np.ndarray:
    """classification_margin (search.cpp:458-466) of packed records."""
    p = codes[:, :3].astype(np.int64)
    m = codes[:, 3:].astype(np.int64)
    t = np.asarray(target, np.int64)
    d = (np.maximum(np.abs(p - t), np.abs(m - t)) if basis == 0 else np.abs(p - m)).astype(np.float64)
    low = v_th * r_novib
    per = np.where(d > v_th, d - v_th, low - d)
    return per.min(axis=1)


def select_best(codes: np.ndarray, target, v_th: float, r_novib: float, basis: int = 0) -> int:
    """Index of the first maximum margin (search.cpp:468-489 in canonical order)."""
    return int(np.argmax(margins(codes, target, v_th, r_novib, basis)))
