"""Pins the CPU oracle (oracle/cv_oracle.c) to the reference before trusting it.

Golden fixtures were produced by the reference itself (tests/golden/make_golden.py
over oracle/_ref, i.e. the reference's src/color.cpp + src/search.cpp).  When
the reference build is present the oracle is also compared to it directly.
"""
import os

import numpy as np
import pytest

from cvtest_util import golden, sha_records
from paper_2507_22901_b200 import workloads as W
from paper_2507_22901_b200.workloads import uniform_grid

pytestmark = []


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs])


def test_known_answer_constants(oracle):
    ka = golden("known_answers.json")
    assert np.array_equal(oracle.thresholds(), unhex(ka["thresholds"]))
    assert np.array_equal(oracle.xyz_to_rgb().ravel(), unhex(ka["xyz_to_rgb"]))
    assert np.array_equal(oracle.white(), unhex(ka["white"]))
    assert oracle.white()[1] == 1.0  # test_color.cpp:103-109
    # SURVEY §8(c) spot values
    assert oracle.thresholds()[1] == 0.00015176349177441873
    assert oracle.thresholds()[255] == 0.99554524972107783
    for key, lab in ka["lab"].items():
        rgb = [int(v) for v in key.split(",")]
        assert np.array_equal(oracle.srgb_to_lab(rgb), unhex(lab)), key


def test_code_probes_around_every_threshold(oracle):
    for xh, code, q in golden("known_answers.json")["code_probes"]:
        x = float.fromhex(xh)
        assert oracle.table_code(x) == code
        assert oracle.quantize(x) == q == code


def test_table_code_equals_pow_quantizer_random(oracle):
    rng = np.random.default_rng(3)
    for x in rng.uniform(-0.1, 1.1, 20000):
        assert oracle.table_code(x) == oracle.quantize(x)


@pytest.mark.parametrize("method", [0, 1])
def test_small_grid_cases_match_reference_golden(oracle, method):
    radii, angles = uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    for case in golden("small_cases.json"):
        idx, codes, _ = oracle.search(case["target"], W.bits(case["pattern"]), case["v_th"], case["r_novib"],
                                      radii, angles, delta_basis=case["basis"], method=method)
        assert len(idx) == case["count"], case
        assert sha_records(idx, codes) == case["sha256"], case


def test_cfg0_matches_reference_golden(oracle):
    wl = W.cfg0()
    idx, codes, _ = oracle.search(wl.targets[0], 7, 100.0, 0.25, wl.radii, wl.angles, method=1, workers=4)
    g = golden("workloads.json")["cfg0"]
    assert len(idx) == g["total"] == 4802
    assert sha_records(idx, codes) == g["sha256"]
    # first pair at r = 105, plus (255,69,69), minus (0,209,255)
    assert wl.radii[idx[0] // 1024] == 105.0
    assert codes[0].tolist() == [255, 69, 69, 0, 209, 255]


def test_cfg1_counts_match_reference_golden(oracle):
    wl = W.cfg1()
    g = golden("workloads.json")["cfg1"]
    got = []
    for s in range(0, wl.n_searches, 37):  # a spread sample keeps the CPU suite fast
        idx, _, _ = oracle.search(wl.targets[s], int(wl.patterns[s]), wl.v_th[s], wl.r_novib[s], wl.radii,
                                  wl.angles, method=1, workers=4, want_deltas=False)
        got.append((s, len(idx)))
    for s, n in got:
        assert n == g["counts"][s], s
    assert g["total"] == 3785016


def test_aggregated_matrix_reproduces_golden_csv(oracle):
    radii, angles = uniform_grid(1.0, 76.0, 15.0, 9.0, 359.0, 12.0)
    lines = ["pattern," + ",".join(W.TABLE1_NAMES)]
    for p in W.PATTERNS:
        row = [p]
        for ci in range(9):
            feasible = any(
                len(oracle.search(W.TABLE1[ci], W.bits(p), vt, rn, radii, angles, method=1)[0]) > 0
                for vt in W.V_TH for rn in W.R_NOVIB)
            row.append("1" if feasible else "0")
        lines.append(",".join(row))
    assert "\n".join(lines) + "\n" == golden("matrix_aggregated.csv")


def test_serial_equals_batch_dark_target(oracle):
    # (8,8,8) exercises the linear branch of f^-1.
    radii = W.radii(64, 2.0)
    angles = W.angles(96)
    for p in (7, 5, 1):
        a = oracle.search([8, 8, 8], p, 50.0, 0.5, radii, angles, method=0)
        b = oracle.search([8, 8, 8], p, 50.0, 0.5, radii, angles, method=1, workers=3)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)


@pytest.mark.parametrize("mode,basis", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_oracle_equals_reference_all_modes(oracle, reference, mode, basis):
    radii, angles = uniform_grid(1.0, 91.0, 10.0, 0.0, 350.0, 10.0)
    for t in ([170, 170, 170], [100, 100, 240], [8, 8, 8], [255, 0, 0]):
        for p in (1, 5, 6, 7):
            for method in (0, 1):
                a = oracle.search(t, p, 50.0, 0.5, radii, angles, delta_mode=mode, delta_basis=basis,
                                  method=method)
                b = reference.search(t, p, 50.0, 0.5, radii, angles, delta_mode=mode, delta_basis=basis,
                                     method=method, workers=2)
                for x, y in zip(a, b):
                    assert np.array_equal(x, y)


def test_oracle_equals_reference_custom_white(oracle, reference):
    radii, angles = W.radii(40, 2.5), W.angles(64)
    wp = [0.9642, 1.0, 0.8251]
    a = oracle.search([120, 60, 200], 5, 50.0, 0.5, radii, angles, white=wp)
    b = reference.search([120, 60, 200], 5, 50.0, 0.5, radii, angles, white=wp, workers=1)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


_BIND_CHECK = r"""
import ctypes, ctypes.util, os, sys
sys.path.insert(0, {root!r})
# the product library first, GLOBAL: it exports the same mangled
# colorvibe::batch_search as the reference checker
ctypes.CDLL({gpu!r}, mode=ctypes.RTLD_GLOBAL)
from oracle.oracle import Reference
ref = Reference()

class Dl_info(ctypes.Structure):
    _fields_ = [("dli_fname", ctypes.c_char_p), ("dli_fbase", ctypes.c_void_p),
                ("dli_sname", ctypes.c_char_p), ("dli_saddr", ctypes.c_void_p)]

libdl = ctypes.CDLL(ctypes.util.find_library("dl") or "libc.so.6")
info = Dl_info()
assert libdl.dladdr(ctypes.c_void_p(ref.batch_search_addr()), ctypes.byref(info))
print(os.path.realpath(info.dli_fname.decode()), os.path.realpath(ref.path))
"""


def test_reference_binds_its_own_search():
    """The reference checker must run the REFERENCE's batch_search even when
    libcolorvibe_gpu.so, which exports the identical C++ symbol, was loaded
    first with RTLD_GLOBAL (-Bsymbolic link, oracle/Makefile): otherwise the
    parity tests could compare the product with itself."""
    import subprocess
    import sys

    from cvtest_util import ROOT

    gpu = os.path.join(ROOT, "paper_2507_22901_b200", "libcolorvibe_gpu.so")
    ref_dir = os.path.join(ROOT, "oracle", "_ref")
    if not os.path.exists(gpu) or not os.path.isdir(ref_dir):
        pytest.skip("libraries not built")
    out = subprocess.run([sys.executable, "-c", _BIND_CHECK.format(root=ROOT, gpu=gpu)], capture_output=True,
                         text=True, check=True).stdout.split()
    assert out[0] == out[1] and "/oracle/_ref/" in out[0], out


def test_reference_memo_matches_crop_golden(reference):
    """bench.py's cfg4 CPU baseline (memoized by color)
    against the reference-generated 256x144 per-pixel golden."""
    import hashlib

    from cvtest_util import golden
    from paper_2507_22901_b200 import workloads as W

    g = golden("workloads.json")["cfg4_256x144"]
    wl = W.cfg4(g["width"], g["height"])
    counts, first, codes, nu = reference.search_memo(wl.targets, 7, 50.0, 0.5, wl.radii, wl.angles, threads=4)
    assert nu == g["unique_colors"]
    m = hashlib.sha256()
    m.update(counts.tobytes()); m.update(first.tobytes()); m.update(codes.tobytes())
    assert int(counts.sum()) == g["total"] and m.hexdigest() == g["sha256"]
