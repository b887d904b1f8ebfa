"""C++ drop-in check.

The reference's own, unmodified callers of the hot path -- src/feasibility.cpp
(feasibility_matrix, feasibility.cpp:261-292), src/bench.cpp (run_benchmark,
bench.cpp:84-85, 104), src/codec.cpp (embed_blocks, codec.cpp:80-81) -- plus a
driver with the reference test_search.cpp:177-255 cases (oracle/dropin_main.cpp)
are compiled by oracle/Makefile twice:

  oracle/_ref/dropin_gpu  against include/ and linked to libcolorvibe_gpu.so
                          (batch_search / serial_search / select_best / the
                          color API resolved from the B200 library);
  oracle/_ref/dropin_ref  with the reference's own headers, color.cpp and
                          search.cpp (CPU).

Both must print the same report, line for line: pair-list hashes (80-byte
ColorPair records incl. radius, angle and deltas), the feasibility exports,
the benchmark pair total, codec frames and decode results, and the
reference's exception types and messages.
"""
import os
import subprocess

import pytest

from cvtest_util import ROOT

REF_DIR = os.path.join(ROOT, "oracle", "_ref")


def _binaries():
    gpu, ref = os.path.join(REF_DIR, "dropin_gpu"), os.path.join(REF_DIR, "dropin_ref")
    if not (os.path.exists(gpu) and os.path.exists(ref)):
        pytest.skip("drop-in binaries not built (oracle/Makefile needs /root/reference)")
    return gpu, ref


def test_dropin_binaries_link_the_product_library():
    """dropin_gpu leaves the hot-path symbols undefined (bound to
    libcolorvibe_gpu.so at run time) and defines the reference callers."""
    gpu, _ = _binaries()
    syms = subprocess.run(["nm", "-DC", gpu], capture_output=True, text=True, check=True).stdout
    for name in ("colorvibe::batch_search(", "colorvibe::serial_search(", "colorvibe::select_best("):
        assert any(name in ln and " U " in ln for ln in syms.splitlines()), name
    libs = subprocess.run(["ldd", gpu], capture_output=True, text=True).stdout
    assert "libcolorvibe_gpu.so" in libs and "not found" not in libs.split("libcolorvibe_gpu.so")[1].split("\n")[0]


@pytest.mark.gpu
def test_reference_callers_on_the_gpu_library_match_the_reference():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    gpu, ref = _binaries()
    a = subprocess.run([gpu], capture_output=True, text=True, timeout=600)
    assert a.returncode == 0, a.stderr[-2000:]
    b = subprocess.run([ref], capture_output=True, text=True, timeout=600)
    assert b.returncode == 0, b.stderr[-2000:]
    la, lb = a.stdout.splitlines(), b.stdout.splitlines()
    assert len(la) == len(lb)
    diff = [(x, y) for x, y in zip(la, lb) if x != y]
    assert not diff, diff[:5]
    assert "serial_equals_batch 240/240" in la
    assert "bench combos=756 candidates=36000 pairs=408364 parity=1" in la
