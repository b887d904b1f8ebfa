"""Shared helpers for the test-suite (fixtures live in conftest.py)."""
import hashlib
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f) if name.endswith(".json") else f.read()


def sha_records(idx, codes):
    m = hashlib.sha256()
    m.update(np.ascontiguousarray(idx, np.uint32).tobytes())
    m.update(np.ascontiguousarray(codes, np.uint8).tobytes())
    return m.hexdigest()


def records10_sha(idx, codes, chunk=1 << 24):
    """sha256 over 10-byte records (u32 LE idx, then the 6 code bytes), the
    layout of tests/golden/make_golden.py's cfg2 fixture; chunked so that a
    cfg2 target's ~80M pairs hash in bounded memory."""
    m = hashlib.sha256()
    for a in range(0, len(idx), chunk):
        b = min(a + chunk, len(idx))
        rec = np.empty((b - a, 10), np.uint8)
        rec[:, :4] = np.ascontiguousarray(idx[a:b], "<u4").view(np.uint8).reshape(-1, 4)
        rec[:, 4:] = codes[a:b]
        m.update(rec.tobytes())
    return m.hexdigest()
