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
