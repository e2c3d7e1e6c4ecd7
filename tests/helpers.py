"""Shared test helpers: golden fixtures and digests (test infrastructure)."""
import functools
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
QUERY_NAMES = ["q11", "q12", "q13", "q21", "q22", "q23", "q31", "q32", "q33", "q34",
               "q41", "q42", "q43"]


@functools.lru_cache(maxsize=None)
def golden(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as f:
        return json.load(f)


def golden_rows(rec):
    return [(tuple(g), s) for g, s in rec["result"]]


def col_digest(a):
    """Same definition as tests/golden/make_golden.py: sum((u32)v*(2i+1)) mod 2^64."""
    a = np.asarray(a).astype(np.int64) & 0xFFFFFFFF
    total = 0
    chunk = 1 << 24
    for i in range(0, len(a), chunk):
        w = np.arange(i, min(len(a), i + chunk), dtype=np.uint64) * np.uint64(2) + np.uint64(1)
        with np.errstate(over="ignore"):
            total = (total + int(np.sum(a[i:i + chunk].astype(np.uint64) * w, dtype=np.uint64))) % (1 << 64)
    return f"{total:016x}"


def fixture_tables():
    fx = golden("fixture")["tables"]
    return {t: {c: np.array(v, np.int32) for c, v in cols.items()} for t, cols in fx.items()}
