"""Shared helpers for tests of the product library (libdynbatch.so)."""
import json
import os
import re

import numpy as np

import oracle_lib as O
import paper_1707_02402_b200 as db

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols(headers=("dynbatch.h", "dynbatch_device.h")):
    """Every DYNBATCH_API function declared in include/dynbatch/*.h."""
    names = []
    for h in headers:
        text = open(os.path.join(ROOT, "include", "dynbatch", h)).read()
        names += re.findall(r"DYNBATCH_API[^;]*?\b(db_\w+)\s*\(", text, re.S)
    return names


def gpu_available() -> bool:
    try:
        return db.device_count() > 0
    except Exception:
        return False


def programs_from_json(text):
    return json.loads(text)["programs"]


def ref_batch_for(kind, b, p=40, depth=4, length=16, bp=0.1, seed=0):
    return O.ref_gen_batch(kind, b, p=p, depth=depth, length=length, bp=bp, seed=seed)


def max_norm_err(a, ref):
    """max|a - ref| / max|ref| — the stated metric for tensor-core paths."""
    den = np.max(np.abs(ref))
    return float(np.max(np.abs(a - ref)) / (den if den > 0 else 1.0))
