"""Measured Tier-B errors at every BASELINE IEP config, full size, against the
fp64 oracle (tests/parity_full.py; the same rows the -m gpu tests check).
Writes one JSON object: per config the sampled rows, max-norm and
element-wise error, and their bars.

    python profiles/tierb_parity.py > profiles/r02_tierb_parity.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import parity_full as P  # noqa: E402
import paper_1707_02402_b200 as db  # noqa: E402

db.device_open(0)
out = {"tolerance": {"max_norm": P.TOL_NORM, "elem": P.TOL_ELEM},
       "oracle": "orc_execute kind=resblock (fp64), pinned to torch conv2d fp64 (tests/test_oracle_resblock_torch.py)",
       "device": "k_rb_step: fp16 operands, fp32 accumulation, residual as fp16 hi+lo, fp32 node values",
       "module_seed": "mix_seed(0, 0xd00d)", "configs": {}}
plan = [("cfg1", None, 64)] + [("cfg2", d, 32) for d in (4, 5, 6, 7, 8)] + [("cfg3", None, 128)]
for name, depth, n in plan:
    t0 = time.time()
    rows, dev, ref, sizes, st = P.run_config(name, n, depth=depth)
    e = P.errors(dev, ref)
    per_row = [P.errors(dev[i:i + 1], ref[i:i + 1])["max_norm"] for i in range(len(rows))]
    key = name if depth is None else f"{name}_d{depth}"
    out["configs"][key] = {"rows_checked": len(rows), "batch": int(P.CONFIGS[name]["b"]),
                           "program_nodes": [int(sizes.min()), int(sizes.max())],
                           **e, "worst_row_max_norm": max(per_row),
                           "pass": e["max_norm"] <= P.TOL_NORM and e["elem"] <= P.TOL_ELEM,
                           "expensive_calls": int(st.expensive_calls), "steps": int(st.steps),
                           "seconds": round(time.time() - t0, 1)}
    print(key, out["configs"][key], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
