"""Measured MoE errors at the BASELINE shapes vs fp64 reference arithmetic
on sampled tokens (tests/moe_full.py; the same check the -m gpu tests make),
for the fp16 (precise) and bf16 (wide-range) tensor-core modes.

    python profiles/moe_parity.py > profiles/r02_moe_parity.json
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import moe_full as M  # noqa: E402
import paper_1707_02402_b200 as db  # noqa: E402

db.device_open(0)
out = {"metric": "max|dev - ref| / max|ref| over the sampled tokens' outputs",
       "reference": "fp64 ExpertSet::apply + slot-order combine (tests/moe_full.py) on the oracle's bit-exact "
                    "generators and top_k_gate", "tolerance": {"fp16": M.TOL_FP16, "bf16": M.TOL_BF16}, "runs": {}}
for name, n_tok in (("cfg4", 1024), ("cfg5", 128)):
    c = M.CFG[name]
    toks = M.sample_tokens(c["T"], n_tok)
    t0 = time.time()
    ids, w, ref = M.reference_tokens(c["n"], c["k"], c["d"], c["h"], 0, toks)
    t_ref = time.time() - t0
    for pname, prec in (("fp16", db.MOE_FP16), ("bf16", db.MOE_BF16)):
        t0 = time.time()
        s = db.MoeSession(c["n"], c["k"], c["T"], c["d"], c["h"], seed=0, precision=prec)
        s.forward()
        dev = s.outputs(toks)
        dids, dw, _, _ = s.routing()
        r = {"tokens_checked": int(len(toks)), "tokens": c["T"], "max_norm": M.max_norm(dev, ref),
             "max_abs": float(np.max(np.abs(dev - ref))), "max_abs_ref": float(np.max(np.abs(ref))),
             "routing_equal": bool(np.array_equal(dids[toks], ids)),
             "pass": M.max_norm(dev, ref) <= (M.TOL_FP16 if pname == "fp16" else M.TOL_BF16),
             "seconds": round(time.time() - t0, 1), "reference_seconds": round(t_ref, 1)}
        out["runs"][f"{name}_{pname}"] = r
        print(name, pname, r, file=sys.stderr, flush=True)
        del s
print(json.dumps(out, indent=1))
