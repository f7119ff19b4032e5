"""Step-kernel cycle accounting (profiles/step_waits.py) under each
DYNBATCH_DIAG variant, one subprocess per variant (timing only; the
variants give wrong results): which resource bounds the MMA loop and the
epilogue. usage: python profiles/diag_waits.py [diag ...] > out.json"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
out = {}
for d in (sys.argv[1:] or ["0", "32", "3", "35", "8", "16", "43", "0"]):
    env = dict(os.environ, DYNBATCH_DIAG=d)
    r = subprocess.run([sys.executable, os.path.join(HERE, "step_waits.py")], env=env, capture_output=True,
                       text=True, timeout=600)
    try:
        w = json.loads(r.stdout)
    except json.JSONDecodeError:
        out[d] = {"error": r.stderr[-2000:]}
        continue
    row = {"ms": round(w["ms_per_forward"], 3), "mhz": round(w["mma_loop_mhz"]),
           "mma_thread": {k: round(v, 3) for k, v in w["mma_thread"].items()},
           "producer": {k: round(v, 3) for k, v in w["producer"].items()}}
    for k, v in w["per_kind"].items():
        row[k] = {"mma": round(v["mma_item_cycles_per_tile"]), "win": round(v["window_wait_per_tile"]),
                  "wgt": round(v["weight_wait_per_tile"]), "acc": round(v["acc_wait_per_tile"]),
                  "epi": round(v["epilogue_cycles_per_tile"]), "dep": round(v["producer_dep_wait_per_tile"])}
    out[d] = row
    print(d, json.dumps(row), file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))
