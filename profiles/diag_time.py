"""Production-build (no debug counters) forward time of the cfg3 step kernel
under DYNBATCH_DIAG variants, each in a fresh process, plus the SM clock the
debug build measures for the same variant. Timing only (wrong results).
usage: python profiles/diag_time.py 0 39 103 167 231"""
import json
import os
import subprocess
import sys

CHILD = r"""
import os, sys, json
sys.path.insert(0, %r)
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
_, kt = s.time(5, profile=True)
ms = kt.ms[4] / 5
db.conv_wait_counters(reset=True, enable=True)
s.time(3)
w = db.conv_wait_counters(reset=True, enable=False).reshape(-1)
print(json.dumps({"ms": ms, "mhz": float(w[20]) / max(float(w[21]), 1.0) * 1e3}))
""" % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

IDEAL_MCYC = 4.63  # cfg3: issued MMA cycles per SM and forward at 128 cycles per N=256 MMA
for d in sys.argv[1:] or ["0", "39"]:
    r = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, DYNBATCH_DIAG=d), capture_output=True,
                       text=True, timeout=600)
    try:
        v = json.loads(r.stdout.strip().splitlines()[-1])
    except Exception:
        print(d, "ERROR", r.stderr[-400:], flush=True)
        continue
    mcyc = v["ms"] * v["mhz"] / 1e3
    print(f"diag={d:4s} step kernel {v['ms']:.3f} ms  clock {v['mhz']:.0f} MHz  {mcyc:.2f} Mcycles "
          f"(ideal MMA {IDEAL_MCYC}: {IDEAL_MCYC / mcyc:.2f})", flush=True)
