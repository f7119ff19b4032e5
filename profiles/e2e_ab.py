"""Interleaved A/B of the end-to-end bench figure between library builds
(DYNBATCH_LIB): python profiles/e2e_ab.py lib_a.so lib_b.so [rounds]."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
libs = [a for a in sys.argv[1:] if a.endswith(".so")]
rounds = int(sys.argv[-1]) if not sys.argv[-1].endswith(".so") else 3
res = {l: [] for l in libs}
for _ in range(rounds):
    for l in libs:
        env = dict(os.environ, DYNBATCH_LIB=os.path.abspath(l))
        out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-moe", "--no-cpu-baseline"],
                             env=env, capture_output=True, text=True)
        d = json.loads(out.stdout.strip().splitlines()[-1])
        res[l].append(round(d["e2e"]["value"]))
for l, v in res.items():
    print(l, "e2e programs/s:", v, "median", sorted(v)[len(v) // 2])
