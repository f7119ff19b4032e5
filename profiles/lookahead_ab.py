"""cfg3 forward time per DYNBATCH_LOOKAHEAD (SM-rows of tiles), interleaved."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
sys.path.insert(0, %r)
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
print(min(s.time(10)[0] / 10 for _ in range(3)))
"""
vals = sys.argv[1:] or ["1", "2", "4"]
res = {v: [] for v in vals}
for _ in range(3):
    for v in vals:
        env = dict(os.environ, DYNBATCH_LOOKAHEAD=v)
        out = subprocess.run([sys.executable, "-c", CHILD % ROOT], env=env, capture_output=True, text=True)
        res[v].append(float(out.stdout.strip().splitlines()[-1]))
for v, t in res.items():
    print(f"lookahead {v}: {min(t):.3f} ms (all {[round(x, 3) for x in t]})")
