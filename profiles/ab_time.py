"""Interleaved A/B forward timing of library builds on one box:
python profiles/ab_time.py lib_a.so lib_b.so [...] [--rounds R]. Each round
runs each build in a fresh process (cfg3, 10 timed forwards after 3
warm-ups, best of 3)."""
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
""" % ROOT

args = sys.argv[1:]
rounds = 3
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    args = args[:i] + args[i + 2:]
libs = args
res = {l: [] for l in libs}
for _ in range(rounds):
    for l in libs:
        env = dict(os.environ, DYNBATCH_LIB=os.path.abspath(l))
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        res[l].append(float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else float("nan"))
for l in libs:
    v = sorted(res[l])
    print(f"{l}: ms/forward min {v[0]:.3f} median {v[len(v) // 2]:.3f}  all {[round(x, 3) for x in res[l]]}")
