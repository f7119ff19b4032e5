"""Interleaved A/B of library builds (DYNBATCH_LIB) on cfg1 and cfg3 device
forwards: python profiles/ab_configs.py lib_a.so lib_b.so [...]"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
sys.path.insert(0, %r)
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=%d, vocab=40, width=F, length=16, branch_prob=%s, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
print(min(s.time(20)[0] / 20 for _ in range(3)))
"""
libs = sys.argv[1:]
for name, b, bp in (("cfg1", 64, "0.1"), ("cfg3", 4096, "0.3")):
    res = {l: [] for l in libs}
    for _ in range(3):
        for l in libs:
            env = dict(os.environ, DYNBATCH_LIB=os.path.abspath(l))
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, b, bp)], env=env, capture_output=True, text=True)
            res[l].append(float(out.stdout.strip().splitlines()[-1]))
    print(name, "  ".join(f"{l}: {min(v):.4f} ms" for l, v in res.items()))
