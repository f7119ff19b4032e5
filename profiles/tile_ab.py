"""Step-kernel tile size 128 vs 256 (DYNBATCH_TILE_M), interleaved, on cfg1,
cfg2 depth 4 and cfg3."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import sys
sys.path.insert(0, %r)
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
b = db.Batch.generate(%r, batch=%d, vocab=40, width=F, depth=%d, length=16, branch_prob=%s, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
print(min(s.time(10)[0] / 10 for _ in range(3)))
"""
for name, kind, b, depth, bp in (("cfg1", "chain", 64, 4, "0.1"), ("cfg2_d4", "balanced", 512, 4, "0.1"),
                                  ("cfg2_d6", "balanced", 512, 6, "0.1"), ("cfg3", "chain", 4096, 4, "0.3")):
    res = {"128": [], "256": []}
    for _ in range(2):
        for tm in ("128", "256"):
            env = dict(os.environ, DYNBATCH_TILE_M=tm)
            out = subprocess.run([sys.executable, "-c", CHILD % (ROOT, kind, b, depth, bp)], env=env,
                                 capture_output=True, text=True)
            res[tm].append(float(out.stdout.strip().splitlines()[-1]))
    print(f"{name}: tile 128 {min(res['128']):.3f} ms, tile 256 {min(res['256']):.3f} ms")
