"""Upper bounds of the fused step kernel with the weight and/or window
reloads skipped (DYNBATCH_DIAG bits; results are wrong, timing only)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
for d in (sys.argv[1:] or ["0", "1", "2", "3", "4", "7", "0"]):
    os.environ["DYNBATCH_DIAG"] = d
    _, kt = s.time(5, profile=True)
    print(f"diag={d}: step kernel ms/fwd {kt.ms[4] / 5:.3f}")
