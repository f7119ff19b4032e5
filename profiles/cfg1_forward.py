import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=64, vocab=40, width=F, length=16, branch_prob=0.1, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
s.time(2)
