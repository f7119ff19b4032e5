import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1707_02402_b200 as db
F = 128 * 196
b = db.Batch.generate("chain", batch=4, vocab=10, width=F, length=5, branch_prob=0.4, seed=1)
s = db.IepSession(b, 1001, db.MODULE_RESBLOCK)
s.set_head(10, 7); s.set_training(True)
labels = np.arange(4, dtype=np.int32) % 10
s.train_step(labels)
for f in (2, 4, 1, 3):
    for nm in ("w1", "w2", "b1"):
        try:
            g = s.grad(nm, f)
            print(os.environ.get("DYNBATCH_TRAIN_DGRAD", "1"), f, nm, float(np.linalg.norm(g)), g.reshape(-1)[:4])
        except Exception as e:
            print(f, nm, "ERR", e)
