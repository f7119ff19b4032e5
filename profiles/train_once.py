"""One training step of a chain-heavy batch (for ncu launch lists)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1707_02402_b200 as db  # noqa: E402

b = int(sys.argv[1]) if len(sys.argv) > 1 else 512
batch = db.Batch.generate("chain", batch=b, vocab=40, width=128 * 196, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(batch, 1234, db.MODULE_RESBLOCK)
s.set_head(28, 5)
s.set_training(True)
labels = (np.arange(b) % 28).astype(np.int32)
s.train_step(labels)
s.train_step(labels)
