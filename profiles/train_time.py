"""Training-step time (forward + head + loss + backward, device ms) on
chain-heavy batches, next to the forward alone, and the naive schedule's
step on the same programs (the paper's batched-backward comparison,
PAPER.md:75)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
out = {}
for b in [int(x) for x in (sys.argv[1:] or ["64", "512", "4096"])]:
    batch = db.Batch.generate("chain", batch=b, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
    s = db.IepSession(batch, 1234, db.MODULE_RESBLOCK)
    fwd_ms = s.time(3)[0] / 3
    s.set_head(28, 5)
    s.set_training(True)
    labels = (np.arange(b) % 28).astype(np.int32)
    tr_ms = s.time_train(3, labels)
    row = {"forward_ms": fwd_ms, "train_step_ms": tr_ms, "train_programs_per_s": b / (tr_ms / 1e3),
           "backward_over_forward": (tr_ms - fwd_ms) / fwd_ms}
    if b <= 64:
        n = db.IepSession(batch, 1234, db.MODULE_RESBLOCK)
        n.set_schedule(db.Batch.generate("chain", batch=b, vocab=40, width=8, length=16, branch_prob=0.3,
                                         seed=0).schedule("naive"))
        n.set_head(28, 5)
        n.set_training(True)
        nms = n.time_train(2, labels)
        row["naive_train_step_ms"] = nms
        row["improved_over_naive"] = nms / tr_ms
    out[b] = row
    print(b, json.dumps(row), flush=True)
