"""SGD with the device gradients: first-order prediction of one step's loss
decrease (lr·‖g‖² over every module and head parameter) against the measured
decrease, then the loss over a few steps (tests/test_device_train.py)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 196
NAMES = ("w0", "b0", "w1", "b1", "w2", "b2")
b = int(sys.argv[1]) if len(sys.argv) > 1 else 64
batch = db.Batch.generate("chain", batch=b, vocab=40, width=F, length=16, branch_prob=0.1, seed=0)
s = db.IepSession(batch, 1234, db.MODULE_RESBLOCK)
s.set_head(28, 5)
s.set_training(True)
labels = (np.arange(b) % 28).astype(np.int32)
loss0 = s.train_step(labels)
g2 = 0.0
for f in range(1, 40):
    for n in NAMES:
        g = s.grad(n, f).astype(np.float64)
        g2 += float(np.sum(g * g))
for n in ("head_wp", "head_bp", "head_w1", "head_b1", "head_w2", "head_b2"):
    g = s.grad(n).astype(np.float64)
    g2 += float(np.sum(g * g))
out = {"programs": b, "loss0": loss0, "grad_norm2": g2}
for frac in (1e-3, 1e-2):
    lr = frac * loss0 / g2
    s2 = db.IepSession(batch, 1234, db.MODULE_RESBLOCK)
    s2.set_head(28, 5)
    s2.set_training(True)
    l0 = s2.train_step(labels)
    s2.sgd(lr)
    l1 = s2.train_step(labels)
    out[f"step_{frac}"] = {"lr": lr, "predicted_decrease": lr * g2, "measured_decrease": l0 - l1}
losses = [loss0]
for _ in range(10):
    s.sgd(0.5)
    losses.append(s.train_step(labels))
out["losses_lr_0.5"] = losses
print(json.dumps(out))
