"""Per-tensor relative Frobenius gradient errors of the device training step against the
device-faithful fp64 reference (tests/train_ref.py) on small programs."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import test_device_train as T
from dbtest import max_norm_err


def fro(a, r):
    return float(np.linalg.norm(a - r) / max(np.linalg.norm(r), 1e-300))

cases = [("chain", 2, 4, 4, 2, 0.0, 21), ("chain", 3, 4, 4, 2, 0.0, 22), ("balanced", 1, 2, 2, 8, 0.0, 23), ("balanced", 1, 2, 3, 8, 0.0, 24), ("balanced", 2, 2, 2, 8, 0.0, 25)]
for case in cases:
    s, loss, ref_loss, mod, head, dx = T._run(*case)
    out = [case[0] + str(case[1:5])]
    for f, grads in mod.items():
        e = [round(fro(s.grad(n, f).astype(np.float64), r.reshape(-1)), 4)
             for n, r in zip(T.NAMES, grads) if not (n in ("w0", "b0") and not np.any(r))]
        out.append(f"f{f}:{e}")
    out.append("head:" + str([round(fro(s.grad(n).astype(np.float64), r.reshape(-1)), 4) for n, r in
                              zip(("head_wp", "head_bp", "head_w1", "head_b1", "head_w2", "head_b2"), head)]))
    out.append("in:%.4f" % fro(s.grad("inputs").astype(np.float64), dx.reshape(-1)))
    print(" ".join(out), flush=True)
