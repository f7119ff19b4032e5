import sys, os
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import test_device_train as T
from dbtest import max_norm_err
for case in [("chain", 4, 10, 4, 5, 0.4, 1), ("balanced", 3, 8, 3, 8, 0.0, 2), ("dag", 3, 9, 4, 6, 0.5, 3)]:
    s, loss, ref_loss, mod, head, dx = T._run(*case)
    print(case[0], "loss", loss, ref_loss)
    for f, grads in mod.items():
        errs = []
        for name, ref in zip(T.NAMES, grads):
            if name in ("w0", "b0") and not np.any(ref): continue
            errs.append((name, round(max_norm_err(s.grad(name, f).astype(np.float64), ref.reshape(-1)), 5)))
        print("  f", f, errs)
    print("  head", [round(max_norm_err(s.grad(n).astype(np.float64), r.reshape(-1)), 5) for n, r in zip(("head_wp","head_bp","head_w1","head_b1","head_w2","head_b2"), head)])
    print("  inputs", round(max_norm_err(s.grad("inputs").astype(np.float64), dx.reshape(-1)), 5))
