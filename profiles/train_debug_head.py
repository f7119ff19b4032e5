"""Where the head's bias gradient differs from the faithful fp64 reference."""
import sys
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
import test_device_train as T
for case in [("chain", 2, 4, 4, 2, 0.0, 21), ("chain", 3, 4, 4, 2, 0.0, 22)]:
    s, loss, ref_loss, mod, head, dx = T._run(*case)
    got, ref = s.grad("head_bp").astype(np.float64), head[1]
    d = np.abs(got - ref)
    order = np.argsort(-d)[:8]
    print(case, "max|ref|", np.abs(ref).max(), "n>1e-3*max:", int(np.sum(d > 1e-3 * np.abs(ref).max())))
    for c in order:
        print("   c", c, "dev", got[c], "ref", ref[c], "diff", d[c])
