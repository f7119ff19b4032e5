"""Measured error of the Tier-B residual-block path vs the fp64 oracle
(max|dev-ref|/max|ref| and the element-wise bound of the tests)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_lib as O  # noqa: E402
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 196
for kind, b, p, length, bp, seed in [("chain", 16, 40, 16, 0.3, 0), ("chain", 8, 40, 16, 0.1, 1),
                                     ("balanced", 4, 40, 16, 0.0, 2)]:
    batch = db.Batch.generate(kind, batch=b, vocab=p, width=F, depth=5, length=length, branch_prob=bp,
                              seed=seed)
    out = batch.execute_device(O.mix_seed(seed, 0xd00d), db.MODULE_RESBLOCK).outputs()
    ob = O.gen_batch(kind, b, p=p, depth=5, length=length, bp=bp, seed=seed)
    x = O.random_batch(b, F, O.mix_seed(seed, 0x1127))
    ref = O.execute(ob, O.schedule_improved(ob), x, O.mix_seed(seed, 0xd00d), "resblock").outputs
    err = np.max(np.abs(out - ref)) / np.max(np.abs(ref))
    rms = np.sqrt(np.mean(ref ** 2))
    elem = np.max(np.abs(out - ref) / (np.abs(ref) + rms))
    print(f"{kind} b={b} len<={length} bp={bp}: max-norm {err:.3e}  elementwise {elem:.3e}  "
          f"levels={O.labels(ob)[1] + 1}")
