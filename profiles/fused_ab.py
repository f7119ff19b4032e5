"""cfg3 forward time with the fused per-step conv kernel vs the three
separate conv launches (DYNBATCH_FUSED=0), plus the per-class breakdown."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
for mode in ("1", "0", "1"):
    os.environ["DYNBATCH_FUSED"] = mode
    b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
    s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
    s.time(3)
    ms, _ = s.time(10)
    _, kt = s.time(5, profile=True)
    cls = {c: round(kt.ms[c] / 5, 3) for c in range(8) if kt.launches[c]}
    print(f"fused={mode} ms/forward={ms / 10:.3f}  per-class ms {cls}")
