"""Fused step kernel: forward time vs the conv3x3 #2 lookahead (× SMs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
for la in sys.argv[1:] or ["2", "4", "8", "16", "64"]:
    os.environ["DYNBATCH_LOOKAHEAD"] = la
    ms, _ = s.time(10)
    _, kt = s.time(5, profile=True)
    print(f"lookahead {la}x: ms/forward={ms / 10:.3f} step={kt.ms[4] / 5:.3f}")
