"""Where does the conv MMA thread wait? Runs cfg3 forwards with the per-kind
wait accounting on and prints the share of the MMA loop spent waiting for a
drained accumulator, an A window and a weight stage."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
for mode in ("1", "0"):
    os.environ["DYNBATCH_CONV_PAIR"] = mode
    b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
    s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
    s.time(2)
    db.conv_wait_counters(reset=True, enable=True)
    ms, _ = s.time(5)
    w = db.conv_wait_counters(reset=True, enable=False)
    print(f"pair={mode} ms/forward={ms/5:.3f}")
    for kind in range(6):
        acc, a, bb, tot = (int(x) for x in w[kind])
        if tot:
            print(f"  kind {kind}: acc_wait {acc/tot:6.1%}  A_wait {a/tot:6.1%}  B_wait {bb/tot:6.1%}  (cycles {tot:.3e})")
