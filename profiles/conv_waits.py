"""Where does the conv MMA thread wait? Runs cfg3 forwards with the per-kind
wait accounting on and prints, per conv kind, the share of the MMA loop spent
waiting for a drained accumulator, an A window and a weight stage, and the
loop's coverage of the kernel time (MMA-loop cycles ÷ (issuing CTAs × event
time × SM clock))."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
CLK_GHZ = float(os.environ.get("CLK_GHZ", "1.9"))
for mode in ("0",):
    b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
    s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
    s.time(2)
    ms0, _ = s.time(5)
    _, kt = s.time(5, profile=True)
    db.conv_wait_counters(reset=True, enable=True)
    s.time(5)
    w = db.conv_wait_counters(reset=True, enable=False)
    print(f"ms/forward={ms0/5:.3f}")
    issuers = 148
    for kind in range(3):
        acc, a, bb, tot = (int(x) for x in w[kind])
        if tot:
            cls = 3 + kind % 3
            cover = tot / (issuers * kt.ms[cls] * 1e-3 * CLK_GHZ * 1e9)
            print(f"  kind {kind}: acc_wait {acc/tot:6.1%}  A_wait {a/tot:6.1%}  B_wait {bb/tot:6.1%}  "
                  f"busy {(tot-acc-a-bb)/tot:6.1%}  loop/kernel {cover:6.1%}  kernel ms/fwd {kt.ms[cls]/5:.3f}")
