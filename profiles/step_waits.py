"""MMA-thread wait breakdown of the fused conv step kernel (cfg3)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
CLK_GHZ = float(os.environ.get("CLK_GHZ", "1.9"))
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
_, kt = s.time(5, profile=True)
db.conv_wait_counters(reset=True, enable=True)
s.time(5)
w = db.conv_wait_counters(reset=True, enable=False)
acc, a, bb, tot = (int(x) for x in w[3])
cover = tot / (148 * kt.ms[4] * 1e-3 * CLK_GHZ * 1e9)
print(f"step kernel ms/fwd {kt.ms[4] / 5:.3f}: acc_wait {acc/tot:6.1%}  A_wait {a/tot:6.1%}  B_wait {bb/tot:6.1%}  "
      f"busy {(tot-acc-a-bb)/tot:6.1%}  loop/kernel {cover:6.1%}")
it, dep, sl, ptot = (int(x) for x in w[4])
print(f"window producer: item-ring wait {it/ptot:6.1%}  dependency wait {dep/ptot:6.1%}  "
      f"slot wait {sl/ptot:6.1%}  issuing {(ptot-it-dep-sl)/ptot:6.1%}")
cyc, ns = int(w[5][0]), int(w[5][1])
print(f"effective SM clock in the MMA loop: {cyc / max(ns, 1) * 1e3:.0f} MHz")
