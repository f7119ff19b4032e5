import os, sys
sys.path.insert(0, os.getcwd())
import paper_1707_02402_b200 as db
F = 128 * 196
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(5)
for rep in range(2):
    g, _ = s.time(10)
    p, kt = s.time(10, profile=True)
    print("graph/direct-unprof ms/fwd %.3f  profiled %.3f  classes %s" % (g / 10, p / 10,
          [(db.KERNEL_CLASSES[c], round(kt.ms[c] / 10, 3)) for c in range(8) if kt.launches[c]]), flush=True)
