"""Session sequences with the step barrier on / off (stray write hunt).
argv: sequence of barrier flags, 'k' = keep previous sessions alive."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1707_02402_b200 as db
F = 128 * 196
b = db.Batch.generate("chain", batch=64, vocab=40, width=F, length=16, branch_prob=0.1, seed=0)
sched = db.Batch.generate("chain", batch=64, vocab=40, width=8, length=16, branch_prob=0.1, seed=0).schedule("naive")
ref = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
ref.forward()
want = ref.run().outputs()
keep = []
seq = sys.argv[1]
for i, ch in enumerate(seq):
    if ch == "k":
        continue
    os.environ["DYNBATCH_STEP_BARRIER"] = ch
    try:
        x = db.IepSession(b, 1234, db.MODULE_RESBLOCK, first=0, last=64)
        x.set_schedule(sched)
        x.time(1)
        x.time(2)
        got = x.run().outputs()
        print(seq, i, "barrier", ch, "equal" if np.array_equal(got, want) else "DIFF", flush=True)
    except Exception as e:
        print(seq, i, "barrier", ch, "ERR", e, flush=True)
    if "k" in seq:
        keep.append(x)
    del x
