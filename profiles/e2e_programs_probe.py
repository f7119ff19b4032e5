"""Cost of new programs every call: forward-only loops with and without
set_programs (device build of the CSR), and the pipelined host call with
and without it (wall clock per call)."""
import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
kw = dict(batch=4096, vocab=40, width=F, length=16, branch_prob=0.3)
bs = [db.Batch.generate("chain", seed=s, **kw) for s in (0, 1)]
seqs = [b.prefix_tokens() for b in bs]
toks, offs = [], []
for t, o in seqs:
    pt, po = db.PinnedArray(t.shape, np.int32), db.PinnedArray(o.shape, np.int32)
    pt.array[:] = t; po.array[:] = o
    toks.append(pt); offs.append(po)
s = db.IepSession(bs[0], 1234, db.MODULE_RESBLOCK, program_capacity=4096,
                  node_capacity=max(int(o[-1]) for _, o in seqs),
                  length_capacity=max(int(np.diff(o).max()) for _, o in seqs))
xin = [db.PinnedArray((4096, F), np.float32) for _ in range(2)]
xout = [db.PinnedArray((4096, F), np.float32) for _ in range(2)]
s.forward_host(xin[0].array, xout[0].array); s.synchronize()
n = 12
for mode in ("forward", "set+forward", "async", "set+async"):
    for rep in range(2):
        s.synchronize()
        t0 = time.perf_counter(); hs = []
        for i in range(n):
            a = time.perf_counter()
            if mode.startswith("set"):
                s.set_programs(toks[i % 2].array, offs[i % 2].array)
            hs.append((time.perf_counter() - a) * 1e3)
            if mode.endswith("async"):
                s.forward_host_async(xin[i % 2].array, xout[i % 2].array)
            else:
                s.forward()
        s.synchronize()
        tot = (time.perf_counter() - t0) / n * 1e3
    print(f"{mode:12s} {tot:.2f} ms/call; host ms in set_programs {np.median(hs):.3f}")
