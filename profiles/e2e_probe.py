import os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
xin = [db.PinnedArray((4096, F), np.float32) for _ in range(2)]
xout = [db.PinnedArray((4096, F), np.float32) for _ in range(2)]
s.forward_host(xin[0].array, xout[0].array); s.synchronize()
for mode in ("async", "forward_only", "sync"):
    s.synchronize()
    t0 = time.perf_counter(); ts = []
    for i in range(8):
        a = time.perf_counter()
        if mode == "async": s.forward_host_async(xin[i % 2].array, xout[i % 2].array)
        elif mode == "sync": s.forward_host(xin[i % 2].array, xout[i % 2].array)
        else: s.forward()
        ts.append((time.perf_counter() - a) * 1e3)
    s.synchronize()
    tot = (time.perf_counter() - t0) / 8 * 1e3
    print(mode, f"{tot:.2f} ms/call; host ms per call", [round(x, 2) for x in ts])
