"""Full-size Tier-B parity helpers (BASELINE IEP configs vs the fp64 oracle).

Shared by tests/test_device_resblock_full.py (which asserts the stated
tolerance) and profiles/tierb_parity.py (which records the measured errors).
The device runs the whole BASELINE batch through one session; the oracle
(orc_execute kind=resblock, pinned to torch conv2d by
tests/test_oracle_resblock_torch.py) evaluates a spread of sampled programs,
each as its own one-program batch — rows are independent
(tests/test_executor.cpp:98-119), so a program's output does not depend on
the rest of the batch. Test infrastructure only.
"""
from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np

import oracle_lib as O
import paper_1707_02402_b200 as db

F = 128 * 14 * 14
MODULE_SEED = O.mix_seed(0, 0xd00d)  # bench.py / SURVEY §8(d) convention

# BASELINE.json configs[0..2]
CONFIGS = {
    "cfg1": dict(kind="chain", b=64, p=40, depth=4, length=16, bp=0.1),
    "cfg2": dict(kind="balanced", b=512, p=40, depth=6, length=16, bp=0.1),
    "cfg3": dict(kind="chain", b=4096, p=40, depth=4, length=16, bp=0.3),
}

TOL_NORM = 1e-3   # max|dev − ref| / max|ref| (the north star's figure)
TOL_ELEM = 5e-3   # per element |dev − ref| / (|ref| + rms(ref))


def sub_batch(ob: O.Batch, r: int) -> O.Batch:
    lo, hi = int(ob.prog_off[r]), int(ob.prog_off[r + 1])
    return O.Batch(np.array([0, hi - lo], np.int32), ob.fid[lo:hi].copy(), ob.child0[lo:hi].copy(),
                   ob.child1[lo:hi].copy(), ob.root[r:r + 1].copy(), ob.p)


def spread_rows(ob: O.Batch, n: int) -> list:
    """n programs spread over program size (node count), smallest and
    largest included, ties broken by index."""
    sizes = np.diff(ob.prog_off)
    order = np.lexsort((np.arange(ob.b), sizes))
    if n >= ob.b:
        return list(range(ob.b))
    pick = np.unique(np.round(np.linspace(0, ob.b - 1, n)).astype(int))
    return sorted(int(order[i]) for i in pick)


def oracle_rows(ob: O.Batch, x: np.ndarray, rows, module_seed=MODULE_SEED, threads=None):
    threads = threads or max(1, min(len(rows), len(os.sched_getaffinity(0))))

    def one(r):
        sb = sub_batch(ob, r)
        res = O.execute(sb, O.schedule_improved(sb), np.ascontiguousarray(x[r:r + 1]), module_seed, "resblock")
        assert res.rc == 0, res.rc
        return res.outputs[0]

    with ThreadPoolExecutor(max_workers=threads) as pool:
        return np.stack(list(pool.map(one, rows)))


def errors(dev: np.ndarray, ref: np.ndarray) -> dict:
    den = np.max(np.abs(ref))
    rms = np.sqrt(np.mean(ref ** 2))
    return {"max_norm": float(np.max(np.abs(dev - ref)) / den),
            "elem": float(np.max(np.abs(dev - ref) / (np.abs(ref) + rms))),
            "max_abs": float(np.max(np.abs(dev - ref))),
            "max_abs_ref": float(den)}


def run_config(name, n_rows, depth=None, module_seed=MODULE_SEED):
    """Device outputs for the whole BASELINE batch, oracle outputs for
    n_rows sampled programs. Returns (rows, dev[rows], ref, per-row depth
    labels, session stats)."""
    c = dict(CONFIGS[name])
    if depth is not None:
        c["depth"] = depth
    batch = db.Batch.generate(c["kind"], batch=c["b"], vocab=c["p"], width=F, depth=c["depth"],
                              length=c["length"], branch_prob=c["bp"], seed=0)
    sess = db.IepSession(batch, module_seed, db.MODULE_RESBLOCK)
    sess.forward()
    sess.synchronize()
    dev = sess.run().outputs()
    ob = O.gen_batch(c["kind"], c["b"], p=c["p"], depth=c["depth"], length=c["length"], bp=c["bp"], seed=0)
    x = O.random_batch(c["b"], F, O.mix_seed(0, 0x1127))
    rows = spread_rows(ob, n_rows)
    ref = oracle_rows(ob, x, rows, module_seed)
    sizes = np.diff(ob.prog_off)[rows]
    return rows, dev[rows], ref, sizes, sess.stats()
