import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo")); sys.path.insert(0, os.path.join(os.environ.get("GRAFT_REPO_ROOT", "/root/repo"), "tests"))
import numpy as np, paper_1707_02402_b200 as db
F = 128 * 14 * 14
def batch(seed, b): return db.Batch.generate("chain", batch=b, vocab=10, width=F, length=8, branch_prob=0.4, seed=seed)
a, bb = batch(1, 12), batch(2, 10)
xb = np.random.default_rng(1).uniform(-1, 1, size=(10, F)).astype(np.float32)
def run(sess, x):
    o = np.zeros_like(x); sess.forward_host(x, o); return o
want = run(db.IepSession(bb, 5, db.MODULE_RESBLOCK), xb)
cap = dict(program_capacity=16, node_capacity=400, length_capacity=16)
print("fresh B with capacity equal:", np.array_equal(run(db.IepSession(bb, 5, db.MODULE_RESBLOCK, **cap), xb), want))
s = db.IepSession(bb, 5, db.MODULE_RESBLOCK); s.set_programs(*bb.prefix_tokens())
print("B session, set_programs(B):", np.array_equal(run(s, xb), want))
s = db.IepSession(a, 5, db.MODULE_RESBLOCK, **cap); s.set_programs(*bb.prefix_tokens())
o = run(s, xb)
print("A session (no forward), set_programs(B):", np.array_equal(o, want), [int(r) for r in np.nonzero(np.any(o != want, axis=1))[0]])
print(bb.prefix_tokens())
s = db.IepSession(a, 5, db.MODULE_RESBLOCK, **cap)
xa = np.random.default_rng(0).uniform(-1, 1, size=(12, F)).astype(np.float32)
run(s, xa)
s.set_programs(*bb.prefix_tokens())
o = run(s, xb)
bad = [int(r) for r in np.nonzero(np.any(o != want, axis=1))[0]]
print("A forward, set_programs(B):", np.array_equal(o, want), bad)
t, off = bb.prefix_tokens()
for r in bad:
    d = np.abs(o[r] - want[r]); print(r, t[off[r]:off[r+1]].tolist(), "max diff", d.max(), "n diff", int((d > 0).sum()))
# same but after a forward on B itself
s2 = db.IepSession(bb, 5, db.MODULE_RESBLOCK, **cap); run(s2, xb); s2.set_programs(*bb.prefix_tokens())
print("B forward, set_programs(B):", np.array_equal(run(s2, xb), want))
fresh = db.IepSession(bb, 5, db.MODULE_RESBLOCK); run(fresh, xb)
print("schedules equal:", s.schedule().to_json() == fresh.schedule().to_json())
print("labels equal:", np.array_equal(s.labels(55), fresh.labels(55)))
# run B twice on the A-forwarded session: does a second forward fix it?
o2 = run(s, xb)
print("second forward equal:", np.array_equal(o2, want), "first==second:", np.array_equal(o, o2))
