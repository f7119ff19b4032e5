"""GPU parity of the IEP training step (
db_iep_session_train_step: training forward → head → mean softmax
cross-entropy → backward through the head and the module groups in reverse
step order) against torch fp64 autograd on the oracle's weights
(tests/train_ref.py), with the forward rounded to fp16 where the device's
is (straight-through, so the ReLU masks are the device's; the plain fp64
forward is checked for the loss).

Stated tolerance: a single block (no decision upstream of its gradients
but its own) meets max|dev − ref| / max|ref| ≤ 2e-3 on every gradient;
deeper programs meet a relative Frobenius error ||dev − ref||₂ / ||ref||₂ ≤
5e-2 per gradient tensor; the loss is within 1e-3 relative. A max-norm bound
does not fit a ReLU network differentiated at two slightly different
points: a unit or pooling window whose pre-activation rounds to the other
side of a ReLU or max-pool decision (fp32 vs fp64 accumulation before the
fp16 rounding) routes its whole gradient differently, and the transposed
convolutions spread that difference over every tensor below it. Measured on
the head: one of 512 projection-bias channels moved, every other entry
within 2e-4 (profiles/train_debug_head.py). Trees (unary / binary),
all-binary balanced trees and DAGs with shared children (gradients
accumulate) are covered."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db
from dbtest import max_norm_err
from train_ref import train_step_reference

pytestmark = pytest.mark.gpu

F = 128 * 14 * 14
TOL_FRO = 5e-2   # ||dev − ref||₂ / ||ref||₂ per gradient tensor
TOL_LOSS = 1e-3
NAMES = ("w0", "b0", "w1", "b1", "w2", "b2")


def _run(kind, b, p, depth, length, bp, seed, answers=10):
    batch = db.Batch.generate(kind, batch=b, vocab=p, width=F, depth=depth, length=length, branch_prob=bp,
                              seed=seed)
    ms = 1000 + seed
    s = db.IepSession(batch, ms, db.MODULE_RESBLOCK)
    s.set_head(answers, 7)
    s.set_training(True)
    labels = np.arange(b, dtype=np.int32) % answers
    loss = s.train_step(labels)
    bt = O.gen_batch(kind, b, p=p, depth=depth, length=length, bp=bp, seed=seed)
    x = O.random_batch(b, F, O.mix_seed(seed, 0x1127))
    ref_loss = train_step_reference(bt, x, ms, 7, answers, labels)[0]
    _, mod, head, dx, _ = train_step_reference(bt, x, ms, 7, answers, labels, faithful=True)
    return s, loss, ref_loss, mod, head, dx


def fro_err(got, ref):
    got, ref = np.asarray(got, np.float64).reshape(-1), np.asarray(ref, np.float64).reshape(-1)
    return float(np.linalg.norm(got - ref) / max(np.linalg.norm(ref), 1e-300))


def _check(label, got, ref):
    fro = fro_err(got, ref)
    assert fro <= TOL_FRO, (label, fro)
    return fro


def _check_all(s, loss, ref_loss, mod, head, dx):
    assert abs(loss - ref_loss) <= TOL_LOSS * abs(ref_loss), (loss, ref_loss)
    worst = 0.0
    for f, grads in mod.items():
        for name, ref in zip(NAMES, grads):
            if name in ("w0", "b0") and not np.any(ref):
                continue  # unary blocks have no conv1x1
            worst = max(worst, _check((f, name), s.grad(name, f), ref))
    for name, ref in zip(("head_wp", "head_bp", "head_w1", "head_b1", "head_w2", "head_b2"), head):
        worst = max(worst, _check(name, s.grad(name), ref))
    return max(worst, _check("inputs", s.grad("inputs"), dx))


@pytest.mark.parametrize("kind,b,p,depth,length,bp,seed", [
    ("chain", 4, 10, 4, 5, 0.4, 1),     # unary and binary blocks
    ("balanced", 3, 8, 3, 8, 0.0, 2),   # all-binary trees
    ("dag", 3, 9, 4, 6, 0.5, 3),        # shared children: gradients accumulate
])
def test_train_step_matches_torch_autograd(kind, b, p, depth, length, bp, seed):
    _check_all(*_run(kind, b, p, depth, length, bp, seed))


@pytest.mark.parametrize("kind,b,p,depth,length,bp,seed", [
    ("chain", 1, 4, 4, 2, 0.0, 11),     # one unary block on a leaf
    ("balanced", 1, 4, 2, 8, 0.0, 14),  # one binary block on two leaves
])
def test_train_step_single_block_max_norm(kind, b, p, depth, length, bp, seed):
    s, loss, ref_loss, mod, head, dx = _run(kind, b, p, depth, length, bp, seed)
    for f, grads in mod.items():
        for name, ref in zip(NAMES, grads):
            if name in ("w0", "b0") and not np.any(ref):
                continue
            assert max_norm_err(s.grad(name, f).astype(np.float64), ref.reshape(-1)) <= 2e-3, (f, name)
    assert max_norm_err(s.grad("inputs").astype(np.float64), dx.reshape(-1)) <= 2e-3


def test_train_step_is_repeatable():
    """Gradients are overwritten, not accumulated, by every step."""
    s, loss, *_ = _run("chain", 3, 10, 4, 4, 0.3, 5)
    g1 = s.grad("w1", 2).copy()
    labels = np.arange(3, dtype=np.int32) % 10
    loss2 = s.train_step(labels)
    assert abs(loss2 - loss) <= 1e-6 * abs(loss)
    assert np.allclose(s.grad("w1", 2), g1, rtol=1e-5, atol=1e-9)


def test_train_errors():
    batch = db.Batch.generate("chain", batch=2, vocab=10, width=F, length=4, branch_prob=0.0, seed=3)
    s = db.IepSession(batch, 5, db.MODULE_RESBLOCK)
    with pytest.raises(db.DynbatchError):
        s.train_step(np.zeros(2, np.int32))  # training off
    s.set_training(True)
    with pytest.raises(db.DynbatchError):
        s.train_step(np.zeros(2, np.int32))  # no head
    s.set_head(4, 0)
    with pytest.raises(db.DynbatchError):
        s.train_step(np.array([0, 4], np.int32))  # label out of range
    assert s.grad("w0", 2).size == 0  # a unary function has no conv1x1
    with pytest.raises(db.DynbatchError):
        s.grad("w1", 0)  # function 0 is a leaf: no weights


def test_train_step_is_schedule_invariant():
    """The improved, standard and naive schedules batch the backward
    differently (the paper's comparison) but differentiate the same
    function: the forward is bit-identical across schedules, the gradients
    agree up to summation order."""
    kw = dict(batch=5, vocab=10, width=F, length=6, branch_prob=0.4, seed=9)
    labels = np.arange(5, dtype=np.int32) % 10
    grads = {}
    for strategy in ("improved", "standard", "naive"):
        s = db.IepSession(db.Batch.generate("chain", **kw), 77, db.MODULE_RESBLOCK)
        if strategy == "standard":
            s.set_strategy("standard")
        elif strategy == "naive":
            s.set_schedule(db.Batch.generate("chain", **dict(kw, width=8)).schedule("naive"))
        s.set_head(10, 3)
        s.set_training(True)
        loss = s.train_step(labels)
        grads[strategy] = (loss, s.grad("w1", 2), s.grad("head_w1"), s.grad("inputs"))
    base = grads["improved"]
    for strategy in ("standard", "naive"):
        other = grads[strategy]
        assert other[0] == base[0]  # bit-identical forward → identical loss
        for a, b in zip(other[1:], base[1:]):
            assert fro_err(a, b) <= 1e-5, strategy


def test_train_step_at_cfg1_size():
    """The training step on BASELINE's cfg1 minibatch (64 chain programs of
    up to 16 nodes, p = 40, branch_prob 0.1: 14 steps, 232 expensive calls)
    against torch fp64 autograd, same bars as the deeper programs above."""
    s, loss, ref_loss, mod, head, dx = _run("chain", 64, 40, 4, 16, 0.1, 0, answers=28)
    worst = _check_all(s, loss, ref_loss, mod, head, dx)
    assert worst <= TOL_FRO


def test_sgd_update_descends_by_the_first_order_prediction():
    """One SGD step with the device gradients lowers the loss by ≈ lr·‖g‖²
    (the first-order prediction, over every module and head parameter), and
    a few steps keep lowering it: the update, the rebuilt fp16 operand
    layouts and the gradients agree with each other."""
    kw = dict(batch=6, vocab=10, width=F, length=6, branch_prob=0.4, seed=21)
    s = db.IepSession(db.Batch.generate("chain", **kw), 31, db.MODULE_RESBLOCK)
    s.set_head(10, 4)
    s.set_training(True)
    labels = np.arange(6, dtype=np.int32) % 10
    loss0 = s.train_step(labels)
    g2 = 0.0
    for f in range(1, 10):
        for name in NAMES:
            g = s.grad(name, f).astype(np.float64)
            g2 += float(np.sum(g * g))
    for name in ("head_wp", "head_bp", "head_w1", "head_b1", "head_w2", "head_b2"):
        g = s.grad(name).astype(np.float64)
        g2 += float(np.sum(g * g))
    lr = 2e-3 * loss0 / g2  # a 0.2% predicted decrease: first order dominates
    s.sgd(lr)
    loss1 = s.train_step(labels)
    predicted = lr * g2
    assert loss1 < loss0
    assert abs((loss0 - loss1) - predicted) <= 0.3 * predicted, (loss0 - loss1, predicted)
    losses = [loss1]
    for _ in range(4):
        s.sgd(0.5)
        losses.append(s.train_step(labels))
    assert losses[-1] < losses[0], losses


def test_train_step_after_set_programs_equals_fresh_session():
    """Training on programs set per call (db_iep_session_set_programs, the
    serving-loop API) gives the gradients of a session created on those
    programs: the backward's tables follow the device-built batch."""
    kw = dict(vocab=10, width=F, length=6, branch_prob=0.4)
    a = db.Batch.generate("chain", batch=5, seed=31, **kw)
    bb = db.Batch.generate("chain", batch=4, seed=32, **kw)
    toks, off = bb.prefix_tokens()
    s = db.IepSession(a, 9, db.MODULE_RESBLOCK, program_capacity=8, node_capacity=64, length_capacity=8)
    s.set_head(10, 2)
    s.set_training(True)
    s.train_step(np.arange(5, dtype=np.int32) % 10)
    s.set_programs(toks, off)
    x = np.random.default_rng(0).uniform(-1, 1, size=(4, F)).astype(np.float32)
    out = np.zeros_like(x)
    s.forward_host(x, out)  # the new programs' inputs
    labels = np.arange(4, dtype=np.int32) % 10
    loss = s.train_step(labels)
    fresh = db.IepSession(bb, 9, db.MODULE_RESBLOCK)
    fresh.set_head(10, 2)
    fresh.set_training(True)
    want_out = np.zeros_like(x)
    fresh.forward_host(x, want_out)
    loss_f = fresh.train_step(labels)
    assert np.array_equal(out, want_out)
    assert abs(loss - loss_f) <= 1e-6 * abs(loss_f)
    for name in ("w1", "b2", "head_w1"):
        got = s.grad(name, 2) if not name.startswith("head") else s.grad(name)
        ref = fresh.grad(name, 2) if not name.startswith("head") else fresh.grad(name)
        assert fro_err(got, ref) <= 1e-5, name
    assert fro_err(s.grad("inputs"), fresh.grad("inputs")) <= 1e-5
