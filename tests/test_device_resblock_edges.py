"""Tier-B edge cases through the per-call program API (db_iep_session_set_programs,
the device build of build_program_from_prefix, src/program.cpp:95-142), each
against the fp64 oracle (orc_execute kind=resblock) on the same programs and
inputs:

* single-leaf programs mixed with real ones (a leaf root's output is its
  input map, src/executor.cpp:168-173);
* a batch of leaves only (no step, no kernel beyond the layout passes);
* a 40-block unary chain (deeper than any BASELINE config: the residual
  stream must not compound the fp16 operand rounding);
* a left-deep binary spine (every block binary, one leaf per level).

Tolerances as tests/test_device_resblock.py (max-norm 1e-3, element 5e-3).
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db
from dbtest import max_norm_err

pytestmark = pytest.mark.gpu

F = 128 * 14 * 14
P = 10  # vocabulary: 0 leaf, odd binary, even unary


def _arity(f):
    return 0 if f == 0 else (2 if f % 2 else 1)


def batch_from_prefix(seqs):
    """Oracle CSR of prefix function sequences (children before parents,
    program-local ids; node order does not change the values)."""
    fid, c0, c1, off, root = [], [], [], [0], []
    for seq in seqs:
        base = len(fid)
        pos = 0

        def parse():
            nonlocal pos
            f = seq[pos]
            pos += 1
            kids = [parse() for _ in range(_arity(f))]
            fid.append(f)
            c0.append(kids[0] if kids else -1)
            c1.append(kids[1] if len(kids) > 1 else -1)
            return len(fid) - 1 - base

        root.append(parse())
        assert pos == len(seq)
        off.append(len(fid))
    i32 = lambda v: np.asarray(v, np.int32)  # noqa: E731
    return O.Batch(i32(off), i32(fid), i32(c0), i32(c1), i32(root), P)


def _run(seqs, seed=0, module_seed=5):
    toks = np.array([t for s in seqs for t in s], np.int32)
    off = np.cumsum([0] + [len(s) for s in seqs]).astype(np.int32)
    b = len(seqs)
    init = db.Batch.generate("chain", batch=2, vocab=P, width=F, length=4, branch_prob=0.3, seed=1)
    s = db.IepSession(init, module_seed, db.MODULE_RESBLOCK, program_capacity=max(b, 2),
                      node_capacity=int(off[-1]) + 8, length_capacity=max(len(q) for q in seqs))
    s.set_programs(toks, off)
    x = np.random.default_rng(seed).uniform(-1, 1, size=(b, F)).astype(np.float32)
    out = np.zeros_like(x)
    s.forward_host(x, out)
    ob = batch_from_prefix(seqs)
    r = O.execute(ob, O.schedule_improved(ob), x.astype(np.float64), module_seed, "resblock")
    assert r.rc == 0
    return x, out, r


def _check(dev, ref):
    err = max_norm_err(dev, ref)
    rms = np.sqrt(np.mean(ref ** 2))
    elem = np.max(np.abs(dev - ref) / (np.abs(ref) + rms))
    assert err <= 1e-3, err
    assert elem <= 5e-3, elem


def test_single_leaf_programs_among_real_ones():
    seqs = [[0], [2, 0], [1, 0, 0], [0], [4, 2, 6, 0], [1, 2, 0, 0], [0]]
    x, out, r = _run(seqs)
    _check(out, r.outputs)
    for e in (0, 3, 6):  # leaf roots: the input map itself
        assert np.array_equal(out[e], x[e])


def test_leaves_only_batch():
    x, out, r = _run([[0]] * 5, seed=1)
    assert np.array_equal(out, x)
    assert r.expensive_calls == 0


def test_deep_unary_chain():
    _, out, r = _run([[2, 4, 6, 8] * 10 + [0], [2] * 7 + [0]], seed=2)
    _check(out, r.outputs)


def test_left_deep_binary_spine():
    _, out, r = _run([[1, 0] * 12 + [0], [3, 0, 0]], seed=3)
    _check(out, r.outputs)


@pytest.mark.parametrize("kind", ["chain", "balanced", "dag"])
def test_empty_batch_on_both_tiers(kind):
    """0 programs: no step, empty outputs, zero counters (src/schedule.cpp:147,
    an empty batch has 0 steps)."""
    for mk, width in ((db.MODULE_RESBLOCK, F), (db.MODULE_DENSE, 8)):
        b = db.Batch.generate(kind, batch=0, vocab=P, width=width, length=4, branch_prob=0.3, seed=0)
        r = b.execute_device(5, mk)
        assert r.outputs().shape == (0, width)
        assert r.expensive_calls == 0


def test_moe_layer_rejects_an_empty_batch_like_the_reference():
    # MoeConfig::validate (src/moe.cpp:31): batch must be >= 1
    with pytest.raises(db.DynbatchError) as ei:
        db.MoeSession(8, 2, 0, 256, 256, seed=0, precision=db.MOE_FP16)
    assert "batch must be >= 1" in str(ei.value)
