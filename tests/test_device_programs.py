"""Device program build from prefix function sequences (SURVEY.md §8f item 1:
build_program_from_prefix, src/program.cpp:95-142) and per-call program
updates of a resblock session (db_iep_session_set_programs)."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db

pytestmark = pytest.mark.gpu

F = 128 * 14 * 14


def _batch(seed, b=12, length=8):
    return db.Batch.generate("chain", batch=b, vocab=10, width=F, length=length, branch_prob=0.4, seed=seed)


def _rows(b, seed):
    return np.random.default_rng(seed).uniform(-1, 1, size=(b, F)).astype(np.float32)


def test_set_programs_equals_fresh_session():
    a, bb = _batch(1), _batch(2, b=10)
    toks, off = bb.prefix_tokens()
    s = db.IepSession(a, 5, db.MODULE_RESBLOCK, program_capacity=16, node_capacity=400, length_capacity=16)
    xa = _rows(12, 0)
    out_a = np.zeros_like(xa)
    s.forward_host(xa, out_a)
    s.set_programs(toks, off)
    xb = _rows(10, 1)
    out = np.zeros_like(xb)
    s.forward_host(xb, out)
    fresh = db.IepSession(bb, 5, db.MODULE_RESBLOCK)
    want = np.zeros_like(xb)
    fresh.forward_host(xb, want)
    assert np.array_equal(out, want)
    # the device-built CSR schedules exactly like the reference
    ob = O.gen_batch("chain", 10, p=10, length=8, bp=0.4, seed=2)
    from test_device_iep import _flat_from_json
    assert _flat_from_json(s.schedule().to_json()) == O.schedule_improved(ob)
    # and back to the first programs, pipelined
    ta, oa = a.prefix_tokens()
    s.set_programs(ta, oa)
    again = np.zeros_like(xa)
    s.forward_host_async(xa, again)
    s.synchronize()
    assert np.array_equal(again, out_a)


@pytest.mark.parametrize("toks,off,code", [
    ([], [0, 0], "DB_ERR_INVALID_ARG"),               # empty sequence
    ([99], [0, 1], "DB_ERR_UNKNOWN_FUNCTION"),        # unknown function id
    ([4], [0, 1], "DB_ERR_UNDERFULL_SEQUENCE"),       # unary root without its child
    ([0, 0], [0, 2], "DB_ERR_OVERFULL_SEQUENCE"),     # token after the root closed
])
def test_set_programs_reports_reference_errors(toks, off, code):
    s = db.IepSession(_batch(3), 5, db.MODULE_RESBLOCK)
    with pytest.raises(db.DynbatchError) as ei:
        s.set_programs(np.array(toks, np.int32), np.array(off, np.int32))
        s.synchronize()
    assert code in str(ei.value)


def test_set_programs_capacity_is_enforced():
    s = db.IepSession(_batch(4, b=4), 5, db.MODULE_RESBLOCK)
    toks, off = _batch(5, b=12).prefix_tokens()
    with pytest.raises(db.DynbatchError):
        s.set_programs(toks, off)


def test_pipelined_new_programs_every_call():
    """set_programs before every forward_host_async (the sequences ride the
    call's input upload): each call's outputs equal a fresh session's for
    that call's programs and rows, and a plain forward after a staged
    set_programs builds it too."""
    batches = [_batch(s, b=8 + s) for s in range(3)]
    seqs = [b.prefix_tokens() for b in batches]
    s = db.IepSession(batches[0], 6, db.MODULE_RESBLOCK, program_capacity=16, node_capacity=400,
                      length_capacity=16)
    calls = [0, 1, 2, 1, 0, 2, 2]
    xs = [db.PinnedArray((8 + c, F), np.float32) for c in calls]
    outs = [db.PinnedArray(x.array.shape, np.float32) for x in xs]
    for i, (c, x) in enumerate(zip(calls, xs)):
        x.array[:] = _rows(8 + c, 10 + i)
    for c, x, o in zip(calls, xs, outs):
        s.set_programs(*seqs[c])
        s.forward_host_async(x.array, o.array)
    s.synchronize()
    for i, (c, x, o) in enumerate(zip(calls, xs, outs)):
        fresh = db.IepSession(batches[c], 6, db.MODULE_RESBLOCK)
        want = np.zeros((8 + c, F), np.float32)
        fresh.forward_host(x.array, want)
        assert np.array_equal(o.array, want), i
    # staged by a pipelined set_programs, built by a plain forward
    s.set_programs(*seqs[1])
    s.forward()
    s.synchronize()
    fresh = db.IepSession(batches[1], 6, db.MODULE_RESBLOCK)
    fresh.forward()
    from test_device_iep import _flat_from_json
    assert _flat_from_json(s.schedule().to_json()) == _flat_from_json(fresh.schedule().to_json())


def test_graph_cache_across_more_program_sets_than_it_holds():
    """Forwards are replayed from captured graphs, an LRU of 4 per session:
    cycling through 5 program sets (evictions and re-captures) gives each
    call exactly a fresh session's outputs, and a strategy change re-captures."""
    batches = [_batch(20 + i, b=6 + i, length=7 + i % 3) for i in range(5)]
    seqs = [b.prefix_tokens() for b in batches]
    s = db.IepSession(batches[0], 8, db.MODULE_RESBLOCK, program_capacity=16, node_capacity=400,
                      length_capacity=16)
    want = {}
    for i, b in enumerate(batches):
        fresh = db.IepSession(b, 8, db.MODULE_RESBLOCK)
        x = _rows(6 + i, 30 + i)
        y = np.zeros_like(x)
        fresh.forward_host(x, y)
        want[i] = (x, y)
    for i in [0, 1, 2, 3, 4, 0, 2, 4, 1, 3, 0]:
        s.set_programs(*seqs[i])
        x, y_want = want[i]
        y = np.zeros_like(x)
        s.forward_host(x, y)
        assert np.array_equal(y, y_want), i
    s.set_strategy("online")  # same programs, another device schedule: outputs unchanged
    x, y_want = want[0]
    y = np.zeros_like(x)
    s.forward_host(x, y)
    assert np.array_equal(y, y_want)
