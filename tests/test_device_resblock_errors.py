"""The reference executor's error semantics on the Tier-B (resblock) path
(ADVICE r1 device.cpp:488 / :368).

* a schedule that reads a node before it is written raises MissingOperand
  (src/executor.cpp:48-51) → DB_ERR_MISSING_OPERAND;
* a schedule that writes a node twice raises SingleAssignmentViolation
  (:62-65) → DB_ERR_INTERNAL (src/c_api.cpp:38-60);
  both exactly as the compiled reference reports for the same injected
  faults (db_schedule_inject_fault, src/c_api.cpp:201-221);
* non-finite inputs (:107) or module outputs (:156-159) raise
  NonFiniteValue → DB_ERR_NON_FINITE; so do values beyond the fp16
  operand range of the conv kernels (|x| > 65504), which the reference
  would carry in fp64;
* a host schedule set after a pipelined set_programs describes the new
  programs and is kept;
* a session created where a destroyed one lived reports no stale error
  (its error word is cleared at creation, not first at the forward).
"""
import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db

pytestmark = pytest.mark.gpu

F = 128 * 14 * 14


def _batch(seed=2, b=4):
    return db.Batch.generate("chain", batch=b, vocab=10, width=F, length=8, branch_prob=0.3, seed=seed)


@pytest.mark.parametrize("fault,status,name", [("dependency-order", 7, "MissingOperand"),
                                               ("duplicate", 12, "SingleAssignmentViolation")])
@pytest.mark.parametrize("strategy", ["standard", "improved", "naive"])
def test_broken_schedules_raise_reference_errors_resblock(fault, status, name, strategy):
    b = _batch()
    s = b.schedule(strategy)
    s.inject_fault(fault)
    with pytest.raises(db.DynbatchError) as ei:
        b.execute_device(1, db.MODULE_RESBLOCK, schedule=s)
    assert ei.value.status == status and name in ei.value.message
    # the same fault on the dense path (device presence bitmap) gives the same status
    bd = db.Batch.generate("chain", batch=4, vocab=10, width=8, length=8, branch_prob=0.3, seed=2)
    sd = bd.schedule(strategy)
    sd.inject_fault(fault)
    with pytest.raises(db.DynbatchError) as ed:
        bd.execute_device(1, db.MODULE_DENSE, schedule=sd)
    assert ed.value.status == status


def test_valid_host_schedule_still_runs_after_checks():
    b = _batch(seed=3)
    want = b.execute_device(5, db.MODULE_RESBLOCK).outputs()
    got = b.execute_device(5, db.MODULE_RESBLOCK, schedule=b.schedule("naive")).outputs()
    assert np.array_equal(got, want)


@pytest.mark.parametrize("bad,status", [(np.inf, 9), (np.nan, 9), (-1e5, 9)])
def test_non_finite_or_out_of_range_inputs_raise(bad, status):
    b = _batch(seed=4, b=3)
    s = db.IepSession(b, 7, db.MODULE_RESBLOCK)
    x = O.random_batch(3, F, O.mix_seed(4, 0x1127)).astype(np.float32)
    out = np.zeros((3, F), np.float32)
    s.forward_host(x, out)  # clean inputs: fine
    x[1, 1234] = bad
    with pytest.raises(db.DynbatchError) as ei:
        s.forward_host(x, out)
    assert ei.value.status == status and "NonFiniteValue" in ei.value.message
    x[1, 1234] = 0.5
    s.forward_host(x, out)  # the error state does not stick


def test_schedule_after_pipelined_set_programs_is_kept():
    b1, b2 = _batch(seed=5, b=6), _batch(seed=6, b=6)
    t2, o2 = b2.prefix_tokens()
    s = db.IepSession(b1, 9, db.MODULE_RESBLOCK, program_capacity=6, node_capacity=int(max(
        b1.prefix_tokens()[1][-1], o2[-1])), length_capacity=16)
    x = b2.inputs().astype(np.float32)
    out = np.zeros((6, F), np.float32)
    s.forward_host_async(x, out)  # creates the pipeline
    s.synchronize()
    s.set_programs(t2, o2)        # staged (pipelined)
    s.set_schedule(b2.schedule("naive"))
    s.forward_host(x, out)
    assert s.schedule().to_json() == b2.schedule("naive").to_json()
    want = b2.execute_device(9, db.MODULE_RESBLOCK).outputs()
    assert np.array_equal(out.astype(np.float64), want)


def test_new_session_after_destroyed_session_has_no_stale_error():
    """time() synchronizes (and reads the error word) before its first
    forward; the word was once left as cudaMalloc returned it, so a session
    allocated over a freed one's bias vector raised 'device executor error
    <bias bits>' (profiles/stale_error_check.py '00')."""
    b = db.Batch.generate("chain", batch=64, vocab=40, width=F, length=16, branch_prob=0.1, seed=0)
    sched = db.Batch.generate("chain", batch=64, vocab=40, width=8, length=16, branch_prob=0.1, seed=0).schedule("naive")
    ref = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
    ref.forward()
    want = ref.run().outputs()
    for _ in range(3):
        x = db.IepSession(b, 1234, db.MODULE_RESBLOCK, first=0, last=64)
        x.set_schedule(sched)
        x.time(1)
        x.time(2)
        assert np.array_equal(x.run().outputs(), want)
        del x
