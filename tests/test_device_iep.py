"""GPU parity: device scheduler and Tier-A dense executor vs the reference.

Schedules and labels must be bit-identical to the reference
(schedule_improved / max_root_distance_labels); dense outputs are fp64 with
the reference's fused-multiply-add order, so they must be bit-identical too.
Golden fingerprints (tests/golden) pin the BASELINE configs; the compiled
reference (oracle/_ref, prebuilt, travels with the repo) checks fresh seeds.
"""
import json

import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db
from golden.make_golden import IEP, sched_fnv

pytestmark = pytest.mark.gpu


def _flat_from_json(text):
    """FlatSchedule from our schedule_to_json text."""
    d = json.loads(text)
    sgb, gf, gmo, me, mn = [0], [], [0], [], []
    for step in d["steps"]:
        for g in step:
            gf.append(g["function_id"])
            for e, n in g["members"]:
                me.append(e)
                mn.append(n)
            gmo.append(len(me))
        sgb.append(len(gf))
    a = lambda x: np.array(x, np.int32)
    return O.FlatSchedule(a(sgb), a(gf), a(gmo), a(me), a(mn), d["strategy"])


WK = {"chain": "chain", "balanced": "balanced", "dag": "dag"}


@pytest.mark.parametrize("name", list(IEP))
def test_device_improved_schedule_matches_golden(golden, name):
    fp, _ = golden
    c = IEP[name]
    b = db.Batch.generate(WK[c["kind"]], batch=c["b"], vocab=c["p"], width=8, depth=c["depth"],
                          length=c["length"], branch_prob=c["bp"], seed=0)
    s = b.schedule("improved")
    fs = _flat_from_json(s.to_json())
    g = fp["iep"][name]["improved"]
    assert (fs.n_steps, fs.n_groups, fs.expensive_calls()) == (g["steps"], g["groups"],
                                                                 g["expensive_calls"])
    assert sched_fnv(fs) == g["sched_fnv"]
    s.verify(b)


@pytest.mark.parametrize("strategy", ["standard", "online"])
@pytest.mark.parametrize("name", list(IEP))
def test_device_standard_online_schedules_match_golden(golden, name, strategy):
    """§8f item 2: standard (postorder columns) and online (ready rounds =
    node heights) from the device scheduler, pinned to the compiled
    reference's schedule_to_json fingerprints."""
    fp, _ = golden
    c = IEP[name]
    b = db.Batch.generate(WK[c["kind"]], batch=c["b"], vocab=c["p"], width=8, depth=c["depth"],
                          length=c["length"], branch_prob=c["bp"], seed=0)
    s = b.schedule_device(strategy)
    fs = _flat_from_json(s.to_json())
    g = fp["iep"][name][strategy]
    assert (fs.n_steps, fs.n_groups, fs.expensive_calls()) == (g["steps"], g["groups"],
                                                                 g["expensive_calls"])
    assert sched_fnv(fs) == g["sched_fnv"]
    assert fs.strategy == strategy
    s.verify(b)


@pytest.mark.parametrize("strategy", ["improved", "standard", "online"])
@pytest.mark.parametrize("kind,seed", [("chain", 3), ("dag", 4), ("balanced", 5), ("dag", 11)])
def test_device_schedules_equal_host_builders(kind, seed, strategy):
    b = db.Batch.generate(kind, batch=37, vocab=9, width=4, depth=4, length=11, branch_prob=0.5, seed=seed)
    want = b.schedule(strategy).to_json()
    assert b.schedule_device(strategy).to_json() == want
    # a session's per-forward device scheduler with that strategy
    sess = db.IepSession(b, 3)
    sess.set_strategy(strategy)
    sess.forward()
    assert sess.schedule().to_json() == want


def test_device_naive_strategy_is_rejected():
    b = db.Batch.generate("chain", batch=4, vocab=9, width=4, length=6, branch_prob=0.5, seed=1)
    with pytest.raises(db.DynbatchError):
        b.schedule_device("naive")
    with pytest.raises(db.DynbatchError):
        db.IepSession(b, 3).set_strategy("naive")


@pytest.mark.parametrize("seed", [0, 1, 7])
@pytest.mark.parametrize("kind", ["chain", "balanced", "dag"])
def test_device_schedule_and_labels_match_reference_fresh_seeds(kind, seed):
    b = db.Batch.generate(kind, batch=300, vocab=17, width=4, depth=5, length=20,
                          branch_prob=0.35, seed=seed)
    ob = O.gen_batch(kind, 300, p=17, depth=5, length=20, bp=0.35, seed=seed)
    sess = db.IepSession(b, 1)
    sess.forward()
    sess.synchronize()
    fs = _flat_from_json(sess.schedule().to_json())
    assert fs == O.schedule_improved(ob)
    lab, _ = O.labels(ob)
    assert np.array_equal(sess.labels(ob.n_nodes), lab)


def test_device_schedule_empty_and_single_node_programs():
    text = json.dumps({"vocab": [{"id": 0, "arity": 0, "cost": "free"},
                                 {"id": 1, "arity": 2, "cost": "expensive"},
                                 {"id": 2, "arity": 1, "cost": "expensive"}],
                       "programs": [[0], [2, 0], [1, 0, 2, 0], [0]]})
    b = db.Batch.from_json(text, 4, 3)
    s = b.schedule("improved")
    s.verify(b)
    assert s.step_count() == 3
    d = json.loads(s.to_json())
    assert d["steps"][0] == [{"function_id": 0, "members": [[2, 3]]}]


@pytest.mark.parametrize("width", [8, 128])
@pytest.mark.parametrize("strategy", ["improved", "naive", "standard", "online"])
def test_dense_execute_bit_exact_vs_reference(strategy, width):
    b = db.Batch.generate("chain", batch=64, vocab=40, width=width, length=16, branch_prob=0.1,
                          seed=0)
    run = b.execute(b.schedule(strategy), 12345)
    ob, x = O.ref_gen_batch("chain", 64, p=40, width=width, length=16, bp=0.1, seed=0,
                            with_inputs=True)
    r = O.ref_execute(ob, x, width, 12345, strategy)
    assert np.array_equal(run.outputs(), r.outputs)
    assert run.expensive_calls == r.expensive_calls
    assert run.peak_group_rows == r.peak_group_rows
    tr = json.loads(run.trace_json())
    assert len(tr["per_step_seconds"]) == r.steps


def test_dense_matches_committed_reference_fixture(golden):
    _, arr = golden
    b = db.Batch.generate("chain", batch=64, vocab=40, width=128, length=16, branch_prob=0.1,
                          seed=0)
    ms = O.mix_seed(0, 0xd00d)
    run = b.execute(b.schedule("improved"), ms)
    assert np.array_equal(run.outputs(), arr["dense_cfg1_w128_out"])
    run2 = b.execute_device(ms, db.MODULE_DENSE)  # device scheduler, no host schedule
    assert np.array_equal(run2.outputs(), arr["dense_cfg1_w128_out"])


@pytest.mark.parametrize("kind", ["dag", "balanced"])
def test_dense_dag_and_balanced_bit_exact(kind):
    b = db.Batch.generate(kind, batch=48, vocab=12, width=32, depth=5, length=12,
                          branch_prob=0.5, seed=3)
    run = b.execute_device(99, db.MODULE_DENSE)
    ob, x = O.ref_gen_batch(kind, 48, p=12, width=32, depth=5, length=12, bp=0.5, seed=3,
                            with_inputs=True)
    assert np.array_equal(run.outputs(), O.ref_execute(ob, x, 32, 99).outputs)


def test_dense_width_1024_bit_exact():
    b = db.Batch.generate("chain", batch=16, vocab=10, width=1024, length=8, branch_prob=0.3,
                          seed=4)
    run = b.execute_device(5, db.MODULE_DENSE)
    ob, x = O.ref_gen_batch("chain", 16, p=10, width=1024, length=8, bp=0.3, seed=4,
                            with_inputs=True)
    assert np.array_equal(run.outputs(), O.ref_execute(ob, x, 1024, 5).outputs)


def test_broken_schedules_raise_reference_errors():
    b = db.Batch.generate("chain", batch=4, vocab=10, width=8, length=10, branch_prob=0.0, seed=2)
    s = b.schedule("standard")
    s.inject_fault("dependency-order")
    with pytest.raises(db.DynbatchError) as ei:
        b.execute(s, 1)
    assert ei.value.status == 7 and "MissingOperand" in ei.value.message
    s2 = b.schedule("standard")
    s2.inject_fault("duplicate")
    with pytest.raises(db.DynbatchError) as ei:
        b.execute(s2, 1)
    assert ei.value.status == 12


def test_row_independence_and_batch_alone_equality():
    """tests/test_executor.cpp:98-170: a row computes to the same bits alone."""
    b = db.Batch.generate("chain", batch=512, vocab=16, width=16, length=12, branch_prob=0.3,
                          seed=8)
    full = b.execute_device(77, db.MODULE_DENSE).outputs()
    sess = db.IepSession(b, 77, db.MODULE_DENSE, first=100, last=101)
    sess.forward()
    one = sess.run().outputs()
    assert np.array_equal(one[0], full[100])


def test_verify_suite_passes_on_device():
    st, lines = db.verify_run(seeds=12, batch=6, vocab=9, length=10, width=8, seed=0)
    assert st == 0, lines
    st, lines = db.verify_run(seeds=8, batch=5, vocab=9, length=10, width=8, seed=1, parallel=True)
    assert st == 0, lines
