"""CPU tests of the product library: it loads, exports every declared symbol,
and its host logic (fixtures, program graphs, host-built schedules, JSON,
verification, fault injection, error mapping) matches the reference. No
compute runs here; device entry points must fail loudly without a GPU."""
import json

import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db
from dbtest import gpu_available, header_symbols

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_library_exports_every_declared_symbol():
    names = header_symbols()
    assert len(names) >= 27 + 20
    lib = db.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert len(header_symbols(("dynbatch.h",))) == 27


@needs_ref
def test_reference_header_declares_same_27_entry_points():
    import re
    text = open("/root/reference/proj/include/dynbatch/dynbatch.h").read()
    ref = set(re.findall(r"DYNBATCH_API[^;]*?\b(db_\w+)\s*\(", text, re.S))
    ours = set(n for n in header_symbols())
    assert ref <= ours


def test_version_and_null_arguments():
    L = db.lib()
    assert L.db_version()
    assert L.db_batch_generate(None, None) == 1
    assert len(db.last_error()) > 0
    assert L.db_schedule_step_count(None) == -1
    assert L.db_run_expensive_calls(None) == -1
    assert L.db_run_total_seconds(None) == -1.0


@pytest.mark.parametrize("kind,kw", [("chain", dict(batch=64, length=16, branch_prob=0.1)),
                                     ("balanced", dict(batch=32, depth=5)),
                                     ("dag", dict(batch=40, length=12, branch_prob=0.5))])
def test_generated_batches_match_reference_generator(kind, kw):
    b = db.Batch.generate(kind, vocab=40, width=8, seed=3, **kw)
    ob = O.gen_batch(kind, kw["batch"], p=40, depth=kw.get("depth", 4),
                     length=kw.get("length", 16), bp=kw.get("branch_prob", 0.1), seed=3)
    st = b.stats()
    assert st.total_nodes == ob.n_nodes
    assert st.expensive_nodes == int(np.count_nonzero(ob.fid != 0))
    if kind != "dag":  # prefix sequences are the program for trees
        progs = json.loads(b.to_json())["programs"]
        for e, seq in enumerate(progs):
            assert seq == ob.fid[ob.prog_off[e]:ob.prog_off[e + 1]].tolist()


def test_stats_fields():
    b = db.Batch.generate("chain", batch=16, vocab=10, width=8, length=10, branch_prob=0.2, seed=5)
    st = b.stats()
    assert (st.batch, st.vocab, st.width) == (16, 10, 8)
    assert st.d_max < st.s_max and 0 < st.expensive_nodes < st.total_nodes


@pytest.mark.parametrize("strategy", ["naive", "standard", "online"])
@pytest.mark.parametrize("kind", ["chain", "dag", "balanced"])
def test_host_schedules_match_reference(strategy, kind):
    b = db.Batch.generate(kind, batch=24, vocab=12, width=4, depth=4, length=12,
                          branch_prob=0.4, seed=9)
    s = b.schedule(strategy)
    s.verify(b)
    ob = O.gen_batch(kind, 24, p=12, depth=4, length=12, bp=0.4, seed=9)
    if O.ref_available():
        fs = O.ref_schedule(ob, strategy)
    else:
        pytest.skip("needs oracle/_ref for host strategies")
    assert s.to_json() == O.schedule_json(fs)
    assert s.step_count() == fs.n_steps
    assert s.expensive_calls(b) == fs.expensive_calls()


def test_wire_format_and_round_trip():
    text = json.dumps({"vocab": [{"id": 0, "arity": 0, "cost": "free"},
                                 {"id": 1, "arity": 2, "cost": "expensive"},
                                 {"id": 2, "arity": 1, "cost": "expensive"}],
                       "programs": [[1, 0, 2, 0], [0]]})
    b = db.Batch.from_json(text, 8, 1)
    st = b.stats()
    assert st.batch == 2 and st.total_nodes == 5 and st.s_max == 4
    back = json.loads(b.to_json())
    assert back["programs"] == [[1, 0, 2, 0], [0]]
    assert back["vocab"][1] == {"arity": 2, "cost": "expensive", "id": 1}
    b2 = db.Batch.generate("chain", batch=6, vocab=8, width=4, length=9, branch_prob=0.3, seed=2)
    b3 = db.Batch.from_json(b2.to_json(), 4, 1)
    s2, s3 = b2.stats(), b3.stats()
    assert (s2.total_nodes, s2.expensive_nodes, s2.s_max, s2.d_max) == \
        (s3.total_nodes, s3.expensive_nodes, s3.s_max, s3.d_max)


@pytest.mark.parametrize("text,status", [("not json", 10), ('{"vocab": []}', 10),
                                         ('{"vocab": [{"id": 0, "arity": 0, "cost": "free"}], '
                                          '"programs": [[7]]}', 2),
                                         ('{"vocab": [{"id": 0, "arity": 0, "cost": "cheap"}], '
                                          '"programs": [[0]]}', 10),
                                         ('{"vocab": [{"id": 0, "arity": 0, "cost": "free"}, '
                                          '{"id": 1, "arity": 1, "cost": "expensive"}], '
                                          '"programs": [[1]]}', 3),
                                         ('{"vocab": [{"id": 0, "arity": 0, "cost": "free"}], '
                                          '"programs": [[0, 0]]}', 4)])
def test_malformed_json_statuses(text, status):
    with pytest.raises(db.DynbatchError) as ei:
        db.Batch.from_json(text, 4, 1)
    assert ei.value.status == status
    assert len(ei.value.message) > 0


def test_fault_injection_names_the_violation():
    b = db.Batch.generate("chain", batch=4, vocab=10, width=8, length=10, branch_prob=0.0, seed=2)
    s = b.schedule("standard")
    s.verify(b)
    s.inject_fault("dependency-order")
    with pytest.raises(db.DynbatchError) as ei:
        s.verify(b)
    assert ei.value.status == 11 and "DependencyOrderViolation" in ei.value.message
    s2 = b.schedule("standard")
    s2.inject_fault("duplicate")
    with pytest.raises(db.DynbatchError) as ei:
        s2.verify(b)
    assert "DuplicateExecution" in ei.value.message
    with pytest.raises(db.DynbatchError) as ei:
        s2.inject_fault("nonsense")
    assert ei.value.status == 1


def test_memory_model():
    m = db.moe_memory_model(10000, 100, 2048, 2048, 1e6)
    assert m.param_count == 83886080000
    assert abs(m.memory_ratio - 7.3) <= 0.05
    assert m.activation_count == pytest.approx(6.144e11)
    with pytest.raises(db.DynbatchError) as ei:
        db.moe_memory_model(0, 1, 1, 1, 0.0)
    assert ei.value.status == 1


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_device_paths_fail_loudly_without_gpu():
    b = db.Batch.generate("chain", batch=4, vocab=10, width=8, length=10, seed=1)
    with pytest.raises(db.DynbatchError) as ei:
        b.schedule("improved")
    assert ei.value.status == 12 and "CUDA" in ei.value.message
    s = b.schedule("naive")
    with pytest.raises(db.DynbatchError) as ei:
        b.execute(s, 1)
    assert ei.value.status == 12
    with pytest.raises(db.DynbatchError):
        db.moe_run(8, 2, 16, 4, 4)


def test_moe_argument_errors_are_shape_or_arg():
    with pytest.raises(db.DynbatchError) as ei:
        db.moe_run(32, 64, 64, 8, 8, seed=7)  # k > n
    assert ei.value.status == 1
