"""Pins the CPU oracle (oracle/dynbatch_oracle.c) against the reference:
committed golden fixtures (tests/golden, generated from the compiled
reference by tests/golden/make_golden.py) and, when oracle/_ref is present,
the compiled reference itself on fresh seeds."""
import ctypes as C
import re

import numpy as np
import pytest

import oracle_lib as O
from golden.make_golden import IEP, sched_fnv

needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


def test_mt19937_64_known_answer():
    # The C++ standard fixes the 10000th output of a default-seeded mt19937_64.
    buf = C.create_string_buffer(312 * 8 + 16)
    O.oracle().orc_rng_seed(buf, C.c_uint64(5489))
    for _ in range(9999):
        O.oracle().orc_rng_u64(buf)
    assert O.oracle().orc_rng_u64(buf) == 9981545732273789042


@pytest.mark.parametrize("name", list(IEP))
def test_schedule_fingerprints(golden, name):
    fp, _ = golden
    c = IEP[name]
    bt = O.gen_batch(c["kind"], c["b"], p=c["p"], depth=c["depth"], length=c["length"],
                     bp=c["bp"], seed=0)
    g = fp["iep"][name]
    assert bt.n_nodes == g["nodes"]
    fs = O.schedule_improved(bt)
    gi = g["improved"]
    assert (fs.n_steps, fs.n_groups, fs.expensive_calls()) == (gi["steps"], gi["groups"],
                                                                 gi["expensive_calls"])
    assert sched_fnv(fs) == gi["sched_fnv"]
    if bt.n_nodes < 20000:
        assert "%016x" % O.fnv1a64(O.schedule_json(fs).encode()) == gi["json_fnv"]
    x = O.random_batch(bt.b, 128, O.mix_seed(0, 0x1127))
    assert "%016x" % O.fnv1a64(x.tobytes()) == g["inputs_fnv_w128"]
    lab, dmax = O.labels(bt)
    assert dmax == g["d_max"] and fs.n_steps == dmax + 1


def test_schedule_json_golden_string():
    """tests/test_serialize.cpp:69-110 golden dump for two [2, 0] programs."""
    src = open("/root/reference/proj/tests/test_serialize.cpp").read() if __import__("os").path.exists(
        "/root/reference/proj/tests/test_serialize.cpp") else None
    bt = O.Batch(np.array([0, 2, 4], np.int32), np.array([2, 0, 2, 0], np.int32),
                 np.array([1, -1, 1, -1], np.int32), np.array([-1] * 4, np.int32),
                 np.array([0, 0], np.int32), 4)
    text = O.schedule_json(O.schedule_improved(bt))
    assert text.startswith('{\n  "steps": [\n    [\n      {\n        "function_id": 0,')
    assert text.endswith('  ],\n  "strategy": "improved"\n}')
    if src:
        exp = re.search(r'const std::string expected = R"\((.*?)\)";', src, re.S).group(1)
        assert text == exp


def test_dense_execute_matches_reference_fixture(golden):
    _, arr = golden
    bt = O.gen_batch("chain", 64, p=40, length=16, bp=0.1, seed=0)
    x = O.random_batch(64, 128, O.mix_seed(0, 0x1127))
    r = O.execute(bt, O.schedule_improved(bt), x, O.mix_seed(0, 0xd00d), "dense", width=128)
    assert r.rc == 0
    assert np.array_equal(r.outputs, arr["dense_cfg1_w128_out"])  # bit-exact fp64
    assert [r.expensive_calls, r.peak_group_rows, r.steps] == arr["dense_cfg1_w128_trace"].tolist()
    bt2 = O.gen_batch("dag", 24, p=12, length=12, bp=0.5, seed=3)
    x2 = O.random_batch(24, 32, O.mix_seed(3, 0x1127))
    r2 = O.execute(bt2, O.schedule_improved(bt2), x2, 99, "dense", width=32)
    assert np.array_equal(r2.outputs, arr["dense_dag_w32_out"])


def test_moe_matches_reference_fixture(golden):
    fp, arr = golden
    T, n, k, d, h = 512, 64, 2, 64, 96
    xi, sc = O.moe_inputs(T, n, d, 7)
    ids, w = O.topk(sc, k)
    assert np.array_equal(ids, arr["moe_small_ids"])
    assert np.array_equal(w, arr["moe_small_w"])
    out, trace, _ = O.moe_forward(xi, ids, w, n, h, O.mix_seed(7, 0xe4be27))
    assert np.array_equal(out, arr["moe_small_out"])
    assert trace[0] <= n


def test_moe_routing_fingerprint_cfg4(golden):
    fp, _ = golden
    g = fp["moe"]["cfg4"]
    _, s = O.moe_inputs(g["T"], g["n"], 1, 0)
    assert "%016x" % O.fnv1a64(s.tobytes()) == g["scores_fnv"]
    ids, w = O.topk(s, g["k"])
    assert "%016x" % O.fnv1a64(ids.astype(np.int32).tobytes()) == g["routing_fnv"]
    assert "%016x" % O.fnv1a64(w.tobytes()) == g["weights_fnv"]
    counts = np.bincount(ids.ravel(), minlength=g["n"])
    assert (counts.min(), counts.max()) == (g["rows_min"], g["rows_max"])


def test_topk_tie_break():
    """test_moe.cpp:92-111: ties go to the lower expert id; -0.0 ties +0.0."""
    s = np.array([[0.5, 0.5, 0.1, 0.5], [0.0, -0.0, 0.3, -1.0]])
    ids, w = O.topk(s, 2)
    assert ids.tolist() == [[0, 1], [2, 0]]
    assert np.allclose(w.sum(1), 1.0)


@needs_ref
@pytest.mark.parametrize("seed", [1, 2, 5])
@pytest.mark.parametrize("kind", ["chain", "balanced", "dag"])
def test_oracle_vs_reference_fresh_seeds(kind, seed):
    bt = O.gen_batch(kind, 37, p=11, depth=4, length=13, bp=0.4, seed=seed)
    rb = O.ref_gen_batch(kind, 37, p=11, depth=4, length=13, bp=0.4, seed=seed)
    for f in ("prog_off", "fid", "child0", "child1", "root"):
        assert np.array_equal(getattr(bt, f), getattr(rb, f))
    fs = O.schedule_improved(bt)
    assert fs == O.ref_schedule(rb, "improved")
    x = O.random_batch(bt.b, 16, seed)
    a = O.execute(bt, fs, x, seed * 7, "dense", width=16)
    r = O.ref_execute(rb, x, 16, seed * 7)
    assert np.array_equal(a.outputs, r.outputs)
    assert np.array_equal(a.per_function_calls, r.per_function_calls)
    assert (a.expensive_calls, a.peak_group_rows, a.steps) == (r.expensive_calls,
                                                               r.peak_group_rows, r.steps)


def test_resblock_oracle_properties():
    """Tier B (parity unpinned): weights reproducible, row independence, and
    a zero-weight-free sanity: unary block output is >= 0 and finite."""
    a = O.resblock_weights(1, 8, 5, 2)
    b = O.resblock_weights(1, 8, 5, 2)
    assert all(np.array_equal(u, v) for u, v in zip(a, b))
    bt = O.gen_batch("chain", 3, p=6, length=5, bp=0.5, seed=1)
    fs = O.schedule_improved(bt)
    x = O.random_batch(3, 8 * 5 * 5, 11)
    r = O.execute(bt, fs, x, 3, "resblock", C=8, H=5, W=5)
    assert r.rc == 0 and np.all(np.isfinite(r.outputs)) and np.all(r.outputs >= 0)
    # row independence: program 1 alone gives the same bits
    sub = O.Batch(np.array([0, bt.prog_off[2] - bt.prog_off[1]], np.int32),
                  bt.fid[bt.prog_off[1]:bt.prog_off[2]].copy(),
                  bt.child0[bt.prog_off[1]:bt.prog_off[2]].copy(),
                  bt.child1[bt.prog_off[1]:bt.prog_off[2]].copy(), bt.root[1:2].copy(), 6)
    r1 = O.execute(sub, O.schedule_improved(sub), x[1:2], 3, "resblock", C=8, H=5, W=5)
    assert np.array_equal(r1.outputs[0], r.outputs[1])


def test_bench_seed_helper_matches_the_reference_mix_seed():
    """bench.py derives the module seed with its own mix_seed (no oracle
    import on the product path); it must equal the reference's."""
    import bench
    for seed, stream in ((0, 0xd00d), (7, 0x1127), (123456789, 0xe4be27)):
        assert bench._mix_seed(seed, stream) == O.mix_seed(seed, stream)


def test_random_rows_equals_random_batch_rows():
    x = O.random_batch(700, 333, 11)
    rows = [0, 1, 2, 300, 311, 312, 699]
    assert np.array_equal(O.random_rows(rows, 333, 11), x[rows])


def test_moe_sampled_tokens_equal_full_forward():
    """tests/moe_full.reference_tokens (sampled tokens, per-expert numpy fp64)
    agrees with the restated moe_forward_batched on every token."""
    import moe_full as M
    n, k, T, d, h, seed = 12, 3, 90, 16, 24, 4
    xi, sc = O.moe_inputs(T, n, d, seed)
    ids, w = O.topk(sc, k)
    ref, _, _ = O.moe_forward(xi, ids, w, n, h, O.mix_seed(seed, 0xe4be27))
    toks = M.sample_tokens(T, 17)
    sids, sw, out = M.reference_tokens(n, k, d, h, seed, toks)
    assert np.array_equal(sids, ids[toks]) and np.array_equal(sw, w[toks])
    assert np.max(np.abs(out - ref[toks])) <= 1e-12


@needs_ref
@pytest.mark.parametrize("kind,seed", [("chain", 1), ("balanced", 2), ("dag", 3)])
def test_naive_schedule_equals_reference(kind, seed):
    """oracle_lib.schedule_naive (the bench's CPU naive leg) is the reference's
    schedule_naive (src/schedule.cpp:94-105), step for step."""
    bt = O.gen_batch(kind, 12, p=16, depth=4, length=10, bp=0.3, seed=seed)
    assert O.schedule_naive(bt) == O.ref_schedule(bt, "naive")
