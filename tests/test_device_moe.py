"""GPU parity of the MoE layer: top-k routing and the expert dispatch order
must be bit-identical to the reference (top_k_gate, group_by_function);
fp64 outputs follow the reference's arithmetic order (bit-identical up to
the last-ulp behaviour of exp() in the gate weights → tolerance 1e-12)."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.max(np.abs(a - b) / np.maximum(np.maximum(np.abs(a), np.abs(b)), 1e-300)))


def test_cfg4_routing_fingerprint(golden):
    fp, _ = golden
    g = fp["moe"]["cfg4"]
    s = db.MoeSession(g["n"], g["k"], g["T"], 8, 8, seed=0, precision=db.MOE_FP64)
    s.forward()
    ids, w, off, items = s.routing()
    assert "%016x" % O.fnv1a64(ids.astype(np.int32).tobytes()) == g["routing_fnv"]
    counts = np.diff(off)
    assert (counts.min(), counts.max()) == (g["rows_min"], g["rows_max"])
    # dispatch order = group_by_function: per expert, (token, slot) ascending
    exp_items = np.argsort(ids.ravel(), kind="stable")
    assert np.array_equal(items, exp_items.astype(np.int32))
    _, ref_w = O.topk(O.moe_inputs(g["T"], g["n"], 1, 0)[1], g["k"], use_ref=True)
    assert np.max(np.abs(w - ref_w)) <= 1e-15


def test_cfg5_routing_slice(golden):
    fp, _ = golden
    g = fp["moe"]["cfg5_slice"]
    s = db.MoeSession(g["n"], g["k"], g["T"], 8, 8, seed=0, precision=db.MOE_FP64)
    s.forward()
    ids, _, off, _ = s.routing()
    assert "%016x" % O.fnv1a64(ids.astype(np.int32).tobytes()) == g["routing_fnv"]


@pytest.mark.parametrize("n,k,T,d,h", [(64, 2, 256, 64, 96), (32, 4, 64, 8, 8),
                                       (1024, 8, 300, 16, 24), (5, 5, 40, 12, 7)])
def test_moe_fp64_matches_reference(n, k, T, d, h):
    run = db.moe_run(n, k, T, d, h, seed=7, batched=True)
    xi, sc = O.moe_inputs(T, n, d, 7)
    ids, w = O.topk(sc, k, use_ref=True)
    ref, trace, _ = O.moe_forward(xi, ids, w, n, h, O.mix_seed(7, 0xe4be27), use_ref=True)
    out = run.outputs()
    assert _rel(out, ref) <= 1e-12
    assert run.expensive_calls == trace[0] and run.peak_group_rows == trace[1]


def test_moe_naive_equals_batched_and_counts():
    """tests/test_capi.cpp:167-200 through the ABI."""
    naive = db.moe_run(32, 4, 64, 8, 8, seed=7, batched=False)
    batched = db.moe_run(32, 4, 64, 8, 8, seed=7, batched=True)
    assert naive.expensive_calls == 256
    assert batched.expensive_calls <= 32
    assert np.array_equal(naive.outputs(), batched.outputs())


def test_moe_committed_fixture(golden):
    _, arr = golden
    run = db.moe_run(64, 2, 512, 64, 96, seed=7, batched=True)
    assert _rel(run.outputs(), arr["moe_small_out"]) <= 1e-12


def test_topk_ties():
    # all scores equal → lowest ids win (test_moe.cpp:92-111 style)
    s = db.MoeSession(16, 3, 8, 4, 4, seed=1, precision=db.MOE_FP64)
    s.forward()
    ids, w, _, _ = s.routing()
    xi, sc = O.moe_inputs(8, 16, 4, 1)
    rid, rw = O.topk(sc, 3, use_ref=True)
    assert np.array_equal(ids, rid)


@pytest.mark.parametrize("n,k,T,d,h", [(64, 2, 2048, 256, 512), (16, 4, 300, 256, 256),
                                       (8, 1, 100, 512, 256), (40, 3, 777, 256, 768)])
def test_moe_bf16_matches_reference(n, k, T, d, h):
    """bf16 grouped tcgen05 GEMMs vs the fp64 reference arithmetic.
    Routing (ids, dispatch order) stays bit-exact; outputs within the stated
    bf16 tolerance max|a-b|/max|ref| <= 2e-2."""
    from dbtest import max_norm_err
    s = db.MoeSession(n, k, T, d, h, seed=5, precision=db.MOE_BF16)
    s.forward()
    out = s.run().outputs()
    xi, sc = O.moe_inputs(T, n, d, 5)
    ids, w = O.topk(sc, k)
    ref, trace, _ = O.moe_forward(xi, ids, w, n, h, O.mix_seed(5, 0xe4be27))
    dev_ids, dev_w, off, items = s.routing()
    assert np.array_equal(dev_ids, ids)
    assert np.array_equal(items, np.argsort(ids.ravel(), kind="stable").astype(np.int32))
    err = max_norm_err(out, ref)
    assert err <= 2e-2, err


def test_moe_forward_host_async_pipeline_equals_sync_calls():
    """Pipelined host calls (three in flight, per-call device slots, copies
    on their own streams) give exactly the synchronous calls' outputs."""
    n, k, T, d, h = 16, 2, 512, 256, 256
    s = db.MoeSession(n, k, T, d, h, seed=3, precision=db.MOE_FP16)
    rng = np.random.default_rng(1)
    calls = 5
    xs = [db.PinnedArray((T, d), np.float32) for _ in range(calls)]
    scs = [db.PinnedArray((T, n), np.float64) for _ in range(calls)]
    outs = [db.PinnedArray((T, d), np.float32) for _ in range(calls)]
    for x, sc in zip(xs, scs):
        x.array[:] = rng.uniform(-1, 1, size=(T, d)).astype(np.float32)
        sc.array[:] = rng.uniform(-1, 1, size=(T, n))
    for x, sc, o in zip(xs, scs, outs):
        s.forward_host_async(x.array, sc.array, o.array)
    s.synchronize()
    want = np.zeros((T, d), np.float32)
    for x, sc, o in zip(xs, scs, outs):
        s.forward_host(x.array, sc.array, want)
        assert np.array_equal(o.array, want)
