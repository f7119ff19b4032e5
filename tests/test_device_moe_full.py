"""MoE at the BASELINE shapes.

* fp16 tensor-core mode (DB_MOE_FP16) — the precise mode: max|dev − ref| /
  max|ref| ≤ 1e-3 (the north star's figure) against fp64 reference
  arithmetic, at small shapes on every token and at cfg4 / cfg5 on sampled
  tokens (tests/moe_full.py);
* bf16 (DB_MOE_BF16) — the labelled wide-range mode, ≤ 2e-2;
* full-T cfg5 routing (T = 1,048,576, n = 1024, k = 4): the routing
  fingerprint and the per-expert row range from the compiled reference
  (tests/golden/make_golden.py cfg5), dispatch order = stable argsort.
"""
import numpy as np
import pytest

import moe_full as M
import oracle_lib as O
import paper_1707_02402_b200 as db

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,k,T,d,h", [(64, 2, 2048, 256, 512), (16, 4, 300, 256, 256),
                                       (8, 1, 100, 512, 256), (40, 3, 777, 256, 768)])
def test_moe_fp16_matches_reference(n, k, T, d, h):
    s = db.MoeSession(n, k, T, d, h, seed=5, precision=db.MOE_FP16)
    s.forward()
    out = s.outputs()
    xi, sc = O.moe_inputs(T, n, d, 5)
    ids, w = O.topk(sc, k)
    ref, _, _ = O.moe_forward(xi, ids, w, n, h, O.mix_seed(5, 0xe4be27))
    dev_ids, _, _, items = s.routing()
    assert np.array_equal(dev_ids, ids)
    assert np.array_equal(items, np.argsort(ids.ravel(), kind="stable").astype(np.int32))
    assert M.max_norm(out, ref) <= M.TOL_FP16


@pytest.mark.parametrize("precision,tol", [(db.MOE_FP16, M.TOL_FP16), (db.MOE_BF16, M.TOL_BF16)])
def test_cfg4_full_shape_sampled_tokens(precision, tol):
    c = M.CFG["cfg4"]
    s = db.MoeSession(c["n"], c["k"], c["T"], c["d"], c["h"], seed=0, precision=precision)
    s.forward()
    toks = M.sample_tokens(c["T"], 512)
    ids, w, ref = M.reference_tokens(c["n"], c["k"], c["d"], c["h"], 0, toks)
    dev_ids, dev_w, _, _ = s.routing()
    assert np.array_equal(dev_ids[toks], ids)
    assert np.max(np.abs(dev_w[toks] - w)) <= 1e-15
    err = M.max_norm(s.outputs(toks), ref)
    assert err <= tol, err


def test_cfg5_full_shape_routing_and_sampled_tokens(golden):
    """The whole 1,048,576-token cfg5 layer on one B200 (fp16 mode): routing
    pinned to the compiled reference over all tokens, outputs of 96 sampled
    tokens (≈384 experts on their true rows) against fp64."""
    fp, _ = golden
    c = M.CFG["cfg5"]
    g = fp["moe"]["cfg5"]
    assert (g["T"], g["n"], g["k"]) == (c["T"], c["n"], c["k"])
    s = db.MoeSession(c["n"], c["k"], c["T"], c["d"], c["h"], seed=0, precision=db.MOE_FP16)
    s.forward()
    ids, w, off, items = s.routing()
    assert "%016x" % O.fnv1a64(ids.astype(np.int32).tobytes()) == g["routing_fnv"]
    counts = np.diff(off)
    assert (counts.min(), counts.max()) == (g["rows_min"], g["rows_max"])
    assert np.count_nonzero(counts) == g["occupied"]
    assert np.array_equal(items, np.argsort(ids.ravel(), kind="stable").astype(np.int32))
    st = s.stats()
    assert st.expensive_calls == g["occupied"] and st.peak_group_rows == g["rows_max"]
    toks = M.sample_tokens(c["T"], 96)
    rids, _, ref = M.reference_tokens(c["n"], c["k"], c["d"], c["h"], 0, toks)
    assert np.array_equal(ids[toks], rids)
    err = M.max_norm(s.outputs(toks), ref)
    assert err <= M.TOL_FP16, err
