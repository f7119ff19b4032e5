"""GPU parity of the IEP classifier head (head.cu and the
grouped tcgen05 GEMM with bias, fp16 operands, fp32 accumulation and
logits) against the fp64 oracle (orc_head_forward, pinned to torch fp64 in
tests/test_oracle_head.py). Stated tolerance: max|dev − ref| / max|ref| ≤
1e-3, on the device's own root maps (the head alone) and end to end through
db_iep_session_forward_logits_host (module blocks + head)."""
import numpy as np
import pytest

import oracle_lib as O
import paper_1707_02402_b200 as db
from dbtest import max_norm_err

pytestmark = pytest.mark.gpu

F = 128 * 14 * 14
TOL = 1e-3


def test_head_on_device_roots_matches_oracle():
    batch = db.Batch.generate("chain", batch=6, vocab=10, width=F, length=6, branch_prob=0.4, seed=1)
    s = db.IepSession(batch, 77, db.MODULE_RESBLOCK)
    s.forward()
    roots = s.run().outputs()
    s.set_head(28, 5)
    s.head_forward()
    got = s.logits(6)
    ref = O.head_forward(roots, 28, 5)
    err = max_norm_err(got.astype(np.float64), ref)
    assert err <= TOL, err


def test_head_end_to_end_matches_oracle():
    b = 8
    batch = db.Batch.generate("chain", batch=b, vocab=12, width=F, length=8, branch_prob=0.3, seed=4)
    s = db.IepSession(batch, 31, db.MODULE_RESBLOCK)
    s.set_head(10, 9)
    x = O.random_batch(b, F, O.mix_seed(4, 0x1127)).astype(np.float32)
    logits = np.zeros((b, 10), np.float32)
    s.forward_logits_host(x, logits)
    ob = O.gen_batch("chain", b, p=12, length=8, bp=0.3, seed=4)
    roots = O.execute(ob, O.schedule_improved(ob), x.astype(np.float64), 31, "resblock").outputs
    ref = O.head_forward(roots, 10, 9)
    err = max_norm_err(logits.astype(np.float64), ref)
    assert err <= TOL, err


def test_head_many_row_tiles_sampled():
    """300 programs: 58,800 projection rows (230 row tiles over the CTA
    pairs) and 3 FC row tiles (padded to a pair); 12 sampled programs."""
    b = 300
    batch = db.Batch.generate("chain", batch=b, vocab=40, width=F, length=6, branch_prob=0.3, seed=7)
    s = db.IepSession(batch, 3, db.MODULE_RESBLOCK)
    s.forward()
    roots = s.run().outputs()
    s.set_head(28, 2)
    s.head_forward()
    got = s.logits(b)
    pick = np.linspace(0, b - 1, 12).astype(int)
    ref = O.head_forward(roots[pick], 28, 2)
    err = max_norm_err(got[pick].astype(np.float64), ref)
    assert err <= TOL, err
    assert np.all(np.isfinite(got))


def test_head_leaf_root_reads_the_input_map():
    """A program that is a single leaf: its root map is the example's input."""
    batch = db.Batch.generate("chain", batch=2, vocab=10, width=F, length=4, branch_prob=0.0, seed=3)
    s = db.IepSession(batch, 5, db.MODULE_RESBLOCK, program_capacity=2, node_capacity=64,
                      length_capacity=16)
    s.set_head(12, 1)
    s.set_programs(np.array([0, 2, 0], np.int32), np.array([0, 1, 3], np.int32))  # [leaf], [unary(leaf)]
    x = O.random_batch(2, F, 17).astype(np.float32)
    logits = np.zeros((2, 12), np.float32)
    s.forward_logits_host(x, logits)
    ref0 = O.head_forward(x[:1].astype(np.float64), 12, 1)
    assert max_norm_err(logits[:1].astype(np.float64), ref0) <= TOL


def test_head_errors():
    batch = db.Batch.generate("chain", batch=2, vocab=10, width=16, length=4, branch_prob=0.0, seed=3)
    dense = db.IepSession(batch, 5, db.MODULE_DENSE)
    with pytest.raises(db.DynbatchError):
        dense.set_head(10, 0)
    rb = db.Batch.generate("chain", batch=2, vocab=10, width=F, length=4, branch_prob=0.0, seed=3)
    s = db.IepSession(rb, 5, db.MODULE_RESBLOCK)
    with pytest.raises(db.DynbatchError):
        s.head_forward()
    with pytest.raises(db.DynbatchError):
        s.set_head(0, 0)
    with pytest.raises(db.DynbatchError):
        s.set_head(257, 0)
