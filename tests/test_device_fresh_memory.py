"""Sessions created over freed, non-zero device memory report no stale error.

The IEP and MoE sessions' device error words are read by synchronize()
(and by time(), which synchronizes first) before the first forward resets
them; they are cleared at creation. Here the memory a session is likely to
get back from cudaMalloc is first filled with ones and released."""
import numpy as np
import pytest
import torch

import paper_1707_02402_b200 as db

pytestmark = pytest.mark.gpu

F = 128 * 14 * 14


def _dirty_and_release(mib=512):
    x = torch.full((mib << 18,), -1, dtype=torch.int32, device="cuda:0")
    torch.cuda.synchronize()
    del x
    torch.cuda.empty_cache()


@pytest.mark.parametrize("round_", range(3))
def test_iep_session_over_dirty_memory(round_):
    _dirty_and_release()
    b = db.Batch.generate("chain", batch=8, vocab=10, width=F, length=6, branch_prob=0.3, seed=round_)
    s = db.IepSession(b, 3, db.MODULE_RESBLOCK)
    s.synchronize()
    s.time(1)
    want = b.execute_device(3, db.MODULE_RESBLOCK).outputs()
    assert np.array_equal(s.run().outputs(), want)


def test_moe_session_after_destroyed_iep_session():
    """The bench's order: IEP sessions (hundreds of small bias / table
    allocations holding non-zero bytes) are destroyed, then a MoE session's
    time() synchronizes before its first gate."""
    b = db.Batch.generate("chain", batch=64, vocab=40, width=F, length=16, branch_prob=0.1, seed=0)
    for _ in range(2):
        x = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
        x.forward()
        x.synchronize()
        del x
        s = db.MoeSession(64, 2, 4096, 1024, 1024, seed=0, precision=db.MOE_FP16)
        s.time(1)
        s.synchronize()
        del s


@pytest.mark.parametrize("round_", range(3))
def test_moe_session_over_dirty_memory(round_):
    _dirty_and_release()
    s = db.MoeSession(8, 2, 256, 256, 256, seed=round_, precision=db.MOE_FP16)
    s.time(1)
    s.forward()
    s.synchronize()
