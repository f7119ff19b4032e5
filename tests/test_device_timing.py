"""Session timing modes (db_iep_session_time): profile 2 times the fused step
kernel with event-record nodes inside the replayed CUDA graph, in the same
loop as the headline; profile 1 puts events around every direct launch."""
import numpy as np
import pytest

import paper_1707_02402_b200 as db

pytestmark = pytest.mark.gpu

F = 128 * 14 * 14


def test_step_kernel_events_inside_graph_replays():
    b = db.Batch.generate("chain", batch=48, vocab=10, width=F, length=8, branch_prob=0.3, seed=4)
    s = db.IepSession(b, 7, db.MODULE_RESBLOCK)
    want = b.execute_device(7, db.MODULE_RESBLOCK).outputs()
    s.time(2)
    ms, kt = s.time(5, profile=2)
    assert kt.launches[4] == 5
    assert 0.0 < kt.ms[4] <= ms
    _, kp = s.time(5, profile=1)
    assert kp.launches[4] == 5
    assert kt.flops[4] == pytest.approx(kp.flops[4], rel=1e-12)
    # the graph with event nodes is a separate cache entry; plain forwards
    # and a second profile-2 loop (new events on the same exec) still agree
    ms2, kt2 = s.time(3, profile=2)
    assert kt2.launches[4] == 3 and 0.0 < kt2.ms[4] <= ms2
    assert np.array_equal(s.run().outputs(), want)


def test_no_step_events_when_the_forward_is_several_launches():
    # children shared by several parents: one step launch per step with
    # gathers between them, so there is no single kernel to bracket
    b = db.Batch.generate("dag", batch=6, vocab=9, width=F, depth=4, length=8, branch_prob=0.5, seed=3)
    s = db.IepSession(b, 7, db.MODULE_RESBLOCK)
    ms, kt = s.time(2, profile=2)
    assert ms > 0.0
    assert kt.launches[4] in (0, 2)  # 2 only if this batch happens to share no child
