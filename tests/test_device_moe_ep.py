"""GPU parity of the expert-parallel MoE stages (db_moe_ep_*) on one B200.

G ranks are stood in for by G sessions in one process, run stage by stage.
The all-to-alls are concatenations of the row blocks on the device, and no
kernel of one session waits on another. Every rank's outputs must be
bit-identical to the single-GPU tensor-core layer (MoeSession, same precision) on the same token
slice: each output row depends only on its own row of the grouped GEMMs,
whichever rank or tile computes it.
"""
import numpy as np
import pytest

import paper_1707_02402_b200 as db
from paper_1707_02402_b200.moe_ep import split_rows

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _loopback(n, k, T, d, h, seed, G, chunks=0, precision=db.MOE_FP16):
    dev = torch.device("cuda", 0)
    sess = [db.MoeEpSession(n, k, T, d, h, seed, r, G, precision) for r in range(G)]
    E = n // G
    send = [torch.empty((s.items, d), dtype=torch.float16, device=dev) for s in sess]
    counts = [s.dispatch(send[r].data_ptr()) for r, s in enumerate(sess)]  # synchronises
    starts = [np.concatenate([[0], np.cumsum(split_rows(c, G))]) for c in counts]
    recv, cnts = [], []
    for q in range(G):
        recv.append(torch.cat([send[r][starts[r][q]:starts[r][q + 1]] for r in range(G)]).contiguous())
        cnts.append(np.stack([counts[r].reshape(G, E)[q] for r in range(G)]).astype(np.int32))
    torch.cuda.synchronize()
    rets = []
    for q in range(G):
        ret = torch.empty_like(recv[q])
        if chunks:  # layout once, then contiguous expert ranges (chunked exchange)
            from paper_1707_02402_b200.moe_ep import chunk_bounds
            sess[q].layout(cnts[q])
            for e0, e1 in reversed(chunk_bounds(E, chunks)):  # any order: ranges are independent
                sess[q].experts_range(recv[q].data_ptr(), ret.data_ptr(), e0, e1)
        else:
            sess[q].experts(recv[q].data_ptr(), cnts[q], ret.data_ptr())
        sess[q].synchronize()
        rets.append(ret)
    outs = []
    for r in range(G):
        blocks = []
        for q in range(G):
            off = int(cnts[q][:r].sum())
            blocks.append(rets[q][off:off + int(cnts[q][r].sum())])
        back = torch.cat(blocks).contiguous()
        assert back.shape[0] == sess[r].items
        sess[r].combine(back.data_ptr())
        outs.append(sess[r].outputs())
    return outs, cnts


@pytest.mark.parametrize("G,precision", [(1, db.MOE_FP16), (2, db.MOE_FP16), (4, db.MOE_FP16), (8, db.MOE_FP16),
                                         (2, db.MOE_BF16)])
def test_ep_stages_equal_single_gpu_layer(G, precision):
    n, k, T, d, h, seed = 16, 2, 1024, 256, 512, 5
    outs, cnts = _loopback(n, k, T, d, h, seed, G, precision=precision)
    full = db.MoeSession(n, k, T, d, h, seed=seed, precision=precision)
    full.forward()
    ref = full.run().outputs()
    Tl = T // G
    for r in range(G):
        np.testing.assert_array_equal(outs[r], ref[r * Tl:(r + 1) * Tl].astype(np.float32))
    assert sum(int(c.sum()) for c in cnts) == T * k


@pytest.mark.parametrize("G,chunks", [(1, 3), (2, 2), (4, 2), (2, 8)])
def test_ep_expert_ranges_equal_whole_experts_call(G, chunks):
    """layout + experts_range over contiguous expert ranges (the chunked
    exchange's receive side) = one experts() call, bit for bit."""
    n, k, T, d, h, seed = 16, 2, 1024, 256, 512, 5
    whole, _ = _loopback(n, k, T, d, h, seed, G)
    ranged, _ = _loopback(n, k, T, d, h, seed, G, chunks=chunks)
    for a, b in zip(whole, ranged):
        np.testing.assert_array_equal(a, b)


def test_ep_counts_follow_reference_routing():
    """Counts a rank sends per expert = its token slice's routing."""
    import oracle_lib as O
    n, k, T, d, h, seed, G = 16, 2, 512, 256, 256, 9, 4
    x, s = O.moe_inputs(T, n, d, seed)
    ids, _ = O.topk(s, k)
    sess = [db.MoeEpSession(n, k, T, d, h, seed, r, G) for r in range(G)]
    Tl = T // G
    for r, se in enumerate(sess):
        buf = torch.empty((se.items, d), dtype=torch.float16, device="cuda")
        c = se.dispatch(buf.data_ptr())
        np.testing.assert_array_equal(c, np.bincount(ids[r * Tl:(r + 1) * Tl].reshape(-1), minlength=n))


@pytest.mark.parametrize("precision", [db.MOE_FP16, db.MOE_BF16])
def test_moe_ep_layer_world1_equals_session(precision):
    from paper_1707_02402_b200.moe_ep import MoeEpLayer
    n, k, T, d, h, seed = 16, 2, 1024, 256, 512, 11
    layer = MoeEpLayer(n, k, T, d, h, seed, precision=precision)
    layer.forward()
    out = layer.outputs()
    full = db.MoeSession(n, k, T, d, h, seed=seed, precision=precision)
    full.forward()
    np.testing.assert_array_equal(out, full.run().outputs().astype(np.float32))


@pytest.mark.parametrize("chunks", [1, 3, 16])
def test_moe_ep_forward_through_nccl_loopback(chunks):
    """MoeEp::forward with a one-rank NCCL communicator: the count exchange,
    the host plan, the chunked row exchange (ncclSend/ncclRecv to self), the
    per-range GEMMs and the return exchange all run, and the outputs are the
    one-pass layer's bit for bit."""
    from paper_1707_02402_b200.moe_ep import MoeEpLayer
    n, k, T, d, h, seed = 16, 2, 1024, 256, 512, 11
    want = MoeEpLayer(n, k, T, d, h, seed)
    want.forward()
    layer = MoeEpLayer(n, k, T, d, h, seed, loopback=True)
    for _ in range(2):  # twice: buffers and events are reused
        layer.forward(chunks)
        np.testing.assert_array_equal(layer.outputs(), want.outputs())
    assert layer.last_recv_rows == T * k


def test_ep_rejects_indivisible_shapes():
    with pytest.raises(db.DynbatchError):
        db.MoeEpSession(10, 2, 1024, 256, 256, 0, 0, 4)
