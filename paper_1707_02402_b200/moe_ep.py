"""Expert-parallel MoE over torch.distributed.

Tokens are sharded T/G per rank, and experts n/G per rank, both contiguous.
A rank's assignments, stably sorted by expert in (token, slot) order (the
reference group_by_function, src/schedule.cpp:166-169 via
src/moe.cpp:214-224), are then already grouped by destination rank. One
forward is:

  dispatch  gate → sort → rows packed in sorted order       (device kernels)
  exchange  all-to-all of per-expert counts, all-to-allv of the rows
  experts   scatter by (local expert, source rank) → grouped GEMMs → unpack
  exchange  reverse all-to-allv (outputs back to their senders)
  combine   slot-order weighted sum                          (device kernels)

Receivers concatenate by source rank. With contiguous token shards this
reproduces, for every expert, the reference's (token, slot) member order.
On the B200 the whole forward, both exchanges included, runs inside the
library (MoeEp::forward, db_moe_ep_forward): grouped ncclSend/ncclRecv
on its own NCCL communicator, planned by make_ep_plan. `MoeEpLayer` is the
thin wrapper over it. `EpExchange` and the plan helpers below restate the
same protocol over torch.distributed; the CPU tests run it on gloo with
world 2 against the oracle, and check db_moe_ep_plan against `pieces`.

With `chunks` > 1 the exchange overlaps the expert GEMMs:
the local experts are cut into contiguous ranges, and each range's rows
travel in their own batch of point-to-point sends/receives. The GEMMs of
range c start as soon as range c has arrived, while later ranges are still
in flight. Range c's outputs start back while range c+1 computes. Both
buffers keep the unchunked layout. A send block is [destination q][q's
local expert e], and a receive block is [source r][local expert e]. The
pieces of a range are therefore contiguous slices of both, and the results
are bit-identical to chunks = 1.
"""
from __future__ import annotations

import numpy as np


def split_rows(expert_counts: np.ndarray, world: int) -> np.ndarray:
    """Rows this rank sends to each rank: the contiguous expert blocks."""
    return np.asarray(expert_counts, np.int64).reshape(world, -1).sum(axis=1)


def chunk_bounds(E: int, chunks: int):
    """Contiguous local-expert ranges [(e0, e1), ...], as even as possible."""
    chunks = max(1, min(int(chunks), E))
    cuts = [E * c // chunks for c in range(chunks + 1)]
    return [(cuts[c], cuts[c + 1]) for c in range(chunks)]


def pieces(cnt2d: np.ndarray, bounds):
    """Slices of a [peer][local expert] row-block buffer: off[c][q], rows[c][q]
    for expert range c of peer q (cnt2d[q][e] = rows of (q, e))."""
    cnt2d = np.asarray(cnt2d, np.int64)
    G = cnt2d.shape[0]
    peer0 = np.concatenate([[0], np.cumsum(cnt2d.sum(axis=1))])[:-1]
    pre = np.concatenate([np.zeros((G, 1), np.int64), np.cumsum(cnt2d, axis=1)], axis=1)
    off = np.stack([peer0 + pre[:, e0] for e0, _ in bounds])
    rows = np.stack([pre[:, e1] - pre[:, e0] for e0, e1 in bounds])
    return off, rows


class EpExchange:
    """The two exchange steps of one expert-parallel forward."""

    def __init__(self, world: int, n_experts: int, device="cpu", group=None):
        import torch
        self.torch = torch
        self.world, self.n = world, n_experts
        self.E = n_experts // world
        self.device = device
        self.group = group

    def counts(self, expert_counts: np.ndarray) -> np.ndarray:
        """recv[src][e] = rows source `src` sends for local expert e."""
        if self.world == 1:
            return np.asarray(expert_counts, np.int32).reshape(1, self.E)
        import torch.distributed as dist
        t = self.torch
        send = t.as_tensor(np.asarray(expert_counts, np.int32), device=self.device)
        recv = t.empty_like(send)
        dist.all_to_all_single(recv, send, group=self.group)  # equal splits of n/G counts
        return recv.cpu().numpy().reshape(self.world, self.E)

    def rows(self, out, inp, out_rows, in_rows):
        """all-to-allv of row blocks: inp (in_rows[q] rows to rank q) → out."""
        if self.world == 1:
            rows = int(np.sum(in_rows))
            out[:rows].copy_(inp[:rows])
            return out
        import torch.distributed as dist
        dist.all_to_all_single(out[: int(np.sum(out_rows))], inp[: int(np.sum(in_rows))],
                               [int(x) for x in out_rows], [int(x) for x in in_rows], group=self.group)
        return out

    def pieces_async(self, out, out_off, out_rows, inp, in_off, in_rows, rank):
        """One chunk: rows inp[in_off[q] : +in_rows[q]] go to rank q, rows
        from rank q land at out[out_off[q] : +out_rows[q]]. The own piece
        is a local copy. Returns the works to wait on (one grouped batch of
        point-to-point operations; none when nothing crosses ranks)."""
        a, n = int(in_off[rank]), int(in_rows[rank])
        if n:
            b = int(out_off[rank])
            out[b:b + n].copy_(inp[a:a + n])
        if self.world == 1:
            return []
        import torch.distributed as dist
        ops = []
        for q in range(self.world):
            if q == rank:
                continue
            if int(in_rows[q]):
                a = int(in_off[q])
                ops.append(dist.P2POp(dist.isend, inp[a:a + int(in_rows[q])], q, group=self.group))
            if int(out_rows[q]):
                b = int(out_off[q])
                ops.append(dist.P2POp(dist.irecv, out[b:b + int(out_rows[q])], q, group=self.group))
        return dist.batch_isend_irecv(ops) if ops else []


class MoeEpLayer:
    """One rank of the expert-parallel MoE layer on the B200: a thin wrapper
    over the library's db_moe_ep_* session, whose forward runs gate, sort,
    both NCCL exchanges (counts and rows, chunked by expert range and
    overlapped with the grouped tcgen05 GEMMs) and the combine in C++
    (MoeEp::forward). torch.distributed only carries the 128-byte NCCL id
    from rank 0 to the others.

    At world 1 the layer is one device pass (no exchange); `loopback=True`
    still builds a one-rank NCCL communicator so the exchange path runs (tests)."""

    def __init__(self, experts, k, batch, data_dim, hidden, seed=0, group=None, precision=None, loopback=False):
        import torch.distributed as dist

        from . import MOE_FP16, MoeEpSession, moe_ep_nccl_id
        precision = MOE_FP16 if precision is None else precision
        init = dist.is_available() and dist.is_initialized()
        self.rank = dist.get_rank(group) if init else 0
        self.world = dist.get_world_size(group) if init else 1
        self.sess = MoeEpSession(experts, k, batch, data_dim, hidden, seed, self.rank, self.world, precision)
        self.stream = self.sess.stream
        if self.world > 1 or loopback:
            box = [moe_ep_nccl_id() if self.rank == 0 else None]
            if self.world > 1:
                dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0, group=group)
            self.sess.comm_init(box[0])

    def forward(self, chunks: int = 1):
        self.sess.forward(chunks)

    @property
    def last_recv_rows(self) -> int:
        return self.sess.recv_rows

    def outputs(self) -> np.ndarray:
        return self.sess.outputs()
