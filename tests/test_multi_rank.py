"""Multi-rank host logic on CPU (gloo, world_size 2): data-parallel program
shards and MoE token shards are bit-identical to the corresponding rows of
the single-process batch, cover it exactly once, and the bench's
max-over-ranks reduction picks the slowest rank. The IEP path has no
data-path collective, so this is the whole N>1 contract that
can be checked without GPUs."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_lib as O

WORLD = 2
PER = 24


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, port, kind, out_q):
    import json
    import torch
    import paper_1707_02402_b200 as db
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    b = db.Batch.generate_range(rank * PER, (rank + 1) * PER, kind, batch=PER * WORLD, vocab=12,
                                width=16, depth=4, length=10, branch_prob=0.3, seed=7)
    progs = json.loads(b.to_json())["programs"]
    x = b.inputs()
    # max-over-ranks timing as bench.Dist.max does it (gloo on CPU here)
    t = torch.tensor([float(rank + 1) * 1.5])
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    gathered = [None] * WORLD
    dist.all_gather_object(gathered, (rank, progs, x.tobytes(), x.shape))
    if rank == 0:
        out_q.put((gathered, float(t.item())))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["chain", "balanced", "dag"])
def test_program_shards_equal_full_batch_rows(kind):
    import json
    import paper_1707_02402_b200 as db
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, kind, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = db.Batch.generate(kind, batch=PER * WORLD, vocab=12, width=16, depth=4, length=10,
                             branch_prob=0.3, seed=7)
    full_progs = json.loads(full.to_json())["programs"]
    full_x = full.inputs()
    assert tmax == 3.0
    seen = []
    for rank, progs, xb, shape in sorted(gathered, key=lambda g: g[0]):
        assert progs == full_progs[rank * PER:(rank + 1) * PER]
        x = np.frombuffer(xb, dtype=np.float64).reshape(shape)
        assert np.array_equal(x, full_x[rank * PER:(rank + 1) * PER])
        seen += list(range(rank * PER, (rank + 1) * PER))
    assert seen == list(range(PER * WORLD))
    # the oracle agrees with the product on the same rows
    ob = O.gen_batch(kind, PER * WORLD, p=12, depth=4, length=10, bp=0.3, seed=7)
    assert np.array_equal(full_x, O.random_batch(PER * WORLD, 16, O.mix_seed(7, 0x1127)))
    assert ob.n_nodes == full.stats().total_nodes


def test_moe_token_shards_cover_batch():
    """MoE token shards [r·T, (r+1)·T) of gen_moe_inputs rows (the slicing the
    MoE session applies) reproduce the full generator's rows."""
    T, n, d = 40, 8, 4
    xi, sc = O.moe_inputs(T * WORLD, n, d, 3)
    for r in range(WORLD):
        xr, sr = xi[r * T:(r + 1) * T], sc[r * T:(r + 1) * T]
        ids_r, _ = O.topk(sr, 2)
        ids_full, _ = O.topk(sc, 2)
        assert np.array_equal(ids_r, ids_full[r * T:(r + 1) * T])
        assert xr.shape == (T, d)


# ----------------------------------------------- expert-parallel MoE (§8e)
EP = dict(n=8, k=2, T=64, d=16, h=24, seed=3)


def _ep_worker(rank, port, out_q):
    """One rank of the expert-parallel protocol (moe_ep.EpExchange over
    gloo) with numpy stand-ins for the device stages: gate + stable sort +
    pack, count / row all-to-alls, local experts in receive order, reverse
    all-to-allv, slot-order combine."""
    import torch
    from paper_1707_02402_b200.moe_ep import EpExchange, split_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    n, k, T, d, h, seed = (EP[key] for key in ("n", "k", "T", "d", "h", "seed"))
    expert_seed = O.mix_seed(seed, 0xe4be27)
    x_all, s_all = O.moe_inputs(T, n, d, seed)
    Tl, E = T // WORLD, n // WORLD
    sl = slice(rank * Tl, (rank + 1) * Tl)
    ids, w = O.topk(s_all[sl], k)
    items = np.argsort(ids.reshape(-1), kind="stable")  # per-expert (token, slot) order
    counts = np.bincount(ids.reshape(-1), minlength=n).astype(np.int32)
    send = torch.tensor(x_all[sl][items // k])
    gid = torch.tensor((items + rank * Tl * k).astype(np.float64)[:, None])  # global item ids
    ex = EpExchange(WORLD, n)
    cnt = ex.counts(counts)
    recv_rows, send_rows = cnt.sum(axis=1), split_rows(counts, WORLD)
    recv = torch.empty((int(recv_rows.sum()), d), dtype=torch.float64)
    ex.rows(recv, send, recv_rows, send_rows)
    rgid = torch.empty((int(recv_rows.sum()), 1), dtype=torch.float64)
    ex.rows(rgid, gid, recv_rows, send_rows)
    # local experts over the receive buffer: source blocks in rank order,
    # expert-major inside each block
    ret = torch.empty_like(recv)
    members = {e: [] for e in range(E)}
    pos = 0
    for src in range(WORLD):
        for e in range(E):
            c = int(cnt[src, e])
            w1, w2 = O.expert_weights(d, h, expert_seed, rank * E + e)
            rows = recv[pos:pos + c].numpy()
            ret[pos:pos + c] = torch.tensor(np.maximum(rows @ w1, 0.0) @ w2)
            members[e] += rgid[pos:pos + c, 0].numpy().astype(np.int64).tolist()
            pos += c
    back = torch.empty_like(send)
    ex.rows(back, ret, send_rows, recv_rows)
    pos_of_item = np.empty(Tl * k, np.int64)
    pos_of_item[items] = np.arange(Tl * k)
    y = back.numpy()[pos_of_item].reshape(Tl, k, d)
    out = np.zeros((Tl, d))
    for s in range(k):  # slot order, as the reference combine
        out += w[:, s:s + 1] * y[:, s]
    out_q.put((rank, out, members, cnt))
    dist.barrier()
    dist.destroy_process_group()


def test_moe_expert_parallel_protocol_matches_single_process():
    n, k, T, d, h, seed = (EP[key] for key in ("n", "k", "T", "d", "h", "seed"))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = dict((r, (o, m, c)) for r, o, m, c in (q.get(timeout=120) for _ in range(WORLD)))
    for p in procs:
        p.join(timeout=60)
    x_all, s_all = O.moe_inputs(T, n, d, seed)
    ids, w = O.topk(s_all, k)
    ref, _, _ = O.moe_forward(x_all, ids, w, n, h, O.mix_seed(seed, 0xe4be27))
    Tl, E = T // WORLD, n // WORLD
    flat = ids.reshape(-1)
    for r in range(WORLD):
        out, members, cnt = res[r]
        # outputs: the rank's token slice of the single-process layer
        np.testing.assert_allclose(out, ref[r * Tl:(r + 1) * Tl], rtol=1e-10, atol=1e-12)
        # member order of every local expert = the reference's (token, slot) order
        for e in range(E):
            want = np.nonzero(flat == r * E + e)[0].tolist()
            assert members[e] == want, (r, e)
        assert cnt.sum() == sum(len(v) for v in members.values())


def _ep_chunk_worker(rank, port, out_q):
    """The chunked exchange (moe_ep.pieces / EpExchange.pieces_async) moves
    exactly the rows of the single all-to-allv, range by range, both ways."""
    import torch
    from paper_1707_02402_b200.moe_ep import EpExchange, chunk_bounds, pieces, split_rows
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    n, d = 12, 3
    E = n // WORLD
    rng = np.random.default_rng(100 + rank)
    counts = rng.integers(0, 5, size=n).astype(np.int32)
    counts[rank] = 0  # an empty (destination, expert) piece
    items = int(counts.sum())
    send = torch.tensor(rank * 1000.0 + np.arange(items * d, dtype=np.float64).reshape(items, d))
    ex = EpExchange(WORLD, n)
    cnt = ex.counts(counts)
    recv_rows, send_rows = cnt.sum(axis=1), split_rows(counts, WORLD)
    full = torch.zeros((int(recv_rows.sum()), d), dtype=torch.float64)
    ex.rows(full, send, recv_rows, send_rows)
    ok = []
    for chunks in (1, 2, 4, E):
        bounds = chunk_bounds(E, chunks)
        s_off, s_rows = pieces(counts.reshape(WORLD, E), bounds)
        r_off, r_rows = pieces(cnt, bounds)
        recv = torch.full_like(full, -1.0)
        for c in range(len(bounds)):
            for w in ex.pieces_async(recv, r_off[c], r_rows[c], send, s_off[c], s_rows[c], rank):
                w.wait()
        # outputs = received rows negated; back through the reverse pieces
        ret = -recv
        back = torch.full_like(send, 7.0)
        for c in range(len(bounds)):
            for w in ex.pieces_async(back, s_off[c], s_rows[c], ret, r_off[c], r_rows[c], rank):
                w.wait()
        ok.append((chunks, bool(torch.equal(recv, full)), bool(torch.equal(back, -send))))
    out_q.put((rank, ok))
    dist.barrier()
    dist.destroy_process_group()


def test_moe_chunked_exchange_equals_all_to_allv():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ep_chunk_worker, args=(r, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(WORLD)]
    for p in procs:
        p.join(timeout=60)
    for rank, ok in res:
        for chunks, same_recv, same_back in ok:
            assert same_recv and same_back, (rank, chunks)


def test_chunk_bounds_and_pieces():
    from paper_1707_02402_b200.moe_ep import chunk_bounds, pieces
    assert chunk_bounds(8, 3) == [(0, 2), (2, 5), (5, 8)]
    assert chunk_bounds(2, 5) == [(0, 1), (1, 2)]
    cnt = np.array([[1, 2, 3], [4, 0, 6]])
    off, rows = pieces(cnt, [(0, 1), (1, 3)])
    # peer blocks start at 0 and 6; range (1, 3) of peer 1 starts after its expert 0
    assert off.tolist() == [[0, 6], [1, 10]]
    assert rows.tolist() == [[1, 4], [5, 6]]


def test_library_ep_plan_equals_protocol_pieces():
    """db_moe_ep_plan (the C++ plan MoeEp::forward issues its NCCL pieces
    from) equals the protocol's pieces / chunk_bounds on random count
    matrices, for both directions. Host-only: no device needed."""
    import paper_1707_02402_b200 as db
    from paper_1707_02402_b200.moe_ep import chunk_bounds, pieces
    rng = np.random.default_rng(3)
    for G, E, chunks in [(1, 4, 1), (2, 8, 3), (4, 6, 4), (8, 128, 4), (3, 5, 9)]:
        send = rng.integers(0, 60, G * E).astype(np.int32)
        recv = rng.integers(0, 60, (G, E)).astype(np.int32)
        so, sr, ro, rr = db.moe_ep_plan(G, E, send, recv, chunks)
        b = chunk_bounds(E, chunks)
        a_off, a_rows = pieces(send.reshape(G, E), b)
        b_off, b_rows = pieces(recv, b)
        assert np.array_equal(so, a_off) and np.array_equal(sr, a_rows)
        assert np.array_equal(ro, b_off) and np.array_equal(rr, b_rows)
