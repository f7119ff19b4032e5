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
