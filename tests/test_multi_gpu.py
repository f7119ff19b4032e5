"""Multi-GPU tests for a node with ≥ 2 B200s (skipped on one GPU).

* Expert-parallel MoE over the library's own NCCL communicator
  (db_moe_ep_comm_init + db_moe_ep_forward), world 2, chunked exchange:
  every rank's token shard equals the single-GPU layer bit for bit (each
  output row depends only on its own row of the grouped GEMMs).
* IEP program shards (no collective): each rank's shard of a cfg3-shaped
  batch equals the same rows of the one-GPU run bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

WORLD = 2


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _need_gpus():
    import paper_1707_02402_b200 as db
    if db.device_count() < WORLD:
        pytest.skip(f"needs {WORLD} GPUs")


def _ep_rank(rank, port, out_dir):
    import torch.distributed as dist

    import paper_1707_02402_b200 as db
    from paper_1707_02402_b200.moe_ep import MoeEpLayer
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    db.device_open(rank)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)  # carries only the NCCL id
    n, k, T, d, h, seed = 32, 4, 4096, 256, 512, 21
    layer = MoeEpLayer(n, k, T, d, h, seed)
    for chunks in (1, 4):
        layer.forward(chunks)
        np.save(os.path.join(out_dir, f"ep{rank}_{chunks}.npy"), layer.outputs())
    dist.destroy_process_group()


def test_moe_expert_parallel_nccl_world2_equals_one_gpu(tmp_path):
    _need_gpus()
    import paper_1707_02402_b200 as db
    mp.spawn(_ep_rank, args=(_port(), str(tmp_path)), nprocs=WORLD, join=True)
    n, k, T, d, h, seed = 32, 4, 4096, 256, 512, 21
    full = db.MoeSession(n, k, T, d, h, seed=seed, precision=db.MOE_FP16)
    full.forward()
    ref = full.outputs()
    Tl = T // WORLD
    for r in range(WORLD):
        for chunks in (1, 4):
            got = np.load(tmp_path / f"ep{r}_{chunks}.npy")
            np.testing.assert_array_equal(got, ref[r * Tl:(r + 1) * Tl])


def _iep_rank(rank, out_dir):
    import paper_1707_02402_b200 as db
    db.device_open(rank)
    F = 128 * 14 * 14
    B = 256
    first, last = B * rank // WORLD, B * (rank + 1) // WORLD
    b = db.Batch.generate_range(first, last, "chain", batch=B, vocab=40, width=F, length=16, branch_prob=0.3,
                                seed=0)
    s = db.IepSession(b, 77, db.MODULE_RESBLOCK)
    s.forward()
    np.save(os.path.join(out_dir, f"iep{rank}.npy"), s.run().outputs())


def test_iep_program_shards_equal_one_gpu(tmp_path):
    _need_gpus()
    import paper_1707_02402_b200 as db
    mp.spawn(_iep_rank, args=(str(tmp_path),), nprocs=WORLD, join=True)
    F = 128 * 14 * 14
    b = db.Batch.generate("chain", batch=256, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
    ref = b.execute_device(77, db.MODULE_RESBLOCK).outputs()
    got = np.concatenate([np.load(tmp_path / f"iep{r}.npy") for r in range(WORLD)])
    np.testing.assert_array_equal(got, ref)
