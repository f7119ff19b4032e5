"""Independent pin of the Tier-B oracle (orc_execute kind=resblock,
oracle/dynbatch_oracle.c:430-489) against torch.nn.functional.conv2d in fp64.

The reference has no conv module, so the restated residual
block is checked here against a third-party implementation the builder did
not write: the same weights (orc_resblock_weights, input-major
w[(tap·Cin+ci)·C+co]) are re-laid out as torch's [Cout, Cin, kh, kw], and the
programs are evaluated by a recursive walk of the tree (child k is operand k,
leaves fetch inputs[example]: src/executor.cpp:126-151), not by the oracle's
schedule-driven loop. Both sides are fp64 with different summation orders,
so they agree to ~1e-13 relative; the bar is 1e-11.
"""
import numpy as np
import pytest
import torch
import torch.nn.functional as tf

import oracle_lib as O

C, H, W = 128, 14, 14
F = C * H * W


def _arity(fid):
    return 0 if fid == 0 else (2 if fid % 2 == 1 else 1)


def _torch_weights(arity, seed, fid):
    w0, b0, w1, b1, w2, b2 = O.resblock_weights(arity, C, seed, fid)
    # input-major w[(tap·Cin + ci)·C + co] -> [co, ci, kh, kw]
    k1 = torch.from_numpy(w1.reshape(9, C, C)).permute(2, 1, 0).reshape(C, C, 3, 3).contiguous()
    k2 = torch.from_numpy(w2.reshape(9, C, C)).permute(2, 1, 0).reshape(C, C, 3, 3).contiguous()
    k0 = torch.from_numpy(w0.reshape(2 * C, C)).t().reshape(C, 2 * C, 1, 1).contiguous()
    return (k0, torch.from_numpy(b0), k1, torch.from_numpy(b1), k2, torch.from_numpy(b2))


def _block(wts, arity, xs):
    k0, b0, k1, b1, k2, b2 = wts
    if arity == 2:
        x = tf.relu(tf.conv2d(torch.cat(xs, dim=1), k0, b0))
    else:
        x = xs[0]
    t = tf.relu(tf.conv2d(x, k1, b1, padding=1))
    return tf.relu(x + tf.conv2d(t, k2, b2, padding=1))


def torch_execute(bt: O.Batch, inputs: np.ndarray, module_seed: int) -> np.ndarray:
    """Recursive fp64 evaluation of every program's root with torch convs."""
    cache = {}
    out = np.zeros((bt.b, F), np.float64)
    for e in range(bt.b):
        base = int(bt.prog_off[e])
        memo = {}

        def ev(v):
            if v in memo:
                return memo[v]
            f = int(bt.fid[base + v])
            a = _arity(f)
            if a == 0:
                r = torch.from_numpy(inputs[e].reshape(1, C, H, W).copy())
            else:
                if f not in cache:
                    cache[f] = _torch_weights(a, module_seed, f)
                kids = [int(bt.child0[base + v]), int(bt.child1[base + v])][:a]
                r = _block(cache[f], a, [ev(c) for c in kids])
            memo[v] = r
            return r

        out[e] = ev(int(bt.root[e])).reshape(-1).numpy()
    return out


@pytest.mark.parametrize("kind,b,p,depth,length,bp,seed", [
    ("chain", 3, 10, 4, 6, 0.4, 1),     # mixed unary / binary chains
    ("balanced", 2, 8, 3, 8, 0.0, 2),   # all-binary trees
    ("dag", 3, 9, 4, 6, 0.5, 3),        # shared children
])
def test_resblock_oracle_equals_torch_conv2d(kind, b, p, depth, length, bp, seed):
    torch.set_num_threads(max(1, min(8, torch.get_num_threads())))
    bt = O.gen_batch(kind, b, p=p, depth=depth, length=length, bp=bp, seed=seed)
    x = O.random_batch(b, F, O.mix_seed(seed, 0x1127))
    ms = O.mix_seed(seed, 0xd00d)
    r = O.execute(bt, O.schedule_improved(bt), x, ms, "resblock")
    assert r.rc == 0
    want = torch_execute(bt, x, ms)
    assert r.expensive_calls > 0
    err = np.max(np.abs(r.outputs - want)) / np.max(np.abs(want))
    assert err <= 1e-11, err


def test_resblock_weight_layout_is_input_major():
    """One conv3x3 tap/channel picked by hand: the torch re-layout and the
    oracle's input-major index address the same weight."""
    w0, b0, w1, b1, w2, b2 = O.resblock_weights(1, C, 5, 2)
    k1 = _torch_weights(1, 5, 2)[2]
    tap, ci, co = 7, 33, 101  # tap 7 = (kh 2, kw 1)
    assert k1[co, ci, 2, 1].item() == w1[(tap * C + ci) * C + co]
    assert np.all(w0 == 0)  # unary blocks draw no conv1x1 weights
