"""The IEP classifier head's oracle (orc_head_forward, oracle/dynbatch_oracle.c)
pinned to an independent fp64 implementation with torch.nn.functional
(conv2d 1x1, max_pool2d, linear) on the same weights (orc_head_weights).
The head is beyond the reference (its path ends at the root feature maps,
SPEC.md:13), so this cross-check is its parity anchor."""
import numpy as np
import torch
import torch.nn.functional as Fn

import oracle_lib as O


def torch_head(roots, A, seed):
    wp, bp, w1, b1, w2, b2 = (torch.from_numpy(a) for a in O.head_weights(A, seed))
    P = bp.numel()
    x = torch.from_numpy(np.ascontiguousarray(roots, np.float64)).reshape(-1, 128, 14, 14)
    proj = Fn.relu(Fn.conv2d(x, wp.T.reshape(P, 128, 1, 1), bp))           # [b, P, 14, 14]
    pooled = Fn.max_pool2d(proj, 2)                                        # [b, P, 7, 7]
    flat = pooled.permute(0, 2, 3, 1).reshape(x.shape[0], 49 * P)          # pixel-major: q·P + c
    hid = Fn.relu(flat @ w1 + b1)
    return (hid @ w2 + b2).numpy()


def test_head_oracle_matches_torch_fp64():
    rng = np.random.default_rng(5)
    roots = np.maximum(rng.standard_normal((3, 128 * 196)), 0.0)  # ReLU outputs, like the blocks'
    got = O.head_forward(roots, 28, 11)
    ref = torch_head(roots, 28, 11)
    assert got.shape == (3, 28)
    assert np.max(np.abs(got - ref)) <= 1e-10 * max(1.0, np.max(np.abs(ref)))


def test_head_weights_deterministic_and_scaled():
    a = O.head_weights(10, 3)
    b = O.head_weights(10, 3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    wp, _, w1, _, w2, _ = a
    assert np.max(np.abs(wp)) <= 0.5 / np.sqrt(128) and np.max(np.abs(w1)) <= 0.5 / np.sqrt(49 * 512)
    assert np.max(np.abs(w2)) <= 0.5 / np.sqrt(1024)
    assert not np.array_equal(O.head_weights(10, 4)[0], wp)
