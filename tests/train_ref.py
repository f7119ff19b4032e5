"""fp64 reference of one IEP training step (test infrastructure only): the
forward of every program with torch ops on the oracle's weights
(orc_resblock_weights, orc_head_weights), the classifier head, mean
softmax cross-entropy over the programs, and torch autograd's gradients.

The reference executor stops at the root maps (SPEC.md:13 lists training
as out of scope); the backward pass is SURVEY.md §8(f)4 (the
paper's batched backward). Autograd is an implementation the builder did
not write, so it pins the device backward (db_iep_session_train_step).
Gradients come back in the layouts the device reports:
* module weights input-major like the forward's (w[(tap·Cin + ci)·C + co],
  w0[(ci)·C + co] over the 2C concat), biases [C];
* head weights input-major (wp [C][P], w1 [49P][F], w2 [F][A]);
* input maps as CHW rows [b][C·196] (the reference row layout).
"""
import numpy as np
import torch
import torch.nn.functional as tf

import oracle_lib as O

C, H, W = 128, 14, 14
F = C * H * W


def _arity(fid):
    return 0 if fid == 0 else (2 if fid % 2 == 1 else 1)


def _r16(t):
    """The device's fp16 rounding of an operand, straight-through for autograd
    (the gradient itself stays fp64)."""
    return t + (t.to(torch.float16).to(torch.float64) - t).detach()


def _leaf(a):
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, requires_grad=True)


def train_step_reference(bt: O.Batch, inputs, module_seed, head_seed, answers, labels, faithful=False):
    """→ (loss, {fid: [w0, b0, w1, b1, w2, b2] grads (numpy)}, head grads
    [wp, bp, w1, b1, w2, b2], d_inputs [b][F], logits [b][A]).

    faithful: the forward rounds to fp16 exactly where the device's does
    (tensor-core operands: weights, conv inputs, mid, the concat, the head's
    activations; the residual stream stays fp32-exact as hi + lo), so the
    ReLU masks, and therefore the gradients, are the ones of the function the
    device computes; autograd stays fp64 (straight-through rounding). Without
    it, units whose pre-activation is ≈ 0 can switch sides between the fp16
    forward and an exact one, which moves whole gradient columns."""
    r = _r16 if faithful else (lambda t: t)
    raw, mods = {}, {}
    for f in sorted(set(int(x) for x in bt.fid)):
        a = _arity(f)
        if a == 0:
            continue
        w0, b0, w1, b1, w2, b2 = O.resblock_weights(a, C, module_seed, f)
        raw[f] = [_leaf(w0), _leaf(b0), _leaf(w1), _leaf(b1), _leaf(w2), _leaf(b2)]
        w = raw[f]
        k1 = r(w[2]).reshape(9, C, C).permute(2, 1, 0).reshape(C, C, 3, 3)
        k2 = r(w[4]).reshape(9, C, C).permute(2, 1, 0).reshape(C, C, 3, 3)
        k0 = r(w[0]).reshape(2 * C, C).t().reshape(C, 2 * C, 1, 1)
        mods[f] = (a, k0, w[1], k1, w[3], k2, w[5])
    x_in = _leaf(np.asarray(inputs, np.float64).reshape(bt.b, C, H, W))
    roots = []
    for e in range(bt.b):
        base = int(bt.prog_off[e])
        memo = {}

        def ev(v):
            if v in memo:
                return memo[v]
            f = int(bt.fid[base + v])
            if _arity(f) == 0:
                out = x_in[e:e + 1]
            else:
                a, k0, b0, k1, b1, k2, b2 = mods[f]
                kids = [int(bt.child0[base + v]), int(bt.child1[base + v])][:a]
                xs = [ev(c) for c in kids]
                x = tf.relu(tf.conv2d(r(torch.cat(xs, dim=1)), k0, b0)) if a == 2 else xs[0]
                t = r(tf.relu(tf.conv2d(r(x), k1, b1, padding=1)))
                out = tf.relu(x + tf.conv2d(t, k2, b2, padding=1))
            memo[v] = out
            return out

        roots.append(ev(int(bt.root[e])))
    R = torch.cat(roots, dim=0)  # [b, C, 14, 14]
    hw = [_leaf(w) for w in O.head_weights(answers, head_seed)]
    wp, bp, w1, b1, w2, b2 = hw
    P = bp.numel()
    proj = r(tf.relu(tf.conv2d(r(R), r(wp).t().reshape(P, C, 1, 1), bp)))
    pooled = tf.max_pool2d(proj, 2)
    flat = pooled.permute(0, 2, 3, 1).reshape(bt.b, 49 * P)
    hid = r(tf.relu(flat @ r(w1) + b1))
    logits = hid @ r(w2) + b2
    loss = tf.cross_entropy(logits, torch.as_tensor(np.asarray(labels, np.int64)))
    loss.backward()
    mod_grads = {f: [t.grad.numpy().copy() if t.grad is not None else np.zeros(t.shape) for t in r]
                 for f, r in raw.items()}
    head_grads = [t.grad.numpy().copy() for t in hw]
    return (float(loss.item()), mod_grads, head_grads, x_in.grad.numpy().reshape(bt.b, F).copy(),
            logits.detach().numpy().copy())
