"""Full-shape MoE parity helpers (BASELINE cfg4 / cfg5 vs fp64 reference
arithmetic on sampled tokens). Test infrastructure only.

The device runs the whole layer (every token, every expert); the reference
side evaluates a sample of tokens with the oracle's generators
(orc_random_rows: the tokens' input and score rows of gen_moe_inputs,
src/workload.cpp:248-254), the oracle's top_k_gate restatement
(src/moe.cpp:36-69, bit-exact), the oracle's ExpertSet weights
(src/moe.cpp:71-88) and fp64 ExpertSet::apply (src/moe.cpp:98-145: h =
relu(x·W1), y = h·W2), combined per token in slot order (:254-264).
"""
from concurrent.futures import ThreadPoolExecutor
import os

import numpy as np

import oracle_lib as O

# BASELINE.json configs[3], configs[4]; seed 0 as db_moe_run
CFG = {
    "cfg4": dict(n=64, k=2, T=65536, d=1024, h=1024),
    "cfg5": dict(n=1024, k=4, T=1048576, d=2048, h=2048),
}
TOL_FP16 = 1e-3  # max|dev − ref| / max|ref| over the sampled tokens (north star)
TOL_BF16 = 2e-2  # the labelled fast mode


def sample_tokens(T, n):
    return np.unique(np.round(np.linspace(0, T - 1, n)).astype(np.int64))


def reference_tokens(n, k, d, h, seed, tokens, threads=None):
    """(ids, weights, outputs) of the given tokens (ascending), fp64."""
    x = O.random_rows(tokens, d, O.mix_seed(seed, 0x10))
    s = O.random_rows(tokens, n, O.mix_seed(seed, 0x11))
    ids, w = O.topk(s, k)
    es = O.mix_seed(seed, 0xe4be27)
    staged = np.zeros((len(tokens), k, d))

    def one(e):
        w1, w2 = O.expert_weights(d, h, es, int(e))
        t, slot = np.nonzero(ids == e)
        y = np.maximum(x[t] @ w1, 0.0) @ w2
        return t, slot, y

    threads = threads or max(1, min(32, len(os.sched_getaffinity(0))))
    with ThreadPoolExecutor(max_workers=threads) as pool:
        for t, slot, y in pool.map(one, np.unique(ids)):
            staged[t, slot] = y
    out = np.zeros((len(tokens), d))
    for slot in range(k):  # slot order
        out += w[:, slot:slot + 1] * staged[:, slot]
    return ids, w, out


def max_norm(dev, ref):
    return float(np.max(np.abs(dev - ref)) / np.max(np.abs(ref)))
