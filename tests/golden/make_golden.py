"""Generates tests/golden/*.json|npz from the COMPILED REFERENCE (oracle/_ref).

Run in the dev container (needs /root/reference to build oracle/_ref):
    make -C oracle && python tests/golden/make_golden.py

Fingerprints are FNV-1a-64 (offset 0xcbf29ce484222325, prime 0x100000001b3):
  * sched_fnv  — over the int32 arrays step_group_off | group_fid |
                 group_member_off | member_example | member_node of the
                 reference schedule (tests/oracle_lib.FlatSchedule layout);
  * json_fnv   — over schedule_to_json text in the format the reference's own
                 golden test pins (tests/test_serialize.cpp:69-110, nlohmann
                 dump(2), one element per line);
  * inputs_fnv — over the raw little-endian doubles of random_batch.
SURVEY.md §8(c) lists other FNV values whose exact method is not stated; they
could not be reproduced, so these fixtures (method above, values from the
reference itself) replace them.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
import oracle_lib as O  # noqa: E402


def sched_fnv(fs):
    blob = b"".join(np.ascontiguousarray(a, np.int32).tobytes() for a in
                    (fs.step_group_off, fs.group_fid, fs.group_member_off, fs.member_example,
                     fs.member_node))
    return "%016x" % O.fnv1a64(blob)


IEP = {
    "cfg1": dict(kind="chain", b=64, p=40, length=16, bp=0.1, depth=4),
    "cfg2_d4": dict(kind="balanced", b=512, p=40, depth=4, length=16, bp=0.1),
    "cfg2_d5": dict(kind="balanced", b=512, p=40, depth=5, length=16, bp=0.1),
    "cfg2_d6": dict(kind="balanced", b=512, p=40, depth=6, length=16, bp=0.1),
    "cfg2_d7": dict(kind="balanced", b=512, p=40, depth=7, length=16, bp=0.1),
    "cfg2_d8": dict(kind="balanced", b=512, p=40, depth=8, length=16, bp=0.1),
    "cfg3": dict(kind="chain", b=4096, p=40, length=16, bp=0.3, depth=4),
    "dag_small": dict(kind="dag", b=200, p=12, length=12, bp=0.5, depth=4),
}


def moe_routing(T, n, k):
    s = np.zeros((T, n))
    O.ref().refshim_moe_inputs(T, n, 1, 0, None, s.ctypes.data_as(O.P_F64))
    ids, w = O.topk(s, k, use_ref=True)
    counts = np.bincount(ids.ravel(), minlength=n)
    return {"T": T, "n": n, "k": k,
            "routing_fnv": "%016x" % O.fnv1a64(ids.astype(np.int32).tobytes()),
            "weights_fnv": "%016x" % O.fnv1a64(w.tobytes()),
            "scores_fnv": "%016x" % O.fnv1a64(s.tobytes()),
            "rows_min": int(counts.min()), "rows_max": int(counts.max()),
            "occupied": int(np.count_nonzero(counts))}


def cfg5_full():
    """Full-T cfg5 routing (T = 1,048,576, n = 1024, k = 4; 8.6 GB of fp64
    scores) from the compiled reference, merged into fingerprints.json:
        python tests/golden/make_golden.py cfg5"""
    path = os.path.join(HERE, "fingerprints.json")
    with open(path) as f:
        out = json.load(f)
    out["moe"]["cfg5"] = moe_routing(1048576, 1024, 4)
    print("cfg5", out["moe"]["cfg5"], flush=True)
    with open(path, "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)


def main():
    out = {"iep": {}, "moe": {}}
    for name, c in IEP.items():
        bt = O.ref_gen_batch(c["kind"], c["b"], p=c["p"], depth=c["depth"], length=c["length"],
                             bp=c["bp"], seed=0)
        entry = {"spec": c, "nodes": bt.n_nodes,
                 "expensive_nodes": int(np.count_nonzero(bt.fid != 0))}
        for strat in ("improved", "standard", "online", "naive"):
            if strat == "naive" and bt.n_nodes > 20000:
                continue
            fs = O.ref_schedule(bt, strat)
            entry[strat] = {"steps": fs.n_steps, "groups": fs.n_groups,
                            "expensive_calls": fs.expensive_calls(),
                            "members": int(len(fs.member_node)),
                            "sched_fnv": sched_fnv(fs),
                            "json_fnv": "%016x" % O.fnv1a64(O.schedule_json(fs).encode())}
        lab, dmax = O.labels(bt, use_ref=True)
        entry["d_max"] = int(lab.max())
        entry["s_max"] = int(np.diff(bt.prog_off).max())
        x = np.zeros((bt.b, 128))
        O.ref().refshim_random_batch(bt.b, 128, O.ref().refshim_mix_seed(0, 0x1127),
                                     x.ctypes.data_as(O.P_F64))
        entry["inputs_fnv_w128"] = "%016x" % O.fnv1a64(x.tobytes())
        out["iep"][name] = entry
        print(name, entry["improved"], flush=True)

    # MoE routing (cfg4 full, a cfg5 token slice; the full-T cfg5 entry is
    # added by cfg5_full(), which needs 8.6 GB for the scores).
    for name, (T, n, k) in {"cfg4": (65536, 64, 2), "cfg5_slice": (16384, 1024, 4)}.items():
        out["moe"][name] = moe_routing(T, n, k)
        print(name, out["moe"][name], flush=True)

    with open(os.path.join(HERE, "fingerprints.json"), "w") as f:
        json.dump(out, f, indent=1, sort_keys=True)

    # Small numeric fixtures: reference Tier-A dense outputs and MoE outputs.
    arrays = {}
    bt, xin = O.ref_gen_batch("chain", 64, p=40, width=128, length=16, bp=0.1, seed=0,
                              with_inputs=True)
    ms = int(O.ref().refshim_mix_seed(0, 0xd00d))
    r = O.ref_execute(bt, xin, 128, ms)
    arrays["dense_cfg1_w128_out"] = r.outputs
    arrays["dense_cfg1_w128_trace"] = np.array([r.expensive_calls, r.peak_group_rows, r.steps])
    bt2, xin2 = O.ref_gen_batch("dag", 24, p=12, width=32, length=12, bp=0.5, seed=3,
                                with_inputs=True)
    r2 = O.ref_execute(bt2, xin2, 32, 99)
    arrays["dense_dag_w32_out"] = r2.outputs
    T, n, k, d, h = 512, 64, 2, 64, 96
    xi, sc = np.zeros((T, d)), np.zeros((T, n))
    O.ref().refshim_moe_inputs(T, n, d, 7, xi.ctypes.data_as(O.P_F64), sc.ctypes.data_as(O.P_F64))
    ids, w = O.topk(sc, k, use_ref=True)
    es = int(O.ref().refshim_mix_seed(7, 0xe4be27))
    mo, mt, _ = O.moe_forward(xi, ids, w, n, h, es, use_ref=True)
    arrays["moe_small_out"] = mo
    arrays["moe_small_ids"] = ids
    arrays["moe_small_w"] = w
    np.savez_compressed(os.path.join(HERE, "ref_outputs.npz"), **arrays)
    print("wrote fixtures")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "cfg5":
        cfg5_full()
    else:
        main()
