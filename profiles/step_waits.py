"""Cycle accounting of the fused conv step kernel (cfg3), from the debug
build of k_rb_step (db_debug_conv_waits): MMA-thread waits overall and per
tile kind, epilogue cycles per tile kind, producer dependency waits."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=int(os.environ.get("BATCH", "4096")), vocab=40, width=F, length=16,
                      branch_prob=float(os.environ.get("BP", "0.3")), seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
ms, _ = s.time(5)
db.conv_wait_counters(reset=True, enable=True)
s.time(5)
w = db.conv_wait_counters(reset=True, enable=False).reshape(-1).astype(float)
acc, a, bb, tot = w[12:16]
out = {"ms_per_forward": ms / 5, "mma_thread": {"acc_wait": acc / tot, "window_wait": a / tot, "weight_wait": bb / tot,
                                                "busy": (tot - acc - a - bb) / tot},
       "producer": {"item_ring": w[16] / w[19], "dependency": w[17] / w[19], "slot": w[18] / w[19]},
       "mma_loop_mhz": w[20] / max(w[21], 1) * 1e3, "per_kind": {},
       "weight_wait_split": {"first_stage_of_tile": w[46] / tot, "other_stages": w[47] / tot},
       "weight_warp": {"item_wait": w[48] / max(w[50], 1), "stage_free_wait": w[49] / max(w[50], 1)}}
for k, name in enumerate(("conv1x1", "conv3x3_1", "conv3x3_2")):
    cyc, wa, wb, wacc = w[24 + 4 * k: 28 + 4 * k]
    ecyc, etiles = w[36 + 2 * k: 38 + 2 * k]
    n = max(etiles, 1)
    out["per_kind"][name] = {"tiles": int(etiles), "mma_item_cycles_per_tile": cyc / n,
                             "window_wait_per_tile": wa / n, "weight_wait_per_tile": wb / n,
                             "acc_wait_per_tile": wacc / n, "epilogue_cycles_per_tile": ecyc / n,
                             "producer_dep_wait_per_tile": w[42 + k] / n,
                             "share_of_mma_loop": cyc / tot}
print(json.dumps(out, indent=1))
