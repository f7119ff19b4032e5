#!/usr/bin/env python
"""Benchmark of the dynamic-batching executor hot path (one JSON line).

Default workload (BASELINE.json configs[2], "cfg3"): IEP execution-engine
forward over a minibatch of b = 4096 chain-heavy programs (p = 40, length ≤
16, branch 0.3, seed 0), residual conv3x3/conv1x1 + ReLU module bodies on
128×14×14 feature maps, random-init weights (module_seed = mix_seed(0,
0xd00d)). One step = device scheduler (labels + stable (level, function)
bucket sort) + every per-step gather / tcgen05 conv / scatter launch.

Multi-GPU (--gpus N): one process per GPU. Without torchrun's WORLD_SIZE the
script re-launches itself under `torch.distributed.run` with N ranks. Strong
scaling by default, as BASELINE quotes it: the minibatch (cfg3: 4096
programs; cfg5: 1,048,576 tokens) is split into contiguous shards
[r·b/N, (r+1)·b/N), one per rank, with no data-path collective for the IEP
(programs are independent). --scaling weak keeps the per-GPU size fixed.

--impl reference times the reference path on the host cores (the CPU oracle
port of the same module bodies; the reference has no conv module) and prints
the same metric.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IEP exec-engine programs/sec & MoE tokens/sec; speedup vs naive and CPU ref"
F = 128 * 14 * 14
# batch / tokens: the BASELINE configuration's minibatch (the whole job's
# under strong scaling, each GPU's under --scaling weak)
CFG = {
    "cfg3": dict(kind="chain", batch=4096, vocab=40, length=16, branch_prob=0.3, depth=4),
    "cfg1": dict(kind="chain", batch=64, vocab=40, length=16, branch_prob=0.1, depth=4),
    "cfg2": dict(kind="balanced", batch=512, vocab=40, length=16, branch_prob=0.1, depth=6),
}
MOE = {
    "cfg4": dict(experts=64, k=2, tokens=65536, d=1024, h=1024),
    "cfg5": dict(experts=1024, k=4, tokens=1048576, d=2048, h=2048),
}


def shard(total, rank, world):
    """Contiguous shard [first, last) of `total` units owned by `rank`."""
    return total * rank // world, total * (rank + 1) // world


def global_units(total, world, scaling):
    return total if scaling == "strong" else total * world


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg3", choices=sorted(CFG) + sorted(MOE))
    ap.add_argument("--no-moe", action="store_true", help="skip the secondary cfg4 MoE measurement")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--depth", type=int, default=0, help="cfg2: balanced-tree depth (4-8; default 6)")
    ap.add_argument("--ep-chunks", type=int, default=0,
                    help="cfg5: expert ranges the exchange is cut into (overlap with the GEMMs); 0 = 1 at one GPU, "
                         "else 4")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="target CPU work of the bounded CPU-baseline sample")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: the BASELINE minibatch split over the GPUs; weak: that minibatch per GPU")
    ap.add_argument("--dry-run", action="store_true",
                    help="no GPU work: each rank prints its world size and shard (tests the launch on CPU)")
    return ap.parse_args()


def maybe_spawn(args):
    """--gpus N outside torchrun: re-launch this script with N ranks (one
    process per GPU) under torch.distributed.run on 127.0.0.1."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ or args.impl == "reference":
        return
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ----------------------------------------------------------------- dist
class Dist:
    def __init__(self, gpus, cpu=False):
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != gpus:
            raise SystemExit(f"bench.py: {self.world} ranks for --gpus {gpus}")
        self.pg = None
        self.cpu = cpu
        if self.world > 1:
            import torch
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            if cpu:
                dist.init_process_group("gloo")
            else:
                torch.cuda.set_device(self.local)
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
            self.pg = dist

    def barrier(self):
        if self.pg:
            self.pg.barrier()

    def max(self, x):
        if not self.pg:
            return x
        import torch
        t = torch.tensor([float(x)], device="cpu" if self.cpu else "cuda")
        self.pg.all_reduce(t, op=self.pg.ReduceOp.MAX)
        return float(t.item())

    def close(self):
        if self.pg:
            self.pg.destroy_process_group()


# --------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples (SM clock, throttle reasons) tagged with the driver's
    own timestamps; summary() keeps the samples inside the timed window."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, gpu):
        self.gpu, self.rows, self.proc, self.window = gpu, [], None, None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        import datetime
        for line in self.proc.stdout:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                t = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                self.rows.append((t, float(f[1]), float(f[2]), f[4:8]))
            except ValueError:
                continue

    def mark(self, t0, t1):
        self.window = (t0, t1)

    def stop(self):
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        rows = self.rows
        if self.window and rows:
            t0, t1 = self.window
            inside = [r for r in rows if t0 - 0.06 <= r[0] <= t1 + 0.06]
            if not inside:  # window shorter than the sampling period: nearest sample
                inside = [min(rows, key=lambda r: abs(r[0] - 0.5 * (t0 + t1)))]
            rows = inside
        sm = [r[1] for r in rows]
        reasons = sorted({self.NAMES[i] for r in rows for i in range(4)
                          if r[3][i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(r[2] for r in rows) if rows else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def ncu_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f)
    except Exception:
        return {}


# ---------------------------------------------------------- CPU oracle
def cpu_sample_run(cfg, n_programs, threads, seed=0, strategy="improved"):
    """Runs the oracle port (fp64, reference executor semantics) on the first
    n_programs of the workload, sharded over `threads` host threads (ctypes
    releases the GIL), each shard scheduled with schedule_improved or
    schedule_naive (src/schedule.cpp:94-105, one node per step). Returns
    (seconds, programs)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    ob = O.gen_batch(cfg["kind"], n_programs, p=cfg["vocab"], depth=cfg["depth"],
                     length=cfg["length"], bp=cfg["branch_prob"], seed=seed)
    x = O.random_batch(n_programs, F, O.mix_seed(seed, 0x1127))
    ms = O.mix_seed(seed, 0xd00d)
    shards = []
    per = math.ceil(n_programs / threads)
    import numpy as np
    for a in range(0, n_programs, per):
        z = min(n_programs, a + per)
        lo, hi = ob.prog_off[a], ob.prog_off[z]
        sb = O.Batch((ob.prog_off[a:z + 1] - lo).astype(np.int32), ob.fid[lo:hi].copy(),
                     np.where(ob.child0[lo:hi] >= 0, ob.child0[lo:hi], -1).astype(np.int32),
                     np.where(ob.child1[lo:hi] >= 0, ob.child1[lo:hi], -1).astype(np.int32),
                     ob.root[a:z].copy(), ob.p)
        fs = O.schedule_naive(sb) if strategy == "naive" else O.schedule_improved(sb)
        shards.append((sb, fs, np.ascontiguousarray(x[a:z])))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=len(shards)) as pool:
        res = list(pool.map(lambda s: O.execute(s[0], s[1], s[2], ms, "resblock"), shards))
    dt = time.perf_counter() - t0
    assert all(r.rc == 0 for r in res)
    return dt, n_programs


def cpu_threads():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count() or 1


def calibrate_cpu(cfg, target_s):
    threads = cpu_threads()
    dt, n = cpu_sample_run(cfg, threads, threads)  # one program per thread
    rounds = max(1, min(64, int(target_s / max(dt, 1e-3))))
    return threads, threads * rounds


def cpu_baselines(cfg, target_s):
    """The CPU baselines of SURVEY.md §8(d), timed on this box's host cores
    with the fp64 oracle port: (i) improved schedule on every host thread
    (the headline cpu_baseline), (ii) one thread, giving the host-core
    scaling, (iii) the naive per-example schedule on every thread."""
    threads, n = calibrate_cpu(cfg, target_s)
    dt, n = cpu_sample_run(cfg, n, threads)
    per_prog_thread = dt * threads / n  # seconds per program on one thread (approx.)
    n1 = max(2, int(min(target_s / 3, 6.0) / max(per_prog_thread, 1e-4)))
    dt1, _ = cpu_sample_run(cfg, n1, 1)
    nn = max(threads, n // 2)
    dtn, _ = cpu_sample_run(cfg, nn, threads, strategy="naive")
    v, v1, vn = n / dt, n1 / dt1, nn / dtn
    return {"value": v, "unit": "programs/s", "cores": threads, "kind": "port",
            "sample": f"first {n} programs of the workload, oracle fp64 port (oracle/dynbatch_oracle.c, "
                      f"schedule_improved) sharded over {threads} threads, {dt:.1f} s",
            "single_thread": {"value": v1, "sample": f"first {n1} programs on 1 thread, {dt1:.1f} s"},
            "host_core_scaling": {"threads": threads, "speedup_vs_1_thread": v / v1,
                                  "efficiency": v / v1 / threads},
            "naive": {"value": vn, "schedule": "schedule_naive (one node per step), same executor",
                      "sample": f"first {nn} programs over {threads} threads, {dtn:.1f} s",
                      "improved_over_naive": v / vn}}


def pcie_duplex_seconds(nbytes, nbytes_out=None, reps=3):
    """Seconds per simultaneous H2D of nbytes + D2H of nbytes_out (default
    the same; pinned host buffers, two streams): the e2e pipeline's bound on
    this box."""
    import torch
    n = nbytes // 4
    m = (nbytes if nbytes_out is None else nbytes_out) // 4
    h_in = torch.empty(n, dtype=torch.float32).pin_memory()
    h_out = torch.empty(m, dtype=torch.float32).pin_memory()
    d_in = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out = torch.empty(m, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    best = float("inf")
    for _ in range(reps + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    del h_in, h_out, d_in, d_out
    return best


# ------------------------------------------------------------- our arm
def run_ours(args, dist):
    import numpy as np
    import paper_1707_02402_b200 as db
    import torch

    cfg = dict(CFG[args.workload])
    if args.depth:
        cfg["depth"] = args.depth
    N = max(1, dist.world)
    B = global_units(cfg["batch"], N, args.scaling)  # programs in the whole job's minibatch
    first, last = shard(B, dist.rank, N)
    per = last - first
    db.device_open(dist.local)
    clk = ClockSampler(dist.local).start()
    batch = db.Batch.generate_range(first, last, cfg["kind"], batch=B, vocab=cfg["vocab"],
                                    width=F, depth=cfg["depth"], length=cfg["length"],
                                    branch_prob=cfg["branch_prob"], seed=0)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    module_seed = int.from_bytes(_mix_seed(0, 0xd00d).to_bytes(8, "little"), "little")
    # a second batch of programs (the next seed's), for the end-to-end pass
    # where every call brings new programs; the session is sized for both
    batch2 = db.Batch.generate_range(first, last, cfg["kind"], batch=B, vocab=cfg["vocab"],
                                     width=F, depth=cfg["depth"], length=cfg["length"],
                                     branch_prob=cfg["branch_prob"], seed=1)
    seqs = [batch.prefix_tokens(), batch2.prefix_tokens()]
    cap_nodes = max(int(o[-1]) for _, o in seqs)
    cap_len = max(int(np.diff(o).max()) for _, o in seqs)
    sess = db.IepSession(batch, module_seed, db.MODULE_RESBLOCK, program_capacity=per,
                         node_capacity=cap_nodes, length_capacity=cap_len)
    sess.time(max(3, args.warmup))  # warm-up (≥ 3 steps)
    stats = sess.stats()

    dist.barrier()
    t0 = time.time()
    # headline: the forwards as graph replays, with CUDA-event nodes around
    # the fused step kernel only (its own time, for the roofline, from the
    # same loop and thermal state as the headline)
    ms, kst = sess.time(args.steps, profile=2)
    dist.barrier()
    clk.mark(t0, time.time())
    ms_step = dist.max(ms / args.steps)
    value = B / (ms_step / 1e3)
    # second pass with events around every launch: per-kernel-class times
    # for the roofline and the breakdown (not the headline)
    pms, kt = sess.time(args.steps, profile=True)
    # the step kernel's own clock: clock64 cycles over globaltimer ns in its
    # MMA loop (debug-counter build of the kernel, 3 forwards). nvidia-smi's
    # clocks.sm reads the boost target; under the board power limit the
    # delivered SM clock is lower, and this is the figure the kernel saw.
    db.conv_wait_counters(reset=True, enable=True)
    sess.time(3)
    w = db.conv_wait_counters(reset=True, enable=False)
    kernel_mhz = float(w[5][0]) / max(float(w[5][1]), 1.0) * 1e3

    # end-to-end through the public API, every call a new batch: the
    # programs as prefix function sequences (db_iep_session_set_programs:
    # CSR built on the device) and pinned host fp32 input rows → H2D →
    # device scheduler + forward → D2H of the root outputs. The pipelined
    # call overlaps step i's forward with the upload of step i+1 and the
    # download of step i−1 (copy streams, full-duplex PCIe). The two program
    # sets alternate; wall clock over K steps, max over ranks.
    xin = [db.PinnedArray((per, F), np.float32) for _ in range(2)]
    xout = [db.PinnedArray((per, F), np.float32) for _ in range(2)]
    toks, offs = [], []
    for t, o in seqs:
        pt, po = db.PinnedArray(t.shape, np.int32), db.PinnedArray(o.shape, np.int32)
        pt.array[:] = t
        po.array[:] = o
        toks.append(pt)
        offs.append(po)
    rng = np.random.default_rng(dist.rank)
    for x in xin:
        x.array[:] = rng.uniform(-1, 1, size=(per, F)).astype(np.float32)

    def e2e_pass(steps, new_programs):
        for i in range(steps):
            if new_programs:
                sess.set_programs(toks[i % 2].array, offs[i % 2].array)
            sess.forward_host_async(xin[i % 2].array, xout[i % 2].array)
        sess.synchronize()

    e2e_pass(2, True)  # warm-up: creates the copy streams and double buffers
    dist.barrier()
    e2e_steps = max(args.steps, 80)  # steady state: amortises the pipeline fill and drain
    t0 = time.perf_counter()
    e2e_pass(e2e_steps, True)
    e2e_s = dist.max((time.perf_counter() - t0) / e2e_steps)
    prog_bytes = sum(t.array.nbytes + o.array.nbytes for t, o in zip(toks, offs)) / 2
    dist.barrier()
    t0 = time.perf_counter()
    e2e_pass(e2e_steps, False)
    fixed_s = dist.max((time.perf_counter() - t0) / e2e_steps)
    e2e = {"value": B / e2e_s, "unit": "programs/s",
           "h2d_bytes_per_step": int(per * F * 4 + prog_bytes), "d2h_bytes_per_step": per * F * 4,
           "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
           "api": "db_iep_session_set_programs (new prefix sequences every call, CSR built on the device) + "
                  "db_iep_session_forward_host_async (pinned fp32 CHW rows in, root rows out; copies overlap "
                  "the neighbouring steps' forwards)",
           "same_programs_every_call": {"value": B / fixed_s, "ms_per_step": fixed_s * 1e3}}
    # the e2e bound: this box's PCIe with both directions busy (pinned
    # 411 MB each way on two streams, as the pipeline runs them)
    link_s = pcie_duplex_seconds(per * F * 4)
    e2e["roofline"] = {"bound": "pcie (H2D and D2H concurrent)",
                       "achieved": round((per * F * 4) / e2e_s / 1e9, 1),
                       "peak": round((per * F * 4) / link_s / 1e9, 1), "unit": "GB/s per direction",
                       "frac": round(link_s / e2e_s, 4)}

    # roofline of the dominant kernel: the fused conv step (conv1x1 + conv3x3
    # #1 + conv3x3 #2 with the residual on the tensor cores), class 4
    peaks, src = measured_peaks()
    # the step kernel inside the headline loop (graph event nodes); the
    # per-launch profiled pass only when the forward is not one step launch
    src_kernel = kst if kst.launches[4] > 0 else kt
    conv_ms, conv_launches, conv_flops = src_kernel.ms[4], src_kernel.launches[4], src_kernel.flops[4]
    achieved = conv_flops / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else 0.0
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    traffic = ncu_traffic().get("step_bytes_per_launch")
    roofline = {"kernel": "k_rb_step (fused tcgen05 implicit-GEMM conv1x1 + conv3x3 x2 per step)",
                "bound": "tensor", "achieved": round(achieved, 1), "peak": peak, "unit": "TFLOP/s",
                "frac": round(achieved / peak, 4), "peak_source": src + " bf16 sustained (fp16 operands run "
                "at the same tcgen05 kind::f16 rate)",
                "traffic": traffic,
                "algorithmic_flops_per_launch": conv_flops / max(conv_launches, 1),
                "algorithmic_bytes_per_launch": src_kernel.bytes[4] / max(conv_launches, 1),
                "avg_launch_ms": conv_ms / max(conv_launches, 1),
                "timed_in": ("the headline loop (CUDA-graph replays with event-record nodes around the step kernel)"
                             if src_kernel is kst else "the per-launch profiled pass"),
                "share_of_step": round(conv_ms / max(conv_launches, 1) / ms_step, 4) if ms_step > 0 else None}
    kernels = {db.KERNEL_CLASSES[c]: {"ms_per_step": kt.ms[c] / args.steps,
                                      "launches_per_step": kt.launches[c] / args.steps,
                                      "tflops": (kt.flops[c] / (kt.ms[c] / 1e3) / 1e12) if kt.ms[c] and kt.flops[c] else None,
                                      "gbs": (kt.bytes[c] / (kt.ms[c] / 1e3) / 1e9) if kt.ms[c] and kt.bytes[c] else None}
               for c in range(8) if kt.launches[c]}

    out = {"metric": METRIC, "value": value, "unit": "programs/s", "n_gpus": N,
           "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms_step,
           "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
           "dtype": "fp16 tensor-core operands, fp32 accumulate and node values",
           "data": "synthetic (reference generators, seed 0; random-init weights)",
           "config": {"workload": f"{args.workload}: IEP forward, {cfg['kind']} programs p={cfg['vocab']} "
                                  + (f"depth {cfg['depth']}" if cfg["kind"] == "balanced" else
                                     f"len<={cfg['length']} branch={cfg['branch_prob']}")
                                  + f", residual conv modules on 128x14x14, minibatch {B}"
                                  + (f" ({per} programs on this rank)" if N > 1 else ""),
                      "global_batch": B, "programs_per_gpu": per,
                      "parallelism": f"dp{N} (program shards, no collective)",
                      "l2": "inputs (411 MB) and node values (4.9 GB) exceed the 126 MB L2"},
           "e2e": e2e, "roofline": roofline, "kernels": kernels,
           "profiled_ms_per_step": pms / args.steps,
           "gpu_launches": int(stats.kernel_launches) * args.steps,
           "schedule": {"steps": stats.steps, "groups": stats.groups,
                        "expensive_calls": stats.expensive_calls,
                        "peak_group_rows": stats.peak_group_rows},
           "algorithmic_flops_per_step": stats.algorithmic_flops * N,
           "clocks": None}

    # the IEP classifier head on the roots (conv1x1 → pool
    # → FC → FC, tcgen05 GEMMs): device ms per head forward on this batch's
    # roots, next to the module forward it follows
    try:
        sess.set_head(28, module_seed)
        sess.forward()
        hms, hfl = sess.time_head(max(args.steps, 5))
        out["head"] = {"answers": 28, "ms_per_step": hms, "tflops": hfl / (hms / 1e3) / 1e12,
                       "flops_per_step": hfl, "forward_plus_head_programs_per_s": B / ((ms_step + hms) / 1e3),
                       "share_of_forward": hms / ms_step}
    except Exception as e:  # reported, not fatal
        out["head"] = {"error": str(e)}

    # one training step (training forward, head, softmax
    # cross-entropy, backward through the head and the module groups) on this
    # minibatch, and on its first 64 programs the naive schedule's step (the
    # paper's batched-backward comparison)
    try:
        labels = (np.arange(per) % 28).astype(np.int32)
        sess.set_training(True)
        tms = sess.time_train(max(2, min(args.steps, 5)), labels)
        sess.set_training(False)
        nb = min(per, 64)
        sub = [db.IepSession(batch, module_seed, db.MODULE_RESBLOCK, first=0, last=nb) for _ in range(2)]
        sub[1].set_schedule(db.Batch.generate_range(first, first + nb, cfg["kind"], batch=B, vocab=cfg["vocab"],
                                                    width=8, depth=cfg["depth"], length=cfg["length"],
                                                    branch_prob=cfg["branch_prob"], seed=0).schedule("naive"))
        sub_ms = []
        for x in sub:
            x.set_head(28, module_seed)
            x.set_training(True)
            sub_ms.append(x.time_train(2, labels[:nb]))
        out["train"] = {"ms_per_step": tms, "programs_per_s": per / (tms / 1e3),
                        "backward_over_forward": (tms - ms_step) / ms_step,
                        "gemms": "3x3 data and weight gradients as tcgen05 implicit GEMMs (bwd_conv.cu); head and conv1x1 GEMMs on cuBLAS TF32",
                        "naive_vs_improved_64": {"improved_ms": sub_ms[0], "naive_ms": sub_ms[1],
                                                 "speedup": sub_ms[1] / sub_ms[0]}}
        del sub
    except Exception as e:  # reported, not fatal
        out["train"] = {"error": str(e)}

    # naive per-example execution on the GPU (same kernels, one node per
    # step). "naive" runs each step after the previous one, one module call at
    # a time like the reference's naive executor (DYNBATCH_STEP_BARRIER=1);
    # "naive_dataflow" lets the executor overlap independent steps (per-image
    # readiness), which recovers part of the batching by itself.
    try:
        nb = min(per, 64)
        naive_sched = db.Batch.generate_range(first, first + nb, cfg["kind"], batch=B, vocab=cfg["vocab"],
                                              width=8, depth=cfg["depth"], length=cfg["length"],
                                              branch_prob=cfg["branch_prob"], seed=0).schedule("naive")

        def naive_ms(barrier):
            os.environ["DYNBATCH_STEP_BARRIER"] = "1" if barrier else "0"
            try:
                x = db.IepSession(batch, module_seed, db.MODULE_RESBLOCK, first=0, last=nb)
                x.set_schedule(naive_sched)
                x.time(1)  # captures the forward with the barrier setting
                return x.time(2)[0] / 2
            finally:
                os.environ.pop("DYNBATCH_STEP_BARRIER", None)

        nms, dms = naive_ms(True), naive_ms(False)
        imp = db.IepSession(batch, module_seed, db.MODULE_RESBLOCK, first=0, last=nb)
        imp.time(1)
        ims = imp.time(2)[0] / 2
        out["naive_gpu"] = {"programs": nb, "naive_programs_per_s": nb / (nms / 1e3),
                            "naive_dataflow_programs_per_s": nb / (dms / 1e3),
                            "improved_programs_per_s": nb / (ims / 1e3),
                            "speedup_improved_vs_naive": nms / ims,
                            "speedup_improved_vs_naive_dataflow": dms / ims}
    except Exception as e:  # reported, not fatal
        out["naive_gpu"] = {"error": str(e)}

    if not args.no_moe:
        try:
            out["moe"] = run_moe(args, dist, "cfg4", secondary=True)
        except Exception as e:  # reported, not fatal
            out["moe"] = {"error": str(e)}
    clk.stop()
    out["clocks"] = clk.summary()
    out["clocks"]["step_kernel_sm_mhz"] = round(kernel_mhz)
    out["clocks"]["note"] = ("sm_mhz is nvidia-smi's clocks.sm (boost target); step_kernel_sm_mhz is the clock the "
                             "fused step kernel measured itself (clock64 / globaltimer): the board power limit "
                             "holds it below sm_max_mhz while the tensor cores and HBM are busy")
    if dist.rank == 0 and N == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baselines(cfg, args.cpu_seconds)
    return out


def run_moe(args, dist, name, secondary=False):
    """MoE layer forward (gate → stable expert sort → dispatch → grouped
    tcgen05 GEMM1+ReLU → GEMM2 → slot-order combine), fp16 operands (the
    precise mode: ≤ 1e-3 vs fp64, profiles/r02_moe_parity.json). Token
    shard per rank; tokens/s."""
    import numpy as np
    import paper_1707_02402_b200 as db
    c = MOE[name]
    N = max(1, dist.world)
    TG = global_units(c["tokens"], N, args.scaling)
    first, last = shard(TG, dist.rank, N)
    T = last - first
    sess = db.MoeSession(c["experts"], c["k"], TG, c["d"], c["h"], seed=0, precision=db.MOE_FP16,
                         first=first, last=last)
    sess.time(3)
    st = sess.stats()
    dist.barrier()
    ms, _ = sess.time(args.steps)
    dist.barrier()
    ms_step = dist.max(ms / args.steps)
    _, kt = sess.time(args.steps, profile=True)
    peaks, src = measured_peaks()
    g_ms, g_fl = kt.ms[4] + kt.ms[5], kt.flops[4] + kt.flops[5]
    gemm_tf = g_fl / (g_ms / 1e3) / 1e12 if g_ms else 0.0
    res = {"metric": "MoE tokens/sec", "value": TG / (ms_step / 1e3), "unit": "tokens/s",
           "ms_per_step": ms_step, "dtype": "fp16 tensor-core operands (precise mode, <= 1e-3 vs fp64), fp32 accumulate",
           "config": {"workload": f"{name}: n={c['experts']} top-{c['k']} d={c['d']} h={c['h']}, "
                                  f"{TG} tokens" + (f" ({T} on this rank)" if N > 1 else ""),
                      "global_tokens": TG},
           "roofline": {"kernel": "k_moe_gemm (grouped tcgen05 GEMM1+GEMM2)", "bound": "tensor",
                        "achieved": round(gemm_tf, 1),
                        "peak": peaks.get("bf16_tflops_sustained"), "unit": "TFLOP/s",
                        "frac": round(gemm_tf / peaks.get("bf16_tflops_sustained", 1), 4)},
           "kernels": {name_: {"ms_per_step": kt.ms[c_] / args.steps,
                               "gbs": (kt.bytes[c_] / (kt.ms[c_] / 1e3) / 1e9) if kt.ms[c_] and kt.bytes[c_] else None,
                               "hbm_frac": ((kt.bytes[c_] / (kt.ms[c_] / 1e3) / 1e9) / peaks.get("hbm_gbs", 6450))
                               if kt.ms[c_] and kt.bytes[c_] else None,
                               # the north star's reference point: ~8 TB/s nominal HBM3e
                               "hbm_frac_of_8tbs": ((kt.bytes[c_] / (kt.ms[c_] / 1e3) / 1e9) / 8000.0)
                               if kt.ms[c_] and kt.bytes[c_] else None}
                       for c_, name_ in ((3, "gate+sort+dispatch"), (4, "gemm1_relu"), (5, "gemm2"),
                                         (6, "combine")) if kt.launches[c_]},
           "gpu_launches_per_step": int(st.kernel_launches)}
    # end-to-end through the public API: pinned host fp32 inputs + fp64
    # scores → H2D → gate / dispatch / GEMMs / combine → D2H of the fp32
    # outputs, every step; the pipelined call overlaps step i's forward with
    # step i+1's upload and step i−1's download. Two input sets alternate.
    xin = [db.PinnedArray((T, c["d"]), np.float32) for _ in range(2)]
    sc = [db.PinnedArray((T, c["experts"]), np.float64) for _ in range(2)]
    yout = [db.PinnedArray((T, c["d"]), np.float32) for _ in range(2)]
    rng = np.random.default_rng(dist.rank)
    for i in range(2):
        xin[i].array[:] = rng.uniform(-1, 1, size=(T, c["d"])).astype(np.float32)
        sc[i].array[:] = rng.uniform(-1, 1, size=(T, c["experts"]))

    def e2e_pass(steps):
        for i in range(steps):
            sess.forward_host_async(xin[i % 2].array, sc[i % 2].array, yout[i % 2].array)
        sess.synchronize()

    e2e_pass(3)
    dist.barrier()
    e2e_steps = max(args.steps, 40)
    t0 = time.perf_counter()
    e2e_pass(e2e_steps)
    e2e_s = dist.max((time.perf_counter() - t0) / e2e_steps)
    h2d, d2h = T * (c["d"] * 4 + c["experts"] * 8), T * c["d"] * 4
    link_s = pcie_duplex_seconds(h2d, d2h)
    res["e2e"] = {"value": TG / e2e_s, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                  "ms_per_step": e2e_s * 1e3, "steps": e2e_steps,
                  "api": "db_moe_session_forward_host_async (pinned fp32 inputs + fp64 scores in, fp32 outputs out; "
                         "copies overlap the neighbouring steps' forwards)",
                  "roofline": {"bound": "pcie (H2D and D2H concurrent)", "achieved_h2d_gbs": round(h2d / e2e_s / 1e9, 1),
                               "peak_h2d_gbs": round(h2d / link_s / 1e9, 1), "frac": round(link_s / e2e_s, 4)}}
    if dist.rank == 0 and N == 1 and not args.no_cpu_baseline and not secondary:
        res["cpu_baseline"] = moe_cpu_baselines(c)
    return res


def moe_cpu_baselines(c, tokens=1024, naive_tokens=256):
    """The compiled reference's own MoE layer (oracle/_ref: moe_forward_batched
    and moe_forward_naive, src/moe.cpp:162-270, fp64, single-threaded as
    shipped) on the first `tokens` tokens of the workload, timed by its own
    trace (total_seconds; the ExpertSet construction is outside it)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import oracle_lib as O
    if not O.ref_available():
        return {"unavailable": "oracle/_ref not built"}
    n, k, d, h = c["experts"], c["k"], c["d"], c["h"]
    out = {"unit": "tokens/s", "cores": 1, "kind": "reference"}
    for name, T, batched in (("batched", tokens, True), ("naive", naive_tokens, False)):
        x, sc = O.moe_inputs(T, n, d, 0)
        ids, w = O.topk(sc, k, use_ref=True)
        _, _, secs = O.moe_forward(x, ids, w, n, h, O.mix_seed(0, 0xe4be27), use_ref=True, batched=batched)
        out[name] = {"value": T / secs[2], "sample": f"first {T} tokens, {secs[2]:.2f} s (trace total_seconds)"}
    out["value"] = out["batched"]["value"]
    out["sample"] = out["batched"]["sample"] + ", moe_forward_batched on 1 thread"
    out["batched_over_naive"] = out["batched"]["value"] / out["naive"]["value"]
    return out


def run_moe_ep(args, dist, name):
    """Expert-parallel MoE layer (cfg5: n=1024 top-4, d=h=2048): tokens
    T/G and experts n/G per rank, NCCL all-to-all of counts and rows for
    dispatch and combine (paper_1707_02402_b200.moe_ep). Strong scaling by
    default: the 1,048,576-token layer split over the ranks (one rank runs
    all of it)."""
    import torch
    import paper_1707_02402_b200 as db
    from paper_1707_02402_b200.moe_ep import MoeEpLayer
    c = MOE[name]
    N = max(1, dist.world)
    db.device_open(dist.local)
    torch.cuda.set_device(dist.local)
    T = global_units(c["tokens"], N, args.scaling)
    layer = MoeEpLayer(c["experts"], c["k"], T, c["d"], c["h"], seed=0)
    chunks = args.ep_chunks or (1 if N == 1 else 4)
    clk = ClockSampler(dist.local).start()
    for _ in range(3):
        layer.forward(chunks)
    layer.sess.synchronize()
    dist.barrier()
    t0 = time.time()
    stream = torch.cuda.ExternalStream(layer.sess.stream, device=torch.device("cuda", dist.local))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        layer.forward(chunks)
    e1.record(stream)
    e1.synchronize()
    dist.barrier()
    clk.mark(t0, time.time())
    ms_step = dist.max(e0.elapsed_time(e1) / args.steps)
    clk.stop()
    peaks, src = measured_peaks()
    flops = 4.0 * T * c["k"] * c["d"] * c["h"]  # GEMM1 + GEMM2 over all ranks
    achieved = flops / N / (ms_step / 1e3) / 1e12
    peak = peaks.get("bf16_tflops_sustained")
    rows = dist.max(layer.last_recv_rows)
    return {"metric": "MoE tokens/sec (expert parallel)", "value": T / (ms_step / 1e3), "unit": "tokens/s",
            "ms_per_step": ms_step, "dtype": "fp16 tensor-core operands (precise mode), fp32 accumulate",
            "config": {"workload": f"{name}: n={c['experts']} top-{c['k']} d={c['d']} h={c['h']}, "
                                   f"{T} tokens, {T // N} tokens and {c['experts'] // N} experts per GPU",
                       "global_tokens": T,
                       "parallelism": (f"ep{N} (NCCL point-to-point exchange by expert range, overlapped with the "
                                       "GEMMs)") if N > 1 else "ep1 (no exchange: one device pass)",
                       "exchange_chunks": chunks},
            "roofline": {"kernel": "whole EP layer (gate, sort, pack, 2x all-to-all, grouped GEMMs, combine)",
                         "bound": "tensor", "achieved": round(achieved, 1), "peak": peak,
                         "unit": "TFLOP/s per GPU", "frac": round(achieved / peak, 4) if peak else None,
                         "peak_source": src + " bf16 sustained"},
            "max_rows_received": int(rows), "clocks": clk.summary(),
            "gpu_launches_per_step": 14,
            "e2e": None, "e2e_note": "inputs are generated per rank on the device side; no host I/O path",
            "cpu_baseline": (moe_sampled_cpu_baseline(c) if dist.rank == 0 and N == 1 and not args.no_cpu_baseline
                             else None)}


def moe_sampled_cpu_baseline(c, tokens=32):
    """cfg5 on the CPU is infeasible as shipped (ExpertSet alone is 68.7 GB of
    fp64): the fp64 oracle port of moe_forward_batched
    (src/moe.cpp:162-270; scalar fma loops, one thread) on the first `tokens`
    tokens' items, timed by its own module + combine clock (expert weight
    generation outside it), extrapolated FLOP-proportionally per token."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import oracle_lib as O
    n, k, d, h = c["experts"], c["k"], c["d"], c["h"]
    rows = np.arange(tokens, dtype=np.int64)
    x = O.random_rows(rows, d, O.mix_seed(0, 0x10))
    sc = O.random_rows(rows, n, O.mix_seed(0, 0x11))
    ids, w = O.topk(sc, k)
    _, _, secs = O.moe_forward(x, ids, w, n, h, O.mix_seed(0, 0xe4be27))
    return {"value": tokens / secs[2], "unit": "tokens/s", "cores": 1, "kind": "port",
            "sample": f"first {tokens} tokens ({tokens * k} expert items), oracle fp64 port, {secs[2]:.2f} s; "
                      f"extrapolated per token (the full layer needs 68.7 GB of fp64 experts)"}


def _mix_seed(seed, stream):
    M = (1 << 64) - 1

    def sm(s):
        s = (s + 0x9e3779b97f4a7c15) & M
        z = s
        z = ((z ^ (z >> 30)) * 0xbf58476d1ce4e5b9) & M
        z = ((z ^ (z >> 27)) * 0x94d049bb133111eb) & M
        return s, z ^ (z >> 31)

    s = seed ^ ((0x9e3779b97f4a7c15 + (stream << 1)) & M)
    s, a = sm(s)
    s ^= stream
    s, b = sm(s)
    return a ^ b


# ------------------------------------------------------ reference arm
def run_reference(args, n_gpus):
    cfg = dict(CFG[args.workload])
    if args.depth:
        cfg["depth"] = args.depth
    threads, n = calibrate_cpu(cfg, min(args.cpu_seconds, 6.0))
    for _ in range(max(0, args.warmup)):
        cpu_sample_run(cfg, n, threads)
    times = []
    for _ in range(args.steps):
        dt, _ = cpu_sample_run(cfg, n, threads)
        times.append(dt)
    sec = sum(times) / len(times)
    value = n / sec
    return {"metric": METRIC, "value": value, "unit": "programs/s", "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generators, seed 0; random-init weights)",
            "impl": "reference",
            "config": {"workload": f"{args.workload}: IEP forward, residual conv modules on 128x14x14 "
                                   f"(CPU oracle port; the reference has no conv module)",
                       "programs_per_step": n},
            "cpu_baseline": {"value": value, "unit": "programs/s", "cores": threads, "kind": "port",
                             "sample": f"first {n} programs of the workload per step, fp64 oracle port "
                                       f"sharded over {threads} threads"},
            "e2e": {"value": value, "unit": "programs/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def dry_run(args, dist):
    """The launch without GPU work: world size and this rank's shard."""
    N = max(1, dist.world)
    if args.workload in MOE:
        total = global_units(MOE[args.workload]["tokens"], N, args.scaling)
    else:
        total = global_units(CFG[args.workload]["batch"], N, args.scaling)
    first, last = shard(total, dist.rank, N)
    counts = [0] * N
    if dist.pg:  # every rank's shard size, gathered to check the split
        import torch
        t = torch.zeros(N, dtype=torch.int64)
        t[dist.rank] = last - first
        dist.pg.all_reduce(t)
        counts = t.tolist()
    else:
        counts = [last - first]
    return {"dry_run": True, "rank": dist.rank, "world": N, "gpus": args.gpus, "workload": args.workload,
            "scaling": args.scaling, "total": total, "shard": [first, last], "shard_sizes": counts}


def main():
    args = parse()
    if args.impl == "reference":
        # CPU arm: rank 0 alone runs and prints; other ranks exit without work.
        if int(os.environ.get("RANK", "0")) == 0:
            print(json.dumps(run_reference(args, int(os.environ.get("WORLD_SIZE", args.gpus)))), flush=True)
        return
    maybe_spawn(args)
    dist = Dist(args.gpus, cpu=args.dry_run)
    if args.dry_run:  # one atomic write per rank (ranks share the pipe)
        sys.stdout.flush()
        os.write(1, (json.dumps(dry_run(args, dist)) + "\n").encode())
        dist.close()
        return
    if args.workload in MOE:
        r = run_moe_ep(args, dist, args.workload) if args.workload == "cfg5" else run_moe(args, dist, args.workload)
        r.update({"n_gpus": max(1, dist.world), "steps": args.steps, "warmup": 3,
                  "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None,
                  "data": "synthetic (reference generators, seed 0; random-init experts)",
                  "metric": METRIC, "gpu_launches": r["gpu_launches_per_step"] * args.steps})
        if dist.rank == 0:
            print(json.dumps(r), flush=True)
        dist.close()
        return
    out = run_ours(args, dist)
    if dist.rank == 0:
        print(json.dumps(out), flush=True)
    dist.close()


if __name__ == "__main__":
    main()
