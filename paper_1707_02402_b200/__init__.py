"""dynbatch-b200 — Python host mirror of the drop-in C ABI.

The product is ``libdynbatch.so`` (built in-tree from ``csrc/``): the
reference's 27 ``db_*`` entry points (include/dynbatch/dynbatch.h) plus device
sessions (include/dynbatch/dynbatch_device.h). This module only binds them
with ctypes, mirroring the reference's C API names, argument meaning and
error behaviour (every failing call raises :class:`DynbatchError` carrying
the ``db_status`` and ``db_last_error()`` text). There is no Python or CPU
compute path: if the shared library is missing this import fails loudly.
"""
from __future__ import annotations

import ctypes as C
import json
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DYNBATCH_LIB selects another build of the library (A/B timing of variants)
LIB_PATH = os.environ.get("DYNBATCH_LIB") or os.path.join(_HERE, "libdynbatch.so")

DB_OK = 0
STATUS = {0: "DB_OK", 1: "DB_ERR_INVALID_ARG", 2: "DB_ERR_UNKNOWN_FUNCTION",
          3: "DB_ERR_UNDERFULL_SEQUENCE", 4: "DB_ERR_OVERFULL_SEQUENCE",
          5: "DB_ERR_INVALID_PROGRAM", 6: "DB_ERR_DEPENDENCY_VIOLATION",
          7: "DB_ERR_MISSING_OPERAND", 8: "DB_ERR_SHAPE_MISMATCH", 9: "DB_ERR_NON_FINITE",
          10: "DB_ERR_PARSE", 11: "DB_ERR_VERIFICATION_FAILED", 12: "DB_ERR_INTERNAL"}
STRATEGY = {"naive": 0, "standard": 1, "improved": 2, "online": 3}
WORKLOAD = {"balanced": 0, "balanced-tree": 0, "chain": 1, "chain-heavy": 1, "dag": 2,
            "random-dag": 2}
MODULE_DENSE, MODULE_RESBLOCK = 0, 1
MOE_FP64, MOE_BF16, MOE_FP16 = 0, 1, 2


class DynbatchError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


class WorkloadOpts(C.Structure):
    _fields_ = [("kind", C.c_int), ("batch", C.c_int64), ("vocab", C.c_int32),
                ("width", C.c_int32), ("depth", C.c_int32), ("length", C.c_int32),
                ("branch_prob", C.c_double), ("seed", C.c_uint64)]


class BatchStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("batch", "vocab", "width", "s_max", "d_max",
                                         "total_nodes", "expensive_nodes")]


class MoeOpts(C.Structure):
    _fields_ = [("experts", C.c_int64), ("active_per_example", C.c_int64), ("batch", C.c_int64),
                ("data_dim", C.c_int64), ("hidden", C.c_int64), ("seed", C.c_uint64)]


class MemoryModel(C.Structure):
    _fields_ = [("param_count", C.c_int64), ("activation_count", C.c_double),
                ("memory_ratio", C.c_double)]


class VerifyOpts(C.Structure):
    _fields_ = [("seeds", C.c_int32), ("batch", C.c_int64), ("vocab", C.c_int32),
                ("length", C.c_int32), ("width", C.c_int32), ("seed", C.c_uint64),
                ("parallel", C.c_int32)]


class ModuleOpts(C.Structure):
    _fields_ = [("module_kind", C.c_int32), ("channels", C.c_int32), ("height", C.c_int32),
                ("width_px", C.c_int32), ("program_capacity", C.c_int64), ("node_capacity", C.c_int64),
                ("length_capacity", C.c_int32), ("reserved", C.c_int32)]


class SessionStats(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("steps", "groups", "expensive_calls", "peak_group_rows",
                                         "members", "kernel_launches", "h2d_bytes", "d2h_bytes")] + \
               [("algorithmic_flops", C.c_double), ("algorithmic_bytes", C.c_double)]


class KernelTimes(C.Structure):
    _fields_ = [("ms", C.c_double * 8), ("launches", C.c_int64 * 8), ("flops", C.c_double * 8),
                ("bytes", C.c_double * 8)]


# Profiler classes (db_kernel_times_t): IEP uses scheduler, plan, gather and
# the fused conv step (class 4); MoE uses gate+sort (3), GEMM1 (4), GEMM2 (5)
# and combine (6).
KERNEL_CLASSES = ["scheduler", "plan", "gather", "moe_gate_sort", "conv_step|moe_gemm1",
                  "moe_gemm2", "layout|combine", "dense_step"]

LOG_FN = C.CFUNCTYPE(None, C.c_char_p, C.c_void_p)
VP = C.c_void_p
PVP = C.POINTER(C.c_void_p)

# name -> (restype, argtypes); the 27 reference entry points first.
SIGNATURES = {
    "db_version": (C.c_char_p, []),
    "db_last_error": (C.c_char_p, []),
    "db_string_free": (None, [VP]),
    "db_batch_generate": (C.c_int32, [C.POINTER(WorkloadOpts), PVP]),
    "db_batch_load_json": (C.c_int32, [C.c_char_p, C.c_int32, C.c_uint64, PVP]),
    "db_batch_to_json": (C.c_int32, [VP, PVP]),
    "db_batch_stats": (C.c_int32, [VP, C.POINTER(BatchStats)]),
    "db_batch_free": (None, [VP]),
    "db_schedule_build": (C.c_int32, [VP, C.c_int, PVP]),
    "db_schedule_build_device": (C.c_int32, [VP, C.c_int, PVP]),
    "db_schedule_verify": (C.c_int32, [VP, VP]),
    "db_schedule_step_count": (C.c_int64, [VP]),
    "db_schedule_expensive_calls": (C.c_int32, [VP, VP, C.POINTER(C.c_int64)]),
    "db_schedule_to_json": (C.c_int32, [VP, PVP]),
    "db_schedule_inject_fault": (C.c_int32, [VP, C.c_char_p]),
    "db_schedule_free": (None, [VP]),
    "db_execute": (C.c_int32, [VP, VP, C.c_uint64, PVP]),
    "db_run_outputs": (C.c_int32, [VP, C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)]),
    "db_run_expensive_calls": (C.c_int64, [VP]),
    "db_run_peak_group_rows": (C.c_int64, [VP]),
    "db_run_module_seconds": (C.c_double, [VP]),
    "db_run_stacking_seconds": (C.c_double, [VP]),
    "db_run_total_seconds": (C.c_double, [VP]),
    "db_run_trace_json": (C.c_int32, [VP, PVP]),
    "db_run_free": (None, [VP]),
    "db_moe_run": (C.c_int32, [C.POINTER(MoeOpts), C.c_int32, PVP]),
    "db_moe_memory_model": (C.c_int32, [C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_double,
                                        C.POINTER(MemoryModel)]),
    "db_verify_run": (C.c_int32, [C.POINTER(VerifyOpts), LOG_FN, VP]),
    # device extensions (dynbatch_device.h)
    "db_device_count": (C.c_int32, []),
    "db_device_open": (C.c_int32, [C.c_int32]),
    "db_host_alloc": (VP, [C.c_int64]),
    "db_host_free": (None, [VP]),
    "db_batch_generate_range": (C.c_int32, [C.POINTER(WorkloadOpts), C.c_int64, C.c_int64, PVP]),
    "db_batch_inputs": (C.c_int32, [VP, C.POINTER(C.POINTER(C.c_double)), C.POINTER(C.c_int64),
                                    C.POINTER(C.c_int64)]),
    "db_iep_session_time": (C.c_int32, [VP, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                        C.POINTER(KernelTimes)]),
    "db_moe_session_time": (C.c_int32, [VP, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                        C.POINTER(KernelTimes)]),
    "db_iep_session_create": (C.c_int32, [VP, C.c_int64, C.c_int64, C.c_uint64,
                                          C.POINTER(ModuleOpts), PVP]),
    "db_iep_session_set_schedule": (C.c_int32, [VP, VP]),
    "db_iep_session_set_strategy": (C.c_int32, [VP, C.c_int]),
    "db_iep_session_forward": (C.c_int32, [VP]),
    "db_iep_session_forward_host": (C.c_int32, [VP, VP, VP]),
    "db_iep_session_forward_host_async": (C.c_int32, [VP, VP, VP]),
    "db_iep_session_set_programs": (C.c_int32, [VP, VP, VP, C.c_int64]),
    "db_iep_session_synchronize": (C.c_int32, [VP]),
    "db_iep_session_stream": (VP, [VP]),
    "db_iep_session_stats": (C.c_int32, [VP, C.POINTER(SessionStats)]),
    "db_iep_session_schedule": (C.c_int32, [VP, PVP]),
    "db_iep_session_run": (C.c_int32, [VP, PVP]),
    "db_iep_session_labels": (C.c_int32, [VP, VP, C.c_int64]),
    "db_iep_session_set_head": (C.c_int32, [VP, C.c_int32, C.c_uint64]),
    "db_iep_session_head_forward": (C.c_int32, [VP]),
    "db_iep_session_logits": (C.c_int32, [VP, VP, C.c_int64]),
    "db_iep_session_forward_logits_host": (C.c_int32, [VP, VP, VP]),
    "db_iep_session_time_head": (C.c_int32, [VP, C.c_int32, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "db_iep_session_set_training": (C.c_int32, [VP, C.c_int32]),
    "db_iep_session_train_step": (C.c_int32, [VP, VP, C.POINTER(C.c_float)]),
    "db_iep_session_grad_size": (C.c_int32, [VP, C.c_int32, C.c_int32, C.POINTER(C.c_int64)]),
    "db_iep_session_grad": (C.c_int32, [VP, C.c_int32, C.c_int32, VP, C.c_int64]),
    "db_iep_session_time_train": (C.c_int32, [VP, C.c_int32, VP, C.POINTER(C.c_double)]),
    "db_iep_session_sgd": (C.c_int32, [VP, C.c_float]),
    "db_iep_session_free": (None, [VP]),
    "db_execute_device": (C.c_int32, [VP, VP, C.c_uint64, C.POINTER(ModuleOpts), PVP]),
    "db_moe_session_create": (C.c_int32, [C.POINTER(MoeOpts), C.c_int32, C.c_int64, C.c_int64,
                                          PVP]),
    "db_moe_session_forward": (C.c_int32, [VP]),
    "db_moe_session_forward_host": (C.c_int32, [VP, VP, VP, VP]),
    "db_moe_session_synchronize": (C.c_int32, [VP]),
    "db_moe_session_forward_host_async": (C.c_int32, [VP, VP, VP, VP]),
    "db_moe_session_stream": (VP, [VP]),
    "db_moe_session_stats": (C.c_int32, [VP, C.POINTER(SessionStats)]),
    "db_moe_session_routing": (C.c_int32, [VP, VP, VP, VP, VP]),
    "db_moe_session_run": (C.c_int32, [VP, PVP]),
    "db_moe_session_outputs": (C.c_int32, [VP, VP, C.c_int64, VP]),
    "db_moe_session_free": (None, [VP]),
    "db_moe_ep_create": (C.c_int32, [C.POINTER(MoeOpts), C.c_int32, C.c_int32, C.c_int32, PVP]),
    "db_moe_ep_sizes": (C.c_int32, [VP, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int32)]),
    "db_moe_ep_dispatch": (C.c_int32, [VP, VP, VP]),
    "db_moe_ep_experts": (C.c_int32, [VP, VP, VP, VP]),
    "db_moe_ep_layout": (C.c_int32, [VP, VP]),
    "db_moe_ep_forward_local": (C.c_int32, [VP]),
    "db_moe_ep_experts_range": (C.c_int32, [VP, VP, VP, C.c_int32, C.c_int32]),
    "db_moe_ep_combine": (C.c_int32, [VP, VP]),
    "db_moe_ep_outputs": (C.c_int32, [VP, VP]),
    "db_moe_ep_synchronize": (C.c_int32, [VP]),
    "db_moe_ep_stream": (VP, [VP]),
    "db_moe_ep_free": (None, [VP]),
    "db_moe_ep_nccl_id": (C.c_int32, [VP]),
    "db_moe_ep_comm_init": (C.c_int32, [VP, VP]),
    "db_moe_ep_forward": (C.c_int32, [VP, C.c_int32]),
    "db_moe_ep_recv_rows": (C.c_int32, [VP, C.POINTER(C.c_int64)]),
    "db_moe_ep_plan": (C.c_int32, [C.c_int32, C.c_int32, VP, VP, C.c_int32, C.POINTER(C.c_int32), VP, VP, VP, VP]),
    "db_moe_run_device": (C.c_int32, [C.POINTER(MoeOpts), C.c_int32, PVP]),
}

_lib = None


def lib():
    """Loads libdynbatch.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python __graft_entry__.py build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name, None)
            if fn is None and "DYNBATCH_LIB" in os.environ:
                continue  # an older build under A/B timing (profiles/ab_time.py)
            if fn is None:
                raise ImportError(f"{LIB_PATH} does not export {name}: rebuild it")
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def last_error() -> str:
    return lib().db_last_error().decode()


def check(status: int):
    if status != DB_OK:
        raise DynbatchError(status, last_error())


def _take_string(p: C.c_void_p) -> str:
    s = C.cast(p, C.c_char_p).value.decode()
    lib().db_string_free(p)
    return s


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Handle:
    _free = None

    def __init__(self, h):
        self.h = h

    def close(self):
        if self.h:
            getattr(lib(), self._free)(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Batch(_Handle):
    """db_batch: vocabulary + programs + seeded input rows."""
    _free = "db_batch_free"

    @classmethod
    def generate(cls, kind="chain", batch=8, vocab=40, width=128, depth=4, length=16,
                 branch_prob=0.1, seed=0):
        o = WorkloadOpts(WORKLOAD[kind] if isinstance(kind, str) else kind, batch, vocab, width,
                         depth, length, branch_prob, seed)
        h = C.c_void_p()
        check(lib().db_batch_generate(C.byref(o), C.byref(h)))
        return cls(h)

    @classmethod
    def generate_range(cls, first, last, kind="chain", batch=8, vocab=40, width=128, depth=4,
                       length=16, branch_prob=0.1, seed=0):
        """Programs [first, last) of generate(...), bit-identical to those rows."""
        o = WorkloadOpts(WORKLOAD[kind] if isinstance(kind, str) else kind, batch, vocab, width,
                         depth, length, branch_prob, seed)
        h = C.c_void_p()
        check(lib().db_batch_generate_range(C.byref(o), first, last, C.byref(h)))
        return cls(h)

    @classmethod
    def from_json(cls, text: str, width: int, input_seed: int):
        h = C.c_void_p()
        check(lib().db_batch_load_json(text.encode(), width, input_seed, C.byref(h)))
        return cls(h)

    def to_json(self) -> str:
        p = C.c_void_p()
        check(lib().db_batch_to_json(self.h, C.byref(p)))
        return _take_string(p)

    def stats(self) -> BatchStats:
        s = BatchStats()
        check(lib().db_batch_stats(self.h, C.byref(s)))
        return s

    def inputs(self) -> np.ndarray:
        d = C.POINTER(C.c_double)()
        r, w = C.c_int64(), C.c_int64()
        check(lib().db_batch_inputs(self.h, C.byref(d), C.byref(r), C.byref(w)))
        if r.value * w.value == 0:
            return np.zeros((r.value, w.value))
        return np.ctypeslib.as_array(d, shape=(r.value, w.value)).copy()

    def prefix_tokens(self):
        """The programs as concatenated prefix function sequences and their
        offsets (the JSON wire format's programs, src/serialize.cpp:37-80)."""
        progs = json.loads(self.to_json())["programs"]
        off = np.zeros(len(progs) + 1, np.int32)
        off[1:] = np.cumsum([len(p) for p in progs])
        toks = np.fromiter((f for p in progs for f in p), np.int32, count=int(off[-1]))
        return toks, off

    def schedule(self, strategy="improved") -> "Schedule":
        h = C.c_void_p()
        check(lib().db_schedule_build(self.h, STRATEGY[strategy], C.byref(h)))
        return Schedule(h)

    def schedule_device(self, strategy="improved") -> "Schedule":
        """The schedule built by the device scheduler (improved, standard or online)."""
        h = C.c_void_p()
        check(lib().db_schedule_build_device(self.h, STRATEGY[strategy], C.byref(h)))
        return Schedule(h)

    def execute(self, schedule: "Schedule", module_seed: int) -> "Run":
        h = C.c_void_p()
        check(lib().db_execute(self.h, schedule.h, module_seed, C.byref(h)))
        return Run(h)

    def execute_device(self, module_seed: int, module_kind=MODULE_DENSE, schedule=None) -> "Run":
        h = C.c_void_p()
        opts = ModuleOpts(module_kind, 128, 14, 14)
        check(lib().db_execute_device(self.h, schedule.h if schedule else None, module_seed,
                                      C.byref(opts), C.byref(h)))
        return Run(h)


class Schedule(_Handle):
    _free = "db_schedule_free"

    def verify(self, batch: Batch):
        check(lib().db_schedule_verify(self.h, batch.h))

    def step_count(self) -> int:
        return lib().db_schedule_step_count(self.h)

    def expensive_calls(self, batch: Batch) -> int:
        v = C.c_int64()
        check(lib().db_schedule_expensive_calls(self.h, batch.h, C.byref(v)))
        return v.value

    def to_json(self) -> str:
        p = C.c_void_p()
        check(lib().db_schedule_to_json(self.h, C.byref(p)))
        return _take_string(p)

    def inject_fault(self, kind: str):
        check(lib().db_schedule_inject_fault(self.h, kind.encode()))


class Run(_Handle):
    _free = "db_run_free"

    def outputs(self) -> np.ndarray:
        d = C.POINTER(C.c_double)()
        r, w = C.c_int64(), C.c_int64()
        check(lib().db_run_outputs(self.h, C.byref(d), C.byref(r), C.byref(w)))
        if r.value * w.value == 0:
            return np.zeros((r.value, w.value))
        return np.ctypeslib.as_array(d, shape=(r.value, w.value)).copy()

    @property
    def expensive_calls(self):
        return lib().db_run_expensive_calls(self.h)

    @property
    def peak_group_rows(self):
        return lib().db_run_peak_group_rows(self.h)

    @property
    def module_seconds(self) -> float:
        return lib().db_run_module_seconds(self.h)

    @property
    def stacking_seconds(self) -> float:
        return lib().db_run_stacking_seconds(self.h)

    @property
    def total_seconds(self) -> float:
        return lib().db_run_total_seconds(self.h)

    def trace_json(self) -> str:
        p = C.c_void_p()
        check(lib().db_run_trace_json(self.h, C.byref(p)))
        return _take_string(p)


def moe_run(experts, k, batch, data_dim, hidden, seed=0, batched=True) -> Run:
    o = MoeOpts(experts, k, batch, data_dim, hidden, seed)
    h = C.c_void_p()
    check(lib().db_moe_run(C.byref(o), 1 if batched else 0, C.byref(h)))
    return Run(h)


def moe_memory_model(experts, k, hidden, data_dim, m) -> MemoryModel:
    out = MemoryModel()
    check(lib().db_moe_memory_model(experts, k, hidden, data_dim, m, C.byref(out)))
    return out


def verify_run(seeds=6, batch=6, vocab=9, length=10, width=8, seed=0, parallel=False, log=None):
    lines = []

    def _cb(line, _user):
        lines.append(line.decode())
        if log:
            log(line.decode())

    cb = LOG_FN(_cb)
    o = VerifyOpts(seeds, batch, vocab, length, width, seed, 1 if parallel else 0)
    st = lib().db_verify_run(C.byref(o), cb, None)
    return st, lines


class IepSession(_Handle):
    """Device-resident IEP batch: forward = device scheduler + step kernels."""
    _free = "db_iep_session_free"
    _time = "db_iep_session_time"

    def __init__(self, batch: Batch, module_seed: int, module_kind=MODULE_DENSE, first=0, last=0,
                 program_capacity=0, node_capacity=0, length_capacity=0):
        h = C.c_void_p()
        opts = ModuleOpts(module_kind, 128, 14, 14, program_capacity, node_capacity, length_capacity, 0)
        check(lib().db_iep_session_create(batch.h, first, last, module_seed, C.byref(opts),
                                          C.byref(h)))
        super().__init__(h)

    def time(self, iters: int, profile=False):
        """Device ms of `iters` forwards (CUDA events on the session stream)
        and, with profile, per-kernel-class times: True / 1 = events around
        every launch (direct launches); 2 = the unprofiled forwards (graph
        replays) with events around the fused step kernel only (class 4)."""
        ms = C.c_double()
        kt = KernelTimes()
        check(getattr(lib(), self._time)(self.h, iters, int(profile), C.byref(ms), C.byref(kt)))
        return ms.value, kt

    def set_schedule(self, schedule):
        check(lib().db_iep_session_set_schedule(self.h, schedule.h if schedule else None))

    def set_strategy(self, strategy: str):
        """Device scheduler strategy for every forward: improved, standard or online."""
        check(lib().db_iep_session_set_strategy(self.h, STRATEGY[strategy]))

    def set_programs(self, tokens: np.ndarray, seq_off: np.ndarray):
        """Replace the programs by prefix function sequences (concatenated
        tokens, offsets[b+1]); the CSR is built on the device."""
        t = np.ascontiguousarray(tokens, np.int32)
        o = np.ascontiguousarray(seq_off, np.int32)
        check(lib().db_iep_session_set_programs(self.h, _ptr(t), _ptr(o), len(o) - 1))

    def forward(self):
        check(lib().db_iep_session_forward(self.h))

    def forward_host_async(self, inputs: np.ndarray, outputs: np.ndarray):
        """Pipelined forward_host (overlaps the copies with the neighbouring
        calls' forwards); keep the arrays alive until synchronize()."""
        check(lib().db_iep_session_forward_host_async(self.h, _ptr(inputs), _ptr(outputs)))

    def forward_host(self, inputs: np.ndarray, outputs: np.ndarray):
        check(lib().db_iep_session_forward_host(self.h, _ptr(inputs), _ptr(outputs)))

    def synchronize(self):
        check(lib().db_iep_session_synchronize(self.h))

    @property
    def stream(self) -> int:
        return lib().db_iep_session_stream(self.h) or 0

    def stats(self) -> SessionStats:
        s = SessionStats()
        check(lib().db_iep_session_stats(self.h, C.byref(s)))
        return s

    def schedule(self) -> Schedule:
        h = C.c_void_p()
        check(lib().db_iep_session_schedule(self.h, C.byref(h)))
        return Schedule(h)

    def run(self) -> Run:
        h = C.c_void_p()
        check(lib().db_iep_session_run(self.h, C.byref(h)))
        return Run(h)

    def labels(self, n_nodes: int) -> np.ndarray:
        out = np.zeros(n_nodes, np.int32)
        check(lib().db_iep_session_labels(self.h, _ptr(out), n_nodes))
        return out

    # IEP classifier head (db_iep_session_set_head …): conv1x1 → pool → FC → FC
    def set_head(self, answers: int = 28, seed: int = 0):
        check(lib().db_iep_session_set_head(self.h, answers, seed))
        self._answers = answers

    def head_forward(self):
        check(lib().db_iep_session_head_forward(self.h))

    def logits(self, b: int) -> np.ndarray:
        out = np.zeros((b, self._answers), np.float32)
        check(lib().db_iep_session_logits(self.h, _ptr(out), out.size))
        return out

    def forward_logits_host(self, inputs: np.ndarray, logits: np.ndarray):
        check(lib().db_iep_session_forward_logits_host(self.h, _ptr(inputs), _ptr(logits)))

    # training (db_iep_session_set_training …)
    GRADS = ("w0", "b0", "w1", "b1", "w2", "b2", "head_wp", "head_bp", "head_w1", "head_b1", "head_w2",
             "head_b2", "inputs")

    def set_training(self, on: bool = True):
        check(lib().db_iep_session_set_training(self.h, 1 if on else 0))

    def train_step(self, labels) -> float:
        lab = np.ascontiguousarray(labels, np.int32)
        loss = C.c_float()
        check(lib().db_iep_session_train_step(self.h, _ptr(lab), C.byref(loss)))
        return loss.value

    def grad(self, name: str, fid: int = -1) -> np.ndarray:
        which = self.GRADS.index(name)
        n = C.c_int64()
        check(lib().db_iep_session_grad_size(self.h, which, fid, C.byref(n)))
        out = np.zeros(n.value, np.float32)
        check(lib().db_iep_session_grad(self.h, which, fid, _ptr(out), n.value))
        return out

    def time_train(self, iters: int, labels) -> float:
        lab = np.ascontiguousarray(labels, np.int32)
        ms = C.c_double()
        check(lib().db_iep_session_time_train(self.h, iters, _ptr(lab), C.byref(ms)))
        return ms.value

    def sgd(self, lr: float):
        """w -= lr·grad for every module and head weight and bias, with the
        last train_step's gradients; the next forward uses the new weights."""
        check(lib().db_iep_session_sgd(self.h, float(lr)))

    def time_head(self, iters: int):
        """(device ms per head forward, algorithmic FLOPs per head forward)."""
        ms, fl = C.c_double(), C.c_double()
        check(lib().db_iep_session_time_head(self.h, iters, C.byref(ms), C.byref(fl)))
        return ms.value, fl.value


class MoeSession(_Handle):
    _free = "db_moe_session_free"
    _time = "db_moe_session_time"

    def __init__(self, experts, k, batch, data_dim, hidden, seed=0, precision=MOE_BF16, first=0,
                 last=0):
        o = MoeOpts(experts, k, batch, data_dim, hidden, seed)
        h = C.c_void_p()
        check(lib().db_moe_session_create(C.byref(o), precision, first, last, C.byref(h)))
        super().__init__(h)
        self.n, self.k, self.d = experts, k, data_dim
        self.T = (last - first) if last > first else batch

    def forward(self):
        check(lib().db_moe_session_forward(self.h))

    def time(self, iters: int, profile: bool = False):
        """Device ms of `iters` forwards (CUDA events on the session stream)
        and, with profile, per-kernel-class times."""
        ms = C.c_double()
        kt = KernelTimes()
        check(getattr(lib(), self._time)(self.h, iters, 1 if profile else 0, C.byref(ms),
                                         C.byref(kt)))
        return ms.value, kt

    def forward_host(self, inputs, scores, outputs):
        check(lib().db_moe_session_forward_host(self.h, _ptr(inputs), _ptr(scores), _ptr(outputs)))

    def forward_host_async(self, inputs, scores, outputs):
        """Pipelined forward_host (pinned buffers; results after synchronize())."""
        check(lib().db_moe_session_forward_host_async(self.h, _ptr(inputs), _ptr(scores), _ptr(outputs)))

    def synchronize(self):
        check(lib().db_moe_session_synchronize(self.h))

    @property
    def stream(self) -> int:
        return lib().db_moe_session_stream(self.h) or 0

    def stats(self) -> SessionStats:
        s = SessionStats()
        check(lib().db_moe_session_stats(self.h, C.byref(s)))
        return s

    def routing(self):
        ids = np.zeros((self.T, self.k), np.int32)
        w = np.zeros((self.T, self.k), np.float64)
        off = np.zeros(self.n + 1, np.int32)
        items = np.zeros(self.T * self.k, np.int32)
        check(lib().db_moe_session_routing(self.h, _ptr(ids), _ptr(w), _ptr(off), _ptr(items)))
        return ids, w, off, items

    def run(self) -> Run:
        h = C.c_void_p()
        check(lib().db_moe_session_run(self.h, C.byref(h)))
        return Run(h)

    def outputs(self, rows=None) -> np.ndarray:
        """fp32 output rows of the last forward (all, or the given tokens)."""
        if rows is None:
            out = np.zeros((self.T, self.d), np.float32)
            check(lib().db_moe_session_outputs(self.h, None, self.T, _ptr(out)))
            return out
        r = np.ascontiguousarray(rows, np.int64)
        out = np.zeros((len(r), self.d), np.float32)
        check(lib().db_moe_session_outputs(self.h, _ptr(r), len(r), _ptr(out)))
        return out


class MoeEpSession(_Handle):
    """One rank of the expert-parallel MoE layer (db_moe_ep_*): tokens
    [rank·T/G, (rank+1)·T/G) and experts [rank·n/G, (rank+1)·n/G). Buffers
    are device pointers (e.g. torch CUDA tensors' data_ptr()); the exchange
    between the stages is the caller's (paper_1707_02402_b200.moe_ep)."""
    _free = "db_moe_ep_free"

    def __init__(self, experts, k, batch, data_dim, hidden, seed=0, rank=0, world=1, precision=MOE_FP16):
        o = MoeOpts(experts, k, batch, data_dim, hidden, seed)
        h = C.c_void_p()
        check(lib().db_moe_ep_create(C.byref(o), precision, rank, world, C.byref(h)))
        super().__init__(h)
        self.n, self.k, self.d, self.rank, self.world = experts, k, data_dim, rank, world
        self.precision = precision
        t, it, e = C.c_int64(), C.c_int64(), C.c_int32()
        check(lib().db_moe_ep_sizes(self.h, C.byref(t), C.byref(it), C.byref(e)))
        self.tokens, self.items, self.local_experts = t.value, it.value, e.value

    def dispatch(self, send_ptr: int) -> np.ndarray:
        """Gate + sort + pack into send_ptr; returns rows per global expert."""
        counts = np.zeros(self.n, np.int32)
        check(lib().db_moe_ep_dispatch(self.h, C.c_void_p(send_ptr), _ptr(counts)))
        return counts

    def experts(self, recv_ptr: int, recv_counts: np.ndarray, ret_ptr: int):
        cnt = np.ascontiguousarray(recv_counts, np.int32).reshape(self.world, self.local_experts)
        check(lib().db_moe_ep_experts(self.h, C.c_void_p(recv_ptr), _ptr(cnt), C.c_void_p(ret_ptr)))

    def forward_local(self):
        """World 1: the whole layer in one device pass (no exchange)."""
        check(lib().db_moe_ep_forward_local(self.h))

    def layout(self, recv_counts: np.ndarray):
        """Receive-side layout for the chunked form of experts()."""
        cnt = np.ascontiguousarray(recv_counts, np.int32).reshape(self.world, self.local_experts)
        check(lib().db_moe_ep_layout(self.h, _ptr(cnt)))

    def experts_range(self, recv_ptr: int, ret_ptr: int, e_begin: int, e_end: int):
        """Local experts [e_begin, e_end) only (after layout())."""
        check(lib().db_moe_ep_experts_range(self.h, C.c_void_p(recv_ptr), C.c_void_p(ret_ptr), e_begin, e_end))

    def combine(self, ret_ptr: int):
        check(lib().db_moe_ep_combine(self.h, C.c_void_p(ret_ptr)))

    def comm_init(self, unique_id: bytes):
        """Join the ranks' NCCL communicator (id from moe_ep_nccl_id on rank 0)."""
        buf = (C.c_char * 128).from_buffer_copy(bytes(unique_id))
        check(lib().db_moe_ep_comm_init(self.h, buf))

    def forward(self, chunks: int = 1):
        """The whole layer, exchange on the library's NCCL communicator."""
        check(lib().db_moe_ep_forward(self.h, chunks))

    @property
    def recv_rows(self) -> int:
        r = C.c_int64()
        check(lib().db_moe_ep_recv_rows(self.h, C.byref(r)))
        return r.value

    def outputs(self) -> np.ndarray:
        out = np.zeros((self.tokens, self.d), np.float32)
        check(lib().db_moe_ep_outputs(self.h, _ptr(out)))
        return out

    def synchronize(self):
        check(lib().db_moe_ep_synchronize(self.h))

    @property
    def stream(self) -> int:
        return lib().db_moe_ep_stream(self.h) or 0


def moe_ep_nccl_id() -> bytes:
    """A fresh 128-byte NCCL unique id (ncclGetUniqueId), for rank 0."""
    buf = (C.c_char * 128)()
    check(lib().db_moe_ep_nccl_id(buf))
    return bytes(buf)


def moe_ep_plan(G, E, send_counts, recv_counts, chunks):
    """The exchange plan (db_moe_ep_plan): (send_off, send_rows, recv_off,
    recv_rows), each [C][G]."""
    sc = np.ascontiguousarray(send_counts, np.int32).reshape(-1)
    rc = np.ascontiguousarray(recv_counts, np.int32).reshape(-1)
    cmax = max(1, min(int(chunks), int(E)))
    outs = [np.zeros((cmax, G), np.int64) for _ in range(4)]
    nc = C.c_int32()
    check(lib().db_moe_ep_plan(G, E, _ptr(sc), _ptr(rc), chunks, C.byref(nc), *(_ptr(o) for o in outs)))
    return tuple(o[:nc.value] for o in outs)


def device_count() -> int:
    return lib().db_device_count()


def device_open(device: int):
    check(lib().db_device_open(device))


class PinnedArray:
    """numpy view of page-locked host memory from db_host_alloc."""

    def __init__(self, shape, dtype=np.float32):
        dtype = np.dtype(dtype)
        n = int(np.prod(shape)) * dtype.itemsize
        self.ptr = lib().db_host_alloc(n)
        if not self.ptr:
            raise MemoryError("db_host_alloc failed")
        buf = (C.c_char * n).from_address(self.ptr)
        self.array = np.frombuffer(buf, dtype=dtype).reshape(shape)

    def __del__(self):
        try:
            if self.ptr:
                self.array = None
                lib().db_host_free(self.ptr)
                self.ptr = None
        except Exception:
            pass


def conv_wait_counters(reset=False, enable=True):
    """MMA-thread wait cycles of the conv kernels (diagnostics)."""
    lib().db_debug_conv_waits.restype = C.c_int32
    lib().db_debug_conv_waits.argtypes = [VP, C.c_int32, C.c_int32]
    out = np.zeros(64, np.uint64)
    check(lib().db_debug_conv_waits(_ptr(out), 1 if reset else 0, 1 if enable else 0))
    return out.reshape(16, 4)
