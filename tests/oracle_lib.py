"""ctypes bindings for the CPU oracle — TEST INFRASTRUCTURE ONLY.

Two libraries, both built by ``oracle/Makefile``:

* ``oracle/liboracle.so`` — our plain-C restatement (``oracle/dynbatch_oracle.c``);
* ``oracle/_ref/libdbref.so`` — the unmodified reference C++ core
  (/root/reference/proj/src/*.cpp) plus ``oracle/ref_shim.cpp`` glue. It is
  built in the dev container and travels to the GPU box as a prebuilt file.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import
this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdbref.so")

P_I32 = C.POINTER(C.c_int32)
P_I64 = C.POINTER(C.c_int64)
P_F64 = C.POINTER(C.c_double)

_oracle = None
_ref = None


def _ptr(a, t):
    if a is None:
        return C.cast(None, t)
    return a.ctypes.data_as(t)


def oracle():
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        lib.orc_mix_seed.restype = C.c_uint64
        lib.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.orc_rng_u64.restype = C.c_uint64
        lib.orc_fnv1a64.restype = C.c_uint64
        lib.orc_fnv1a64.argtypes = [C.c_void_p, C.c_int64, C.c_uint64]
        lib.orc_gen_batch.restype = C.c_int64
        lib.orc_gen_batch.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_double,
                                      C.c_uint64, P_I32, P_I32, P_I32, P_I32, P_I32]
        lib.orc_random_batch.argtypes = [C.c_int64, C.c_int64, C.c_uint64, P_F64]
        lib.orc_random_rows.argtypes = [P_I64, C.c_int64, C.c_int64, C.c_uint64, P_F64]
        lib.orc_labels.argtypes = [C.c_int64, P_I32, P_I32, P_I32, P_I32, P_I32, P_I32]
        lib.orc_schedule_improved.argtypes = [C.c_int64, C.c_int, P_I32, P_I32, P_I32, P_I32, P_I32,
                                              P_I64, P_I32, P_I32, P_I32, P_I32, P_I32]
        lib.orc_execute.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                    P_I32, P_I32, P_I32, P_I32, P_I32, C.c_int64,
                                    P_I32, P_I32, P_I32, P_I32, P_I32, P_F64, C.c_uint64,
                                    P_F64, P_I64, P_I64, P_F64]
        lib.orc_resblock_weights.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int] + [P_F64] * 6
        lib.orc_dense_weights.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, P_F64, P_F64]
        lib.orc_topk.argtypes = [P_F64, C.c_int64, C.c_int64, C.c_int64, P_I32, P_F64]
        lib.orc_expert_weights.argtypes = [C.c_int64, C.c_int64, C.c_uint64, C.c_int64, P_F64, P_F64]
        lib.orc_moe_forward.argtypes = [P_F64, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                        P_I32, P_F64, C.c_uint64, P_I32, C.c_int64, P_F64, P_I64, P_F64]
        lib.orc_head_weights.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64] + [P_F64] * 6
        lib.orc_head_forward.argtypes = [C.c_int64, P_F64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_uint64,
                                         P_F64]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.refshim_gen_batch.restype = C.c_int64
        lib.refshim_gen_batch.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_double, C.c_uint64, P_I32, P_I32, P_I32, P_I32, P_I32,
                                          P_F64]
        lib.refshim_mix_seed.restype = C.c_uint64
        lib.refshim_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        lib.refshim_random_batch.argtypes = [C.c_int64, C.c_int64, C.c_uint64, P_F64]
        lib.refshim_schedule.argtypes = [C.c_int, C.c_int64, C.c_int, P_I32, P_I32, P_I32, P_I32,
                                         P_I32, P_I64, P_I32, P_I32, P_I32, P_I32, P_I32]
        lib.refshim_labels.argtypes = [C.c_int64, P_I32, P_I32, P_I32, P_I32, P_I32, P_I32]
        lib.refshim_execute.argtypes = [C.c_int, C.c_int64, C.c_int, C.c_int, P_I32, P_I32, P_I32,
                                        P_I32, P_I32, P_F64, C.c_uint64, P_F64, P_I64, P_I64, P_F64]
        lib.refshim_module_weights.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_int, P_F64, P_F64]
        lib.refshim_moe_inputs.argtypes = [C.c_int64, C.c_int64, C.c_int64, C.c_uint64, P_F64, P_F64]
        lib.refshim_topk.argtypes = [P_F64, C.c_int64, C.c_int64, C.c_int64, P_I32, P_F64]
        lib.refshim_moe_forward.argtypes = [P_F64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_int64, P_I32, P_F64, C.c_uint64, C.c_int, P_F64,
                                            P_I64, P_F64]
        lib.db_schedule_to_json.argtypes = [C.c_void_p, C.POINTER(C.c_char_p)]
        _ref = lib
    return _ref


# ------------------------------------------------------------------ batches --

KINDS = {"balanced": 0, "chain": 1, "dag": 2}


@dataclass
class Batch:
    """Program batch in CSR form (see oracle/dynbatch_oracle.h)."""

    prog_off: np.ndarray
    fid: np.ndarray
    child0: np.ndarray
    child1: np.ndarray
    root: np.ndarray
    p: int

    @property
    def b(self) -> int:
        return len(self.root)

    @property
    def n_nodes(self) -> int:
        return int(self.prog_off[-1]) if len(self.prog_off) else 0

    def args(self):
        return (_ptr(self.prog_off, P_I32), _ptr(self.fid, P_I32), _ptr(self.child0, P_I32),
                _ptr(self.child1, P_I32), _ptr(self.root, P_I32))


def _alloc_batch(b, n, p):
    return Batch(np.zeros(b + 1, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int32),
                 np.zeros(n, np.int32), np.zeros(b, np.int32), p)


def gen_batch(kind, b, p=40, depth=4, length=16, bp=0.1, seed=0) -> Batch:
    """orc_gen_batch — restated gen_batch (src/workload.cpp:214-246)."""
    lib = oracle()
    k = KINDS[kind] if isinstance(kind, str) else kind
    n = lib.orc_gen_batch(k, b, p, depth, length, bp, seed, None, None, None, None, None)
    bt = _alloc_batch(b, n, p)
    lib.orc_gen_batch(k, b, p, depth, length, bp, seed, *bt.args())
    return bt


def ref_gen_batch(kind, b, p=40, width=1, depth=4, length=16, bp=0.1, seed=0, with_inputs=False):
    """The reference's own gen_batch via the shim."""
    lib = ref()
    k = KINDS[kind] if isinstance(kind, str) else kind
    n = lib.refshim_gen_batch(k, b, p, width, depth, length, bp, seed, None, None, None, None,
                              None, None)
    bt = _alloc_batch(b, n, p)
    inputs = np.zeros((b, width), np.float64) if with_inputs else None
    lib.refshim_gen_batch(k, b, p, width, depth, length, bp, seed, *bt.args(), _ptr(inputs, P_F64))
    return (bt, inputs) if with_inputs else bt


def random_batch(rows, width, seed) -> np.ndarray:
    out = np.empty((rows, width), np.float64)
    oracle().orc_random_batch(rows, width, seed, _ptr(out, P_F64))
    return out


def random_rows(rows, width, seed) -> np.ndarray:
    """Rows `rows` (ascending) of random_batch(·, width, seed), generated in
    one pass without the rows in between."""
    r = np.ascontiguousarray(rows, np.int64)
    assert np.all(np.diff(r) > 0)
    out = np.zeros((len(r), width), np.float64)
    oracle().orc_random_rows(_ptr(r, P_I64), len(r), width, seed, _ptr(out, P_F64))
    return out


def mix_seed(seed, stream) -> int:
    return int(oracle().orc_mix_seed(seed, stream))


# ---------------------------------------------------------------- schedules --

@dataclass
class FlatSchedule:
    step_group_off: np.ndarray
    group_fid: np.ndarray
    group_member_off: np.ndarray
    member_example: np.ndarray
    member_node: np.ndarray
    strategy: str = "improved"

    @property
    def n_steps(self):
        return len(self.step_group_off) - 1

    @property
    def n_groups(self):
        return len(self.group_fid)

    def args(self):
        return (_ptr(self.step_group_off, P_I32), _ptr(self.group_fid, P_I32),
                _ptr(self.group_member_off, P_I32), _ptr(self.member_example, P_I32),
                _ptr(self.member_node, P_I32))

    def expensive_calls(self):
        return int(np.count_nonzero(self.group_fid != 0))

    def steps(self):
        """Nested python form: [[(fid, [(example, node), ...]), ...], ...]."""
        out = []
        for s in range(self.n_steps):
            groups = []
            for g in range(self.step_group_off[s], self.step_group_off[s + 1]):
                a, z = self.group_member_off[g], self.group_member_off[g + 1]
                groups.append((int(self.group_fid[g]),
                               list(zip(self.member_example[a:z].tolist(),
                                        self.member_node[a:z].tolist()))))
            out.append(groups)
        return out

    def __eq__(self, other):
        return all(np.array_equal(getattr(self, f), getattr(other, f)) for f in
                   ("step_group_off", "group_fid", "group_member_off", "member_example",
                    "member_node"))


def _alloc_sched(counts):
    s, g, m = (int(x) for x in counts)
    return FlatSchedule(np.zeros(s + 1, np.int32), np.zeros(g, np.int32), np.zeros(g + 1, np.int32),
                        np.zeros(m, np.int32), np.zeros(m, np.int32))


def schedule_improved(bt: Batch) -> FlatSchedule:
    lib = oracle()
    counts = np.zeros(3, np.int64)
    rc = lib.orc_schedule_improved(bt.b, bt.p, *bt.args(), _ptr(counts, P_I64), None, None, None,
                                   None, None)
    assert rc == 0, rc
    fs = _alloc_sched(counts)
    rc = lib.orc_schedule_improved(bt.b, bt.p, *bt.args(), _ptr(counts, P_I64), *fs.args())
    assert rc == 0, rc
    return fs


STRATEGIES = {"naive": 0, "standard": 1, "improved": 2, "online": 3}


def ref_schedule(bt: Batch, strategy="improved") -> FlatSchedule:
    lib = ref()
    counts = np.zeros(3, np.int64)
    rc = lib.refshim_schedule(STRATEGIES[strategy], bt.b, bt.p, *bt.args(), _ptr(counts, P_I64),
                              None, None, None, None, None)
    assert rc == 0, rc
    fs = _alloc_sched(counts)
    fs.strategy = strategy
    rc = lib.refshim_schedule(STRATEGIES[strategy], bt.b, bt.p, *bt.args(), _ptr(counts, P_I64),
                              *fs.args())
    assert rc == 0, rc
    return fs


def labels(bt: Batch, use_ref=False):
    out = np.zeros(bt.n_nodes, np.int32)
    dmax = np.zeros(1, np.int32)
    if use_ref:
        rc = ref().refshim_labels(bt.b, *bt.args(), _ptr(out, P_I32), _ptr(dmax, P_I32))
        return out, int(out.max()) if len(out) else 0
    rc = oracle().orc_labels(bt.b, bt.prog_off.ctypes.data_as(P_I32), _ptr(bt.child0, P_I32),
                             _ptr(bt.child1, P_I32), _ptr(bt.root, P_I32), _ptr(out, P_I32),
                             _ptr(dmax, P_I32))
    assert rc == 0
    return out, int(dmax[0])


def schedule_json(fs: FlatSchedule) -> str:
    """Byte-identical restatement of schedule_to_json (src/serialize.cpp:82-99),
    i.e. nlohmann::json::dump(2) of {"steps": [...], "strategy": "..."}."""
    parts = ['{\n  "steps": [']
    steps = fs.steps()
    if not steps:
        parts = ['{\n  "steps": [],\n  "strategy": "%s"\n}' % fs.strategy]
        return "".join(parts)
    step_strs = []
    for groups in steps:
        if not groups:
            step_strs.append("\n    []")
            continue
        gs = []
        for fid, members in groups:
            if members:
                ms = ",".join("\n          [\n            %d,\n            %d\n          ]" % m
                              for m in members)
                mem = "[" + ms + "\n        ]"
            else:
                mem = "[]"
            gs.append('\n      {\n        "function_id": %d,\n        "members": %s\n      }'
                      % (fid, mem))
        step_strs.append("\n    [" + ",".join(gs) + "\n    ]")
    parts.append(",".join(step_strs))
    parts.append('\n  ],\n  "strategy": "%s"\n}' % fs.strategy)
    return "".join(parts)


def fnv1a64(data: bytes) -> int:
    return int(oracle().orc_fnv1a64(data, len(data), 0))


# ---------------------------------------------------------------- execution --

@dataclass
class ExecOut:
    outputs: np.ndarray
    expensive_calls: int
    peak_group_rows: int
    steps: int
    per_function_calls: np.ndarray
    seconds: np.ndarray
    rc: int = 0


def execute(bt: Batch, fs: FlatSchedule, inputs: np.ndarray, module_seed: int, kind="dense",
            width=None, C=128, H=14, W=14) -> ExecOut:
    """orc_execute — restated execute (src/executor.cpp:95-176); kind "dense"
    (Tier A, pinned) or "resblock" (Tier B, parity unpinned)."""
    lib = oracle()
    mk = 0 if kind == "dense" else 1
    if mk == 1:
        width = C * H * W
    inputs = np.ascontiguousarray(inputs, np.float64)
    out = np.zeros((bt.b, width), np.float64)
    trace = np.zeros(3, np.int64)
    pfc = np.zeros(bt.p, np.int64)
    secs = np.zeros(3, np.float64)
    rc = lib.orc_execute(mk, bt.b, bt.p, width, C, H, W, *bt.args(), fs.n_steps, *fs.args(),
                         _ptr(inputs, P_F64), module_seed, _ptr(out, P_F64), _ptr(trace, P_I64),
                         _ptr(pfc, P_I64), _ptr(secs, P_F64))
    return ExecOut(out, int(trace[0]), int(trace[1]), int(trace[2]), pfc, secs, rc)


def ref_execute(bt: Batch, inputs: np.ndarray, width: int, module_seed: int,
                strategy="improved") -> ExecOut:
    lib = ref()
    inputs = np.ascontiguousarray(inputs, np.float64)
    out = np.zeros((bt.b, width), np.float64)
    trace = np.zeros(3, np.int64)
    pfc = np.zeros(bt.p, np.int64)
    secs = np.zeros(3, np.float64)
    rc = lib.refshim_execute(STRATEGIES[strategy], bt.b, bt.p, width, *bt.args(),
                             _ptr(inputs, P_F64), module_seed, _ptr(out, P_F64),
                             _ptr(trace, P_I64), _ptr(pfc, P_I64), _ptr(secs, P_F64))
    return ExecOut(out, int(trace[0]), int(trace[1]), int(trace[2]), pfc, secs, rc)


def resblock_weights(arity, C, seed, fid):
    w0 = np.zeros(2 * C * C); b0 = np.zeros(C)
    w1 = np.zeros(9 * C * C); b1 = np.zeros(C)
    w2 = np.zeros(9 * C * C); b2 = np.zeros(C)
    oracle().orc_resblock_weights(arity, C, seed, fid, *(_ptr(a, P_F64) for a in
                                                          (w0, b0, w1, b1, w2, b2)))
    return w0, b0, w1, b1, w2, b2


# ---------------------------------------------------------------------- MoE --

def moe_inputs(T, n, d, seed):
    """gen_moe_inputs (src/workload.cpp:248-254)."""
    return (random_batch(T, d, mix_seed(seed, 0x10)), random_batch(T, n, mix_seed(seed, 0x11)))


def topk(scores: np.ndarray, k: int, use_ref=False):
    T, n = scores.shape
    ids = np.zeros((T, k), np.int32)
    w = np.zeros((T, k), np.float64)
    s = np.ascontiguousarray(scores, np.float64)
    if use_ref:
        rc = ref().refshim_topk(_ptr(s, P_F64), T, n, k, _ptr(ids, P_I32), _ptr(w, P_F64))
    else:
        rc = oracle().orc_topk(_ptr(s, P_F64), T, n, k, _ptr(ids, P_I32), _ptr(w, P_F64))
    assert rc == 0, rc
    return ids, w


def expert_weights(d, h, expert_seed, eid):
    """ExpertSet expert `eid` (src/moe.cpp:71-88): w1 [d][h], w2 [h][d]."""
    w1 = np.zeros(d * h, np.float64)
    w2 = np.zeros(h * d, np.float64)
    oracle().orc_expert_weights(d, h, expert_seed, eid, _ptr(w1, P_F64), _ptr(w2, P_F64))
    return w1.reshape(d, h), w2.reshape(h, d)


def moe_forward(inputs, ids, weights, n, h, expert_seed, use_ref=False, subset=None, batched=True):
    T, d = inputs.shape
    k = ids.shape[1]
    out = np.zeros((T, d), np.float64)
    trace = np.zeros(3, np.int64)
    secs = np.zeros(3, np.float64)
    x = np.ascontiguousarray(inputs, np.float64)
    ids = np.ascontiguousarray(ids, np.int32)
    weights = np.ascontiguousarray(weights, np.float64)
    if use_ref:
        rc = ref().refshim_moe_forward(_ptr(x, P_F64), T, d, h, n, k, _ptr(ids, P_I32),
                                       _ptr(weights, P_F64), expert_seed, 1 if batched else 0, _ptr(out, P_F64),
                                       _ptr(trace, P_I64), _ptr(secs, P_F64))
    else:
        sub = None if subset is None else np.ascontiguousarray(subset, np.int32)
        rc = oracle().orc_moe_forward(_ptr(x, P_F64), T, d, h, n, k, _ptr(ids, P_I32),
                                      _ptr(weights, P_F64), expert_seed, _ptr(sub, P_I32),
                                      0 if sub is None else len(sub), _ptr(out, P_F64),
                                      _ptr(trace, P_I64), _ptr(secs, P_F64))
    assert rc == 0, rc
    return out, trace, secs


def schedule_naive(bt: Batch) -> FlatSchedule:
    """schedule_naive (src/schedule.cpp:94-105): one step per node, examples
    in order, each program's nodes in postorder_flatten order (children
    first, src/program.cpp:274-298). Python loops: small batches only (the
    bench's CPU naive sample and tests)."""
    sgo, gf, gmo, me, mn = [0], [], [0], [], []
    for e in range(bt.b):
        off = int(bt.prog_off[e])
        order, done, stack = [], set(), [[int(bt.root[e]), 0]]
        while stack:
            fr = stack[-1]
            kids = [c for c in (int(bt.child0[off + fr[0]]), int(bt.child1[off + fr[0]])) if c >= 0]
            if fr[1] < len(kids):
                c = kids[fr[1]]
                fr[1] += 1
                if c not in done:
                    stack.append([c, 0])
            else:
                done.add(fr[0])
                order.append(fr[0])
                stack.pop()
        for node in order:
            gf.append(int(bt.fid[off + node]))
            me.append(e)
            mn.append(node)
            gmo.append(len(me))
            sgo.append(len(gf))
    a = lambda v: np.asarray(v, np.int32)  # noqa: E731
    return FlatSchedule(a(sgo), a(gf), a(gmo), a(me), a(mn), "naive")


# ------------------------------------------------------------- IEP head --

HEAD = {"C": 128, "P": 512, "F": 1024}


def head_weights(A, seed, C=128, P=512, F=1024):
    """orc_head_weights: (wp [C][P], bp, w1 [49P][F], b1, w2 [F][A], b2)."""
    wp, bp = np.zeros(C * P), np.zeros(P)
    w1, b1 = np.zeros(49 * P * F), np.zeros(F)
    w2, b2 = np.zeros(F * A), np.zeros(A)
    oracle().orc_head_weights(C, P, F, A, seed, *(_ptr(a, P_F64) for a in (wp, bp, w1, b1, w2, b2)))
    return wp.reshape(C, P), bp, w1.reshape(49 * P, F), b1, w2.reshape(F, A), b2


def head_forward(roots: np.ndarray, A, seed, C=128, P=512, F=1024) -> np.ndarray:
    """orc_head_forward: logits [b][A] of CHW root rows (fp64)."""
    roots = np.ascontiguousarray(roots, np.float64)
    b = roots.shape[0]
    out = np.zeros((b, A), np.float64)
    rc = oracle().orc_head_forward(b, _ptr(roots, P_F64), C, P, F, A, seed, _ptr(out, P_F64))
    assert rc == 0, rc
    return out
