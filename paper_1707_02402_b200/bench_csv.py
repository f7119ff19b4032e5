"""bench-iep / bench-moe with the reference CLI's flags and CSV schemas
(tools/dynbatch_cli.cpp:109-262 and 264-358), run through this library's C
ABI, so tooling that reads the reference's benchmark CSVs reads device runs
unchanged.

    python -m paper_1707_02402_b200.bench_csv bench-iep --b 1,8,64,512 --width 64
    python -m paper_1707_02402_b200.bench_csv bench-moe --n 16,64 --k 4 --b 256

Same protocol as the reference: naive is the speedup reference; repetitions
are interleaved over the schedulers (rep-major), the first sweep is a
discarded warm-up, one repetition aggregates `inner` executions and rows are
medians; the static call-count bounds are checked on every row. Exit codes
follow the CLI (tools/dynbatch_cli.cpp:24-37): 0 ok, 1 usage (and
DB_ERR_INVALID_ARG), 2 verification or any other library error; messages go
to stderr as "error: …". Timings are this library's
db_run_{module,stacking,total}_seconds: device execution instead of the
reference's host loop.
"""
import argparse
import os
import sys

import numpy as np

from . import Batch, DynbatchError, moe_run

EXIT_OK, EXIT_USAGE, EXIT_VERIFICATION = 0, 1, 2
SHAPES = {"balanced-tree": "balanced", "chain-heavy": "chain", "random-dag": "dag"}
IEP_HEADER = "scheduler,b,p,s_max,d_max,calls,module_ms,stack_ms,total_ms,speedup\n"
MOE_HEADER = ("impl,n,k,b,data_dim,hidden,calls,expert_ms,stack_ms,total_ms,speedup,"
              "speedup_per_call\n")


class VerificationError(Exception):
    pass


def median(values):
    v = sorted(values)
    n = len(v)
    return v[n // 2] if n % 2 else 0.5 * (v[n // 2 - 1] + v[n // 2])


def check_call_bounds(scheduler, calls, st):
    """tools/dynbatch_cli.cpp:132-155."""
    if scheduler == "naive":
        ok, bound = calls == st.expensive_nodes, f"census {st.expensive_nodes}"
    elif scheduler == "standard":
        ok, bound = calls <= min(st.vocab, st.batch) * st.s_max, "min(p,b)*s_max"
    elif scheduler == "improved":
        ok, bound = calls <= st.vocab * (st.d_max + 1), "p*(d_max+1)"
    elif scheduler == "online":
        ok, bound = calls <= st.vocab * st.d_max, "p*d_max"
    else:
        ok, bound = True, ""
    if not ok:
        raise VerificationError(f"{scheduler} made {calls} expensive calls, violating bound {bound}")


def bench_iep(a, out):
    out.write(IEP_HEADER)
    rows = [[] for _ in a.schedulers]
    for b in a.b:
        batch = Batch.generate(SHAPES[a.shape], batch=b, vocab=a.p, width=a.width, depth=a.depth,
                               length=a.s, branch_prob=a.branch_prob, seed=a.seed)
        st = batch.stats()
        naive = batch.schedule("naive")
        scheds = [naive]
        for name in a.schedulers:
            if name == "naive":
                scheds.append(naive)
                continue
            s = batch.schedule(name)
            s.verify(batch)
            scheds.append(s)
        stats = [{"module": [], "stack": [], "total": [], "calls": 0} for _ in scheds]
        for rep in range(a.reps + 1):
            for si, s in enumerate(scheds):
                m = k = t = 0.0
                for _ in range(1 if rep == 0 else a.inner):
                    run = batch.execute(s, a.seed)
                    m += run.module_seconds
                    k += run.stacking_seconds
                    t += run.total_seconds
                    stats[si]["calls"] = run.expensive_calls
                if rep > 0:
                    stats[si]["module"].append(m)
                    stats[si]["stack"].append(k)
                    stats[si]["total"].append(t)
        naive_module = median(stats[0]["module"])
        for si, name in enumerate(a.schedulers):
            r = stats[si + 1]
            check_call_bounds(name, r["calls"], st)
            mod = median(r["module"])
            rows[si].append("%s,%d,%d,%d,%d,%d,%.6f,%.6f,%.6f,%.4f\n" % (
                name, st.batch, st.vocab, st.s_max, st.d_max, r["calls"], mod * 1e3 / a.inner,
                median(r["stack"]) * 1e3 / a.inner, median(r["total"]) * 1e3 / a.inner,
                naive_module / mod))
    for scheduler_rows in rows:
        for row in scheduler_rows:
            out.write(row)


def bench_moe(a, out):
    out.write(MOE_HEADER)
    for n in a.n:
        per = [{"expert": [], "stack": [], "total": [], "calls": 0} for _ in range(2)]
        max_rel = 0.0
        ref = None
        for rep in range(a.reps + 1):
            for batched in (0, 1):
                e = k = t = 0.0
                for p in range(1 if rep == 0 else a.inner):
                    run = moe_run(n, a.k, a.b, a.data_dim, a.hidden, a.seed, batched=bool(batched))
                    e += run.module_seconds
                    k += run.stacking_seconds
                    t += run.total_seconds
                    per[batched]["calls"] = run.expensive_calls
                    if rep == a.reps and p + 1 == a.inner:
                        y = run.outputs()
                        if batched == 0:
                            ref = y
                        else:
                            den = np.maximum(np.maximum(np.abs(ref), np.abs(y)), 1e-300)
                            max_rel = max(max_rel, float(np.max(np.abs(ref - y) / den)))
                if rep > 0:
                    per[batched]["expert"].append(e)
                    per[batched]["stack"].append(k)
                    per[batched]["total"].append(t)
        if max_rel > 1e-9:
            raise VerificationError(f"batched MOE outputs diverge from naive (rel {max_rel}) at n={n}")
        naive_med = median(per[0]["expert"])
        for batched in (0, 1):
            s = per[batched]
            med = median(s["expert"])
            per_call = (naive_med / per[0]["calls"]) / (med / s["calls"])
            out.write("%s,%d,%d,%d,%d,%d,%d,%.6f,%.6f,%.6f,%.4f,%.4f\n" % (
                "batched" if batched else "naive", n, a.k, a.b, a.data_dim, a.hidden, s["calls"],
                med * 1e3 / a.inner, median(s["stack"]) * 1e3 / a.inner, median(s["total"]) * 1e3 / a.inner,
                naive_med / med, per_call))


def _ints(text):
    return [int(x) for x in text.split(",") if x]


def _names(text):
    return [x for x in text.split(",") if x]


def parser():
    ap = argparse.ArgumentParser(prog="bench_csv")
    sub = ap.add_subparsers(dest="cmd", required=True)
    i = sub.add_parser("bench-iep")
    i.add_argument("--b", type=_ints, default=[1, 8, 64, 512])
    i.add_argument("--p", type=int, default=40)
    i.add_argument("--width", type=int, default=64)
    i.add_argument("--s", type=int, default=16)
    i.add_argument("--depth", type=int, default=5)
    i.add_argument("--branch-prob", type=float, default=0.1)
    i.add_argument("--shape", choices=list(SHAPES), default="chain-heavy")
    i.add_argument("--schedulers", type=_names, default=["naive", "standard", "improved"])
    i.add_argument("--reps", type=int, default=5)
    i.add_argument("--inner", type=int, default=1)
    i.add_argument("--seed", type=int, default=int(os.environ.get("DYNBATCH_SEED", 0)))
    i.add_argument("--out", default="-")
    m = sub.add_parser("bench-moe")
    m.add_argument("--n", type=_ints, default=[16, 64, 128, 256])
    m.add_argument("--k", type=int, default=4)
    m.add_argument("--b", type=int, default=256)
    m.add_argument("--data-dim", type=int, default=64)
    m.add_argument("--hidden", type=int, default=64)
    m.add_argument("--reps", type=int, default=5)
    m.add_argument("--inner", type=int, default=1)
    m.add_argument("--seed", type=int, default=int(os.environ.get("DYNBATCH_SEED", 0)))
    m.add_argument("--out", default="-")
    return ap


def main(argv=None):
    a = parser().parse_args(argv)
    for name in getattr(a, "schedulers", []):
        if name not in ("naive", "standard", "improved", "online"):
            print(f"error: unknown scheduler '{name}'", file=sys.stderr)
            return EXIT_USAGE
    out = sys.stdout if a.out in ("", "-") else open(a.out, "w")
    try:
        (bench_iep if a.cmd == "bench-iep" else bench_moe)(a, out)
    except VerificationError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_VERIFICATION
    except DynbatchError as e:
        print(f"error: {e}", file=sys.stderr)
        return EXIT_USAGE if getattr(e, "status", None) == 1 else EXIT_VERIFICATION
    finally:
        if out is not sys.stdout:
            out.close()
    return EXIT_OK


if __name__ == "__main__":
    sys.exit(main())
