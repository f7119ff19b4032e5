"""Interleaved A/B forward timing of library builds on one box:
python profiles/ab_time.py lib_a.so lib_b.so[:ENV=VAL,...] [...] [--rounds R]
[--batch B --bp P]. Each round runs each build (with its environment) in a
fresh process (chain programs, default cfg3; 10 timed forwards after 3
warm-ups, best of 3)."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r"""
import os, sys
sys.path.insert(0, %r)
import paper_1707_02402_b200 as db
F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=int(os.environ.get("AB_BATCH", "4096")), vocab=40, width=F, length=16,
                      branch_prob=float(os.environ.get("AB_BP", "0.3")), seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
print(min(s.time(10)[0] / 10 for _ in range(3)))
""" % ROOT

args = sys.argv[1:]
rounds = 3
extra = {}
for flag, env in (("--batch", "AB_BATCH"), ("--bp", "AB_BP")):
    if flag in args:
        i = args.index(flag)
        extra[env] = args[i + 1]
        args = args[:i] + args[i + 2:]
if "--rounds" in args:
    i = args.index("--rounds")
    rounds = int(args[i + 1])
    args = args[:i] + args[i + 2:]
libs = args
res = {l: [] for l in libs}
for _ in range(rounds):
    for l in libs:
        path, _, envs = l.partition(":")
        env = dict(os.environ, DYNBATCH_LIB=os.path.abspath(path), **extra)
        for kv in filter(None, envs.split(",")):
            k, _, v = kv.partition("=")
            env[k] = v
        out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        res[l].append(float(out.stdout.strip().splitlines()[-1]) if out.returncode == 0 else float("nan"))
for l in libs:
    v = sorted(res[l])
    print(f"{l}: ms/forward min {v[0]:.3f} median {v[len(v) // 2]:.3f}  all {[round(x, 3) for x in res[l]]}")
