"""Per-kernel counts of the SASS instructions that prove the tcgen05 / TMA /
TMEM path (UTCHMMA = tcgen05.mma, UTCBAR = tcgen05.commit, LDTM =
tcgen05.ld, UBLKCP = cp.async.bulk, UTCATOMSWS = tcgen05.alloc) in the built
libdynbatch.so, from `cuobjdump -sass`. Static instruction counts (the MMA
loops are not unrolled past the four K=16 steps of a 64-channel chunk).

usage: python profiles/sass_counts.py [lib.so] > profiles/r02_sass_counts.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ("UTCHMMA", "UTCBAR", "LDTM", "UBLKCP", "UTCATOMSWS", "SYNCS", "HMMA", "DFMA")


def main():
    lib = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "paper_1707_02402_b200", "libdynbatch.so")
    sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True, check=True).stdout
    counts, cur = collections.OrderedDict(), None
    arch = sorted(set(re.findall(r"arch = (sm_\w+)", sass)))
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            counts[cur] = collections.Counter()
            continue
        if cur:
            for op in OPS:
                if re.search(r"\b" + op + r"\b", line):
                    counts[cur][op] += 1
    print(f"# cuobjdump -sass {os.path.relpath(lib, ROOT)}  (arch: {', '.join(arch)})")
    print("# kernel | " + " ".join(OPS))
    for f, c in counts.items():
        if not any(c[o] for o in OPS):
            continue
        name = subprocess.run(["c++filt", f], capture_output=True, text=True).stdout.strip()
        name = re.sub(r"\(anonymous namespace\)::", "", name).split("(")[0] if "<" not in name else \
            re.sub(r"\(anonymous namespace\)::", "", name).split(">(")[0] + ">"
        print(f"{name:40s} | " + " ".join(f"{o}={c[o]}" for o in OPS if c[o]))


if __name__ == "__main__":
    main()
