"""Step-kernel time and effective SM clock per (DYNBATCH_CACHE,
DYNBATCH_LOOKAHEAD) setting, interleaved (cfg3). Cache bit 2 drops the
conv3x3 #2 tiles' interior mid lines from L2 once consumed (no write-back;
the default). Bits 0 and 1 selected streaming / evict-last store hints in
the round they were measured (no effect; since removed)."""
import os
import subprocess
import sys

here = os.path.dirname(os.path.abspath(__file__))
settings = [s.split(":") for s in (sys.argv[1:] or ["0:8", "4:8", "4:4", "4:2", "0:4", "0:8"])]
for cache, la in settings:
    env = dict(os.environ, DYNBATCH_CACHE=cache, DYNBATCH_LOOKAHEAD=la)
    out = subprocess.run([sys.executable, os.path.join(here, "step_waits.py")], env=env, capture_output=True,
                         text=True).stdout.strip().splitlines()
    print(f"cache={cache} lookahead={la}: {out[0][:40]} | {out[-1]}")
