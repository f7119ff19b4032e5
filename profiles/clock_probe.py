"""SM clock, power and throttle reasons while cfg3 forwards run back to back
(~6 s), sampled by nvidia-smi every 50 ms; with DYNBATCH_DIAG it shows how
the epilogue's stores move power and clocks."""
import os
import subprocess
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1707_02402_b200 as db  # noqa: E402

F = 128 * 14 * 14
b = db.Batch.generate("chain", batch=4096, vocab=40, width=F, length=16, branch_prob=0.3, seed=0)
s = db.IepSession(b, 1234, db.MODULE_RESBLOCK)
s.time(3)
rows = []
stop = threading.Event()


def sample():
    q = "clocks.sm,power.draw,clocks_throttle_reasons.active,temperature.gpu"
    while not stop.is_set():
        out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", "0"],
                             capture_output=True, text=True).stdout.strip()
        rows.append(out)
        time.sleep(0.05)


t = threading.Thread(target=sample)
t.start()
ms, _ = s.time(1000)
stop.set()
t.join()
print(f"DIAG={os.environ.get('DYNBATCH_DIAG', '0')}: {ms / 1000:.3f} ms/forward over 1000 forwards")
vals = [r.split(", ") for r in rows if r]
clk = sorted(float(v[0]) for v in vals)
pw = sorted(float(v[1]) for v in vals)
print(f"  samples {len(vals)}: sm MHz median {clk[len(clk)//2]:.0f} min {clk[0]:.0f} max {clk[-1]:.0f}; "
      f"power W median {pw[len(pw)//2]:.0f} max {pw[-1]:.0f}; reasons {sorted(set(v[2] for v in vals))}; "
      f"temp {vals[-1][3]}")
