"""step_waits.py for each (library build, DYNBATCH_DIAG) pair, one
subprocess each: python profiles/lib_diag_matrix.py lib1.so,lib2.so 0,43,39"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
libs = sys.argv[1].split(",")
diags = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0"]
for lib in libs:
    for d in diags:
        env = dict(os.environ, DYNBATCH_DIAG=d)
        if lib != "default":
            env["DYNBATCH_LIB"] = os.path.abspath(lib)
        r = subprocess.run([sys.executable, os.path.join(HERE, "step_waits.py")], env=env, capture_output=True,
                           text=True, timeout=600)
        try:
            w = json.loads(r.stdout)
        except json.JSONDecodeError:
            print(lib, d, "ERROR", r.stderr[-500:], flush=True)
            continue
        pk = w["per_kind"]
        print(f"{os.path.basename(lib):16s} diag={d:3s} ms={w['ms_per_forward']:.3f} mhz={w['mma_loop_mhz']:.0f} "
              f"Mcyc={w['ms_per_forward'] * w['mma_loop_mhz'] / 1e3:.2f} busy={w['mma_thread']['busy']:.3f} "
              + " ".join(f"{k[-3:]}:mma={v['mma_item_cycles_per_tile']:.0f},wgt={v['weight_wait_per_tile']:.0f},"
                         f"win={v['window_wait_per_tile']:.0f},epi={v['epilogue_cycles_per_tile']:.0f}"
                         for k, v in pk.items()), flush=True)
