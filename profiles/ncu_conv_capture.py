"""One cfg3 forward (bench.py's workload, same seeds) for an ncu capture of
the conv kernels:

  ncu --set full --clock-control none --import-source on -k regex:k_rb_step \
      -c 16 -o gpurun_out/conv python profiles/ncu_conv_capture.py
  python profiles/summarize_ncu.py gpurun_out/conv.ncu-rep --traffic profiles/ncu_traffic.json

Also prints the algorithmic work of the captured forward, per conv kind."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1707_02402_b200 as db  # noqa: E402

cfg = bench.CFG["cfg3"]
per = cfg["batch"]
batch = db.Batch.generate_range(0, per, cfg["kind"], batch=per, vocab=cfg["vocab"], width=bench.F,
                                depth=cfg["depth"], length=cfg["length"], branch_prob=cfg["branch_prob"],
                                seed=0)
seed = int.from_bytes(bench._mix_seed(0, 0xd00d).to_bytes(8, "little"), "little")
sess = db.IepSession(batch, seed, db.MODULE_RESBLOCK)
sess.forward()
sess.synchronize()
st = sess.stats()
print(f"steps={st.steps} expensive={st.expensive_calls} flops={st.algorithmic_flops:.4e} "
      f"bytes={st.algorithmic_bytes:.4e}")
