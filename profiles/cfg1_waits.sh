for d in 0 39 231; do BATCH=64 BP=0.1 DYNBATCH_DIAG=$d timeout 120 python profiles/step_waits.py > gpurun_out/cfg1_waits_$d.json 2>&1; done
python - <<'P'
import sys,os
sys.path.insert(0,os.getcwd())
import paper_1707_02402_b200 as db
F=128*14*14
b=db.Batch.generate("chain", batch=64, vocab=40, width=F, length=16, branch_prob=0.1, seed=0)
s=db.IepSession(b,1234,db.MODULE_RESBLOCK)
s.time(3)
st=s.stats()
print("steps",st.steps,"groups",st.groups,"expensive",st.expensive_calls,"peak",st.peak_group_rows)
ms,kt=s.time(20,profile=True)
print("ms/fwd",ms/20,[ (db.KERNEL_CLASSES[c], kt.ms[c]/20, kt.launches[c]/20) for c in range(8) if kt.launches[c]])
P
