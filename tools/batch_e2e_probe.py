"""Where the end-to-end time of dmul_many (1024 x 2^18) goes: chunk counts of the two-lane
pipeline (dkss._pipelined_batch), operand preparation, the device call, Natural creation."""
import random, time, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1503_04955_b200.dkss as D
from paper_1503_04955_b200.words import Natural
r=random.Random(1)
pairs=[(r.getrandbits(1<<18)|1<<((1<<18)-1), r.getrandbits(1<<18)|1<<((1<<18)-1)) for _ in range(1024)]
D.dmul_many(pairs)
for chunks in (1, 2, 4, 8, 16):
    D._PIPE_CHUNKS = chunks
    D.dmul_many(pairs)
    ts=[]
    for _ in range(4):
        t=time.perf_counter(); D.dmul_many(pairs); ts.append(time.perf_counter()-t)
    print("chunks", chunks, "e2e ms", round(min(ts)*1e3,2))
# phases
vals=[(D._as_int_len(a,64), D._as_int_len(b,64)) for a,b in pairs]
t0=time.perf_counter()
vals=[(D._as_int_len(a,64), D._as_int_len(b,64)) for a,b in pairs]
da=[D._digits(a, ai) for (a,_),((ai,_),_) in zip(pairs, vals)]
db=[D._digits(b, bi) for (_,b),(_,(bi,_)) in zip(pairs, vals)]
t1=time.perf_counter()
plan=D._plan_for(1<<18, 64); dp=D.device_plan(plan); nc=dp.info["product_limbs"]
C=D._pipelined_batch(plan, da, db, da[0][3], nc)
t2=time.perf_counter()
res=[Natural._from_u32(C[i], 8192, 64) for i in range(1024)]
t3=time.perf_counter()
C2=dp.mul_batch_digits([d[1] for d in da],[d[2] for d in da],[d[1] for d in db],[d[2] for d in db], da[0][3], nc)
t4=time.perf_counter()
print("prep", round((t1-t0)*1e3,2), "pipelined call", round((t2-t1)*1e3,2), "naturals", round((t3-t2)*1e3,2), "single call", round((t4-t3)*1e3,2))
