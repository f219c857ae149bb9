import random, time, os, sys
sys.path.insert(0, os.getcwd())
import paper_1503_04955_b200.dkss as D
r=random.Random(1)
pairs=[(r.getrandbits(1<<18)|1<<((1<<18)-1), r.getrandbits(1<<18)|1<<((1<<18)-1)) for _ in range(1024)]
D.dmul_many(pairs)
for lanes, chunks in ((2,2),(4,8)):
    D._PIPE_LANES=lanes; D._PIPE_CHUNKS=chunks
    res=D.dmul_many(pairs)
    assert res[5].to_int()==pairs[5][0]*pairs[5][1] and res[1023].to_int()==pairs[1023][0]*pairs[1023][1]
    ts=[]
    for _ in range(5):
        t=time.perf_counter(); D.dmul_many(pairs); ts.append(time.perf_counter()-t)
    print("lanes", lanes, "chunks", chunks, "e2e ms min", round(min(ts)*1e3,2), "median", round(sorted(ts)[2]*1e3,2))
