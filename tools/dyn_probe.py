import os, random, sys, time
sys.path.insert(0, "/root/repo")
from paper_1503_04955_b200 import dmul
r = random.Random(1)
for e in [int(x) for x in sys.argv[1:]]:
    N = 1 << e
    a, b = r.getrandbits(N), r.getrandbits(N)
    t = time.time()
    ok = dmul(a, b).to_int() == a * b
    print(e, "mul", ok, round(time.time() - t, 3), flush=True)
    t = time.time()
    ok = dmul(a, a).to_int() == a * a
    print(e, "sqr", ok, round(time.time() - t, 3), flush=True)
