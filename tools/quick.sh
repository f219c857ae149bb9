#!/bin/bash
# parity report + short benches of the main configs (used for iteration on the GPU box)
python tools/gpu_check.py > gpurun_out/gpu_check.log 2>&1; tail -1 gpurun_out/gpu_check.log
for c in mul2^20 batch1024x2^18 mul2^24 mul2^26 mul2^16 ones2^20 ${EXTRA_CONFIGS:-}; do
  python bench.py --config $c --steps ${STEPS:-20} --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err || tail -5 gpurun_out/bench_$c.err
  python - "$c" <<'PY'
import json,sys
c=sys.argv[1]
try:
    d=json.loads(open(f'gpurun_out/bench_{c}.json').read().strip().splitlines()[-1])
except Exception as e:
    print(c,'no result',e); sys.exit()
k=d['kernels']
r=d['roofline']
print(f"{c:16s} ms/step {d['ms_per_step']:.4f} value {d['value']:.2f} Gbit/s  dominant {r['kernel']} ({r['bound']}) frac {r['frac']:.3f} step_frac {r['step_frac']} e2e {d['e2e']['ms']} ms clocks {d['clocks']['sm_mhz']}")
print('   ', ' '.join(f"{n}:{v['ms_per_step']*1e3:.1f}us/{v['bound']}:{v['frac']}" for n,v in k.items()))
PY
done
