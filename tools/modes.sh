#!/bin/bash
# compare pass implementations (DKSS_PASS_MODE: 1 CTA-fused, 2 warp-fused, 3 split, unset auto)
for mode in ${MODES:-1 2 3}; do
  for c in ${CONFIGS:-mul2^20 batch1024x2^18}; do
    DKSS_PASS_MODE=$mode python bench.py --config $c --steps ${STEPS:-10} --warmup 3 --no-cpu --e2e-steps 2 > gpurun_out/m_${mode}_$c.json 2> gpurun_out/m_${mode}_$c.err || tail -3 gpurun_out/m_${mode}_$c.err
    python - "$mode" "$c" <<'PY'
import json,sys
mode,c=sys.argv[1],sys.argv[2]
try: d=json.loads(open(f'gpurun_out/m_{mode}_{c}.json').read().strip().splitlines()[-1])
except Exception as e: print(mode,c,'no result',e); sys.exit()
k=d['kernels']
print(f"mode {mode} {c:16s} ms/step {d['ms_per_step']:.4f} whole_frac {d['roofline']['whole_multiply_frac']:.3f} ", ' '.join(f"{n}:{v['ms_per_mul']*1e3:.1f}us" for n,v in k.items()))
PY
  done
done
