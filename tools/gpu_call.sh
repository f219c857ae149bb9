set -u
mkdir -p gpurun_out
tools/microbench_tc_i8 > gpurun_out/tc_i8_peak.json 2>&1; cat gpurun_out/tc_i8_peak.json
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tensor_core or dmul_2_24 or 2_26 or stages or two_level or kernel_shape" > gpurun_out/tc_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/tc_tests.log
for c in mul2^24 batch1024x2^18 mul2^26; do
python bench.py --config $c --steps 10 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/b_$c.json 2>gpurun_out/b_$c.err; echo "$c rc=$?"
python - $c <<'PY'
import json,sys
c=sys.argv[1]
d=json.loads(open(f'gpurun_out/b_{c}.json').read().strip().splitlines()[-1])
print(c, d['ms_per_step'], d['value'], {k:(v['ms_per_step'],v['launches_per_step']) for k,v in d['kernels'].items()})
PY
done
