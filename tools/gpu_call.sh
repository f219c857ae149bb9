set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t.log
for gw in "24 2" "24 8" "26 8" "20 4"; do set -- $gw; python tools/fourstep_phases.py --bits $1 --world $2 2>&1 | tail -1; done
python bench.py --steps 10 --warmup 3 --no-cpu --e2e-steps 5 > gpurun_out/b24.json 2>gpurun_out/b24.err; echo "bench rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/b24.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['value'], d['e2e'], d['roofline']['kernel'], d['roofline']['frac'])"
