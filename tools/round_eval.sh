#!/bin/bash
# Round evaluation on the GPU box (1 GPU): GPU test suite, smoke, the default bench line and
# the reference arm, short benches of the other configs, then the ncu launch list and one
# full capture of the default workload.  Everything lands in gpurun_out/.
set -u
mkdir -p gpurun_out
TAG=${TAG:-r02}
if [ -z "${SKIP_TESTS:-}" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$TAG.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_$TAG.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
fi
timeout 900 python bench.py > gpurun_out/bench_default_$TAG.json 2> gpurun_out/bench_default_$TAG.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_default_$TAG.json
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
bash tools/quick.sh
if [ -z "${SKIP_NCU:-}" ]; then TAG=$TAG bash tools/ncu_capture.sh; fi
python tools/e2e_probe.py --bits 24 --reps 10 > gpurun_out/e2e_probe24_$TAG.log 2>&1; tail -1 gpurun_out/e2e_probe24_$TAG.log
python tools/h2d_probe.py > gpurun_out/h2d_probe_$TAG.log 2>&1; tail -1 gpurun_out/h2d_probe_$TAG.log
for gw in "24 2" "24 8" "26 8" "20 4"; do set -- $gw; python tools/fourstep_phases.py --bits $1 --world $2 2>&1 | tail -1; done > gpurun_out/fourstep_phases_$TAG.jsonl
DKSS_BENCH_GLOO=1 timeout 600 python bench.py --gpus 2 --config mul2^24 --steps 5 --warmup 3 --no-cpu --e2e-steps 3 > gpurun_out/gloo2_$TAG.json 2> gpurun_out/gloo2_$TAG.err; echo "gloo2 rc=$?"
