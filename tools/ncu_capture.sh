#!/bin/bash
# ncu evidence for the default bench workload (run under gpurun, 1 GPU):
#   1. launch list with per-launch device time (cold-cache, serialised)
#   2. one `--set full` capture of the pass kernels of one multiply
# each ncu run is preceded by the same command without ncu (must exit 0)
set -u
mkdir -p gpurun_out
CMD="python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 3 ${BENCH_ARGS:-}"
TAG=${TAG:-r01}
$CMD > gpurun_out/plain1.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv $CMD \
  > gpurun_out/ncu_launches.log 2>&1
echo "launch list rc=$?"
$CMD > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-k_fwd_pass|k_bottom|k_inv_pass|k_tc_twiddle}" -c ${KCOUNT:-9} \
  -o gpurun_out/full_$TAG $CMD > gpurun_out/ncu_full.log 2>&1
echo "full rc=$?"
