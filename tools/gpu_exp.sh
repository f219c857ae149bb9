# scratch driver for one gpurun call (edited per experiment)
set -u
mkdir -p gpurun_out
python tools/gpu_check.py > gpurun_out/gpu_check_x2.log 2>&1; tail -3 gpurun_out/gpu_check_x2.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_x2.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/gputest_x2.log
for b in 24 26 20 22; do timeout 300 python tools/variant_time.py --bits $b --twiddle auto,tensor; done 2>&1 | tee gpurun_out/variant_x2.jsonl
timeout 600 python tools/variant_time.py --bits 18 --batch 1024 --reps 8 --twiddle auto 2>&1 | tee -a gpurun_out/variant_x2.jsonl
