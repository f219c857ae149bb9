set -u
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/t.log
STEPS=10 bash tools/quick.sh 2>&1 | grep -v "^ALL\|gpu_check" 
