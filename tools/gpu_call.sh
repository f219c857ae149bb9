set -u
DKSS_LIB=paper_1503_04955_b200/_lib/libdkss_exp.so DKSS_HOST_TIMING=1 python tools/e2e_probe.py --bits 24 --reps 5 2>&1 | grep split | tail -6
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
