#!/bin/bash
# time every experiment library in _lib/ on the standard shapes (run under gpurun)
for lib in paper_1503_04955_b200/_lib/libdkss*.so; do
  for cfg in "--bits 20" "--bits 18 --batch 256" "--bits 24"; do
    DKSS_LIB=$lib python tools/exp_time.py $cfg 2>&1 | tail -1
  done
done
