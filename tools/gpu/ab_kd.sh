#!/bin/bash
# A/B: double K-chunks for dW/dX tiles (default) vs 64-row K-chunks (SALUS_KD=0)
for r in 1 2; do
for lib in build/ab/libsalus_kd0.so paper_1902_04610_b200/libsalus.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  SALUS_LIB=$lib timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 300 python bench.py --only c2b 2>&1 | tail -1 | cut -c1-200
done; done
