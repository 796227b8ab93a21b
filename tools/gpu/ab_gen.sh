#!/bin/bash
# A/B: GEN tiles stored through the 4x4 chunk transpose (default) vs 16-byte row stores (SALUS_GEN_T4=0)
timeout 600 python -m pytest tests/test_gpu_math.py -q -x -k "c1 or tiny" 2>&1 | tail -1
for r in 1 2; do for lib in build/ab/libsalus_gent0.so paper_1902_04610_b200/libsalus.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 100 python tools/run_cfg.py c1 srtf 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
done; done
SALUS_LIB=paper_1902_04610_b200/libsalus.so timeout 300 python tools/trace_stages.py c1 fifo 2>&1 | grep -E "kernel|^  s [0-9]"
