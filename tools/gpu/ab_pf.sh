#!/bin/bash
# A/B: L2 prefetch of SGD tiles' fp32 master pages at decode (SALUS_W32_PF=1) vs none
for r in 1 2; do
for lib in build/ab/libsalus_pf.so paper_1902_04610_b200/libsalus.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  SALUS_LIB=$lib timeout 300 python bench.py --only c2b 2>&1 | tail -1 | cut -c1-200
done; done
