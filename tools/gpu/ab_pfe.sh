#!/bin/bash
# A/B: L2 prefetch of SGD masters at decode in eager records (SALUS_W32_PF=1) vs none
for r in 1 2; do for lib in paper_1902_04610_b200/libsalus.so build/ab/libsalus_pfe.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 pack 1 2>&1 | tail -1
  SALUS_LIB=$lib timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c2 pack 2 2>&1 | tail -1
done; done
for lib in paper_1902_04610_b200/libsalus.so build/ab/libsalus_pfe.so; do
  SALUS_LIB=$lib timeout 300 python tools/trace_stages.py job:2048:3:128 fifo 2>&1 | grep -E "kernel|^  s [2-9]"
done
