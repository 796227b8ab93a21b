#!/bin/bash
# A/B on C2a (3 reps each, two interleaved rounds): session-start build, head, head KD=0, head W32 L2 prefetch;
# then the headline's ncu launch list
for r in 1 2; do
for lib in build/ab/libsalus_base.so paper_1902_04610_b200/libsalus.so build/ab/libsalus_kd0.so build/ab/libsalus_pf.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
done; done
mkdir -p gpurun_out/final
SALUS_COOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv \
  --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline --no-side \
  > gpurun_out/final/ncu_launch.log 2>&1; echo launches $?
