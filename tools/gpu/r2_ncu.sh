#!/bin/bash
# final-build ncu evidence: bench launch list (headline only), C2a and C1 full captures
mkdir -p gpurun_out/ncu2
SALUS_COOP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv \
  --log-file gpurun_out/ncu2/launches.csv python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline --no-side \
  > gpurun_out/ncu2/ncu_launch.log 2>&1; echo launches $?
SALUS_COOP=0 timeout 900 ncu --set full --import-source on --clock-control none -c 1 -o gpurun_out/ncu2/c2a \
  python tools/run_cfg.py c2 pack 1 > gpurun_out/ncu2/ncu_c2a.log 2>&1; echo ncu_c2a $?
SALUS_COOP=0 timeout 600 ncu --set full --import-source on --clock-control none -c 1 -o gpurun_out/ncu2/c1 \
  python tools/run_cfg.py c1 fifo 1 > gpurun_out/ncu2/ncu_c1.log 2>&1; echo ncu_c1 $?
