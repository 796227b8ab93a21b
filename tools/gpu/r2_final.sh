#!/bin/bash
# round-2 final: smoke, GPU suite, bench line, ncu launch list + C2a/C1 full captures
mkdir -p gpurun_out/final
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke $? >> gpurun_out/final/status.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/final/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/final/status.txt
timeout 1200 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo bench $? >> gpurun_out/final/status.txt
SALUS_COOP=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12 --csv \
  --log-file gpurun_out/final/launches.csv python bench.py --steps 2 --warmup 3 --no-c5 --no-cpu-baseline \
  > gpurun_out/final/ncu_launch.log 2>&1; echo launches $? >> gpurun_out/final/status.txt
SALUS_COOP=0 timeout 900 ncu --set full --import-source on --clock-control none -c 1 -o gpurun_out/final/c2a \
  python tools/run_cfg.py c2 pack 1 > gpurun_out/final/ncu_c2a.log 2>&1; echo ncu_c2a $? >> gpurun_out/final/status.txt
SALUS_COOP=0 timeout 600 ncu --set full --import-source on --clock-control none -c 1 -o gpurun_out/final/c1 \
  python tools/run_cfg.py c1 fifo 1 > gpurun_out/final/ncu_c1.log 2>&1; echo ncu_c1 $? >> gpurun_out/final/status.txt
