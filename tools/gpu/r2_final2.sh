#!/bin/bash
mkdir -p gpurun_out/final2
for r in 1 2; do for lib in build/ab/libsalus_base.so paper_1902_04610_b200/libsalus.so; do
  echo "== $lib round $r"; SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
done; done > gpurun_out/final2/ab.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_splitk.py -q -s > gpurun_out/final2/splitk.log 2>&1; echo splitk $? >> gpurun_out/final2/status.txt
timeout 1200 python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err; echo bench $? >> gpurun_out/final2/status.txt
