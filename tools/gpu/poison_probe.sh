#!/bin/bash
# configs with split-K and multi-lane/eviction schedules, meta + arena poisoned
export SALUS_POISON=1
for c in "c4 srtf" "c4 pack" "c4 fifo" "c4 fair"; do echo "== $c"; timeout 200 python tools/run_cfg.py $c 1 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_gpu_splitk.py tests/test_gpu_math.py tests/test_gpu_evict.py -x -q 2>&1 | tail -3
