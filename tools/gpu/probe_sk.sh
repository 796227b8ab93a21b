#!/bin/bash
for cfg in job:4096:4:64 job:4096:3:512; do
  echo "=== $cfg split"; timeout 300 python tools/trace_stages.py $cfg fifo 2>&1 | grep -E "kernel|^  s [2-9]"
done > gpurun_out/probe_sk.txt 2>&1
for r in 1 2; do for v in 1 0; do echo "== SALUS_SPLITK=$v"; SALUS_SPLITK=$v timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1; done; done >> gpurun_out/probe_sk.txt 2>&1
