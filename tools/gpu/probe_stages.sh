#!/bin/bash
for cfg in c1 job:4096:4:64 job:4096:2:256 job:2048:3:128 job:1024:3:256 job:512:2:128; do
  echo "=== $cfg"; timeout 300 python tools/trace_stages.py $cfg fifo 2>&1 | grep -v "^  s.* t " | tail -30
done > gpurun_out/stages.txt 2>&1
