#!/bin/bash
# C3 FAIR/8 switch-gap tail, interleaved builds on one box
for r in 1 2 3; do
for lib in build/ab/libsalus_prev.so paper_1902_04610_b200/libsalus.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 200 python bench.py --only c3 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read())['c3']; print(d['requests_per_s'], d['switch_us'], d['same_job_gap_us'])"
done; done
