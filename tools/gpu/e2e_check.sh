#!/bin/bash
for lib in paper_1902_04610_b200/libsalus.so build/ab/libsalus_base.so paper_1902_04610_b200/libsalus.so; do
  SALUS_LIB=$lib timeout 300 python bench.py --no-side --no-c5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib', round(d['value']), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'])"
done
SALUS_TG=0 timeout 300 python bench.py --no-side --no-c5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('TG=0', round(d['value']), 'e2e', round(d['e2e']['value']))"
