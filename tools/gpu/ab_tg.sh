#!/bin/bash
# A/B: loss targets generated in the GEN stage (default) vs hashed in F_L's epilogue (SALUS_TG=0)
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_math.py tests/test_gpu_configs.py -q -x 2>&1 | tail -2
for r in 1 2; do for v in 0 1; do
  echo "== SALUS_TG=$v round $r"
  SALUS_TG=$v timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
  SALUS_TG=$v timeout 100 python tools/run_cfg.py c1 srtf 3 2>&1 | tail -1
  SALUS_TG=$v timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
done; done
