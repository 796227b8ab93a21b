#!/bin/bash
# Quick timing of every config through tools/run_cfg.py plus the bench side sections.
timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
timeout 200 python tools/run_cfg.py c3 fair 2 2>&1 | tail -1
timeout 200 python tools/run_cfg.py c3 pack 2 2>&1 | tail -1
timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
timeout 200 python tools/run_cfg.py c4 pack 1 2>&1 | tail -1
timeout 300 python bench.py --only c2b,c3 2>&1 | tail -1 | cut -c1-900
