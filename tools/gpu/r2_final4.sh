#!/bin/bash
mkdir -p gpurun_out/final4
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/final4/smoke.log 2>&1; echo smoke $? >> gpurun_out/final4/status.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final4/gpu_tests.log 2>&1; echo tests $? >> gpurun_out/final4/status.txt
timeout 1200 python bench.py > gpurun_out/final4/bench.json 2> gpurun_out/final4/bench.err; echo bench $? >> gpurun_out/final4/status.txt
