set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo smoke $? >> gpurun_out/r2_status.txt
timeout 900 python -m pytest tests -m gpu -x -q --ignore=tests/test_gpu_configs.py > gpurun_out/r2_gpu_tests.log 2>&1; echo tests $? >> gpurun_out/r2_status.txt
timeout 1200 python -m pytest tests/test_gpu_configs.py -m gpu -q -s > gpurun_out/r2_gpu_configs.log 2>&1; echo configs $? >> gpurun_out/r2_status.txt
