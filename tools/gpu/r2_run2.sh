# round-2 GPU check: full GPU suite, benchmarked-config parity, bench line
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2b_smoke.log 2>&1; echo smoke $? >> gpurun_out/r2b_status.txt
timeout 900 python -m pytest tests -m gpu -q --ignore=tests/test_gpu_configs.py > gpurun_out/r2b_gpu_tests.log 2>&1; echo tests $? >> gpurun_out/r2b_status.txt
timeout 1500 python -m pytest tests/test_gpu_configs.py -m gpu -q -s > gpurun_out/r2b_gpu_configs.log 2>&1; echo configs $? >> gpurun_out/r2b_status.txt
timeout 1500 python bench.py --steps 5 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err; echo bench $? >> gpurun_out/r2b_status.txt
