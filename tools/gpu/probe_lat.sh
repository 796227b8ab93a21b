#!/bin/bash
# Where the latency-bound configs spend their time (current build)
timeout 300 python tools/trace_stages.py c1 fifo 2>&1 | tail -40
timeout 300 python tools/c4_breakdown.py c4 srtf > gpurun_out/c4_breakdown.json 2>&1
timeout 600 python tools/c4_breakdown.py c5 pack > gpurun_out/c5_breakdown.json 2>&1
