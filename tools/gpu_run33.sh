#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/micro_chol.py 2>&1 | grep -v Warn
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pytest_k.log 2>&1; echo "k=$?"; tail -1 gpurun_out/pytest_k.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "all=$?"; tail -1 gpurun_out/pytest_gpu.log
timeout 600 python tools/timeline.py c2 2 > gpurun_out/timeline.txt 2>&1; rm -f gpurun_out/timeline_trace.json; head -4 gpurun_out/timeline.txt; sed -n '/kernel totals/,/host runtime/p' gpurun_out/timeline.txt | head -12
