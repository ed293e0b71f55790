#!/bin/bash
mkdir -p gpurun_out
TSVD_DAG_TRACE=1 MICRO_CHILD=1 timeout 120 python tools/micro_chol.py 200 4500 2>&1 | grep -v Warn | awk '!seen[$0]++' | head -24
timeout 200 python tools/micro_chol.py 1000 2500 4500 8000 2>&1 | grep -v Warn
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pytest_k.log 2>&1; echo "k=$?"; tail -3 gpurun_out/pytest_k.log
TSVD_DAG_TRACE=1 timeout 300 python tools/probe_c2.py c2 1 2>&1 | grep -v Warn | head -40
