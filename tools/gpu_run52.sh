#!/bin/bash
mkdir -p gpurun_out
TSVD_DAG_TRACE=1 MICRO_CHILD=1 timeout 120 python tools/micro_chol.py 4500 2>&1 | grep -v Warn | tail -7
MICRO_CHILD=1 timeout 120 python tools/micro_chol.py 1000 4500 8000 2>&1 | grep -v Warn
bash tools/gpu_run32.sh
