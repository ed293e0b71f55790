#!/bin/bash
for cs in 0 1; do
  echo "CSTAGE=$cs"
  TSVD_DAG_CSTAGE=$cs TSVD_DAG_TRACE=1 MICRO_CHILD=1 timeout 120 python tools/micro_chol.py 4500 2>&1 | grep -v Warn | tail -9 | grep -E "chain|span|Wstrip|U x"
  TSVD_DAG_CSTAGE=$cs MICRO_CHILD=1 timeout 120 python tools/micro_chol.py 1000 4500 8000 2>&1 | grep -v Warn
done
TSVD_DAG_CSTAGE=1 timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "chol" 2>&1 | tail -1
