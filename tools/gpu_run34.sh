#!/bin/bash
mkdir -p gpurun_out
TSVD_DAG_CHECK=1 TSVD_DAG_TRACE=1 timeout 300 python tools/micro_chol.py 1000 4500 2>&1 | grep -v Warn | awk '!seen[$0]++' | head -60
TSVD_DAG_CHECK=1 TSVD_DAG_TRACE=1 timeout 300 python tools/probe_c2.py c2 1 2>&1 | grep -v Warn | head -40
timeout 300 python tools/micro_chol.py 1000 2500 4500 8000 2>&1 | grep -v Warn
