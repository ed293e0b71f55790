#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pytest_k.log 2>&1; echo "k=$?"; tail -1 gpurun_out/pytest_k.log
for L in 8 12 16 1000; do
  echo "LOOK=$L"
  TSVD_DAG_LOOK=$L TSVD_DAG_TRACE=1 MICRO_CHILD=1 timeout 120 python tools/micro_chol.py 4500 2>&1 | grep -v Warn | tail -7 | grep -E "chain|span"
  TSVD_DAG_LOOK=$L MICRO_CHILD=1 timeout 120 python tools/micro_chol.py 4500 8000 2>&1 | grep -v Warn
  TSVD_DAG_LOOK=$L timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_L$L.log 2>&1
  python - $L <<'PY'
import json, sys
l=[x for x in open(f'gpurun_out/bench_L{sys.argv[1]}.log') if x.startswith('{')]
d=json.loads(l[-1]); print("bench LOOK", sys.argv[1], round(d['value']), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d.get('kernels',{}).items()})
PY
done
