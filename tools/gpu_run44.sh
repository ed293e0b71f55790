#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pytest_k.log 2>&1; echo "k=$?"; tail -1 gpurun_out/pytest_k.log
for ex in 0 32 48 96; do
  TSVD_CORE_EXTRA=$ex timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ex$ex.log 2>&1
  python - $ex <<'PY'
import json, sys
l=[x for x in open(f'gpurun_out/bench_ex{sys.argv[1]}.log') if x.startswith('{')]
d=json.loads(l[-1]); print("extra", sys.argv[1], round(d['value']), round(d['ms_per_step'],2), {k: round(v['ms_per_step'],2) for k,v in d.get('kernels',{}).items()})
PY
done
