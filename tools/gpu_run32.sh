#!/bin/bash
# tile-DAG Cholesky / TRSM: kernel tests first (short timeout), then full GPU suite, bench, timeline
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu > gpurun_out/pytest_k.log 2>&1; echo "k=$?"; tail -3 gpurun_out/pytest_k.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "all=$?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c2.log 2>&1; echo "bench=$?"
python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_c2.log') if x.startswith('{')]
if l:
    d=json.loads(l[-1]); print(d['value'], d['ms_per_step'], d['e2e']['value'], d['roofline']['kernel'], d['roofline']['frac'])
    print({k: round(v['ms_per_step'],2) for k,v in d.get('kernels',{}).items()})
PY
timeout 600 python tools/timeline.py c2 2 > gpurun_out/timeline.txt 2>&1; rm -f gpurun_out/timeline_trace.json; head -4 gpurun_out/timeline.txt; sed -n '/kernel totals/,/host runtime/p' gpurun_out/timeline.txt | head -22
