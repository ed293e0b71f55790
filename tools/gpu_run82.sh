# software-pipelined strips: tests, bench A/B, chol trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for pp in 1; do
TSVD_DAG_PIPE=$pp timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pipe$pp.log 2>&1; echo bench=$? pipe=$pp
tail -1 gpurun_out/bench_pipe$pp.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
TSVD_DAG_TRACE=1 timeout 300 python tools/probe_c2.py c2 1 2>&1 | grep -A9 "dag chol\] nt" | head -10
