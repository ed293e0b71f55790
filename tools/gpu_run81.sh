# prescaled back substitution: tests, bench A/B, trsm trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for pre in 1 0; do
TSVD_TRSM_PRE=$pre timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pre$pre.log 2>&1; echo bench=$? pre=$pre
tail -1 gpurun_out/bench_pre$pre.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
TSVD_DAG_TRACE=1 timeout 300 python tools/probe_c2.py c2 1 2>&1 | grep -A4 "dag trsm" | head -5
