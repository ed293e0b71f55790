# programmatic dependent launch: tests, bench with / without, timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest_gpu.log
for pdl in 1 0 1; do
TSVD_PDL=$pdl timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_pdl$pdl.log 2>&1; echo bench=$? pdl=$pdl
tail -1 gpurun_out/bench_pdl$pdl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], d['e2e']['value']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
timeout 600 python tools/timeline.py c2 2 > gpurun_out/timeline.txt 2>&1; head -4 gpurun_out/timeline.txt | tail -3
