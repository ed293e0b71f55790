# K7 with 8 lanes per pair: tests, bench A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for gl in 16; do
TSVD_K7_GL=$gl timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_gl$gl.log 2>&1; echo bench=$? gl=$gl
tail -1 gpurun_out/bench_gl$gl.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
