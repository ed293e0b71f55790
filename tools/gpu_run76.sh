# GEMM tile-size knob A/B
for b in -1 1; do
TSVD_GEMM_BIG=$b timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_big$b.log 2>&1; echo bench=$? big=$b
tail -1 gpurun_out/bench_big$b.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
