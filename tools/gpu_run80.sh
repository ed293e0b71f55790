# sparse Gram: shared vs global accumulator A/B
for gs in 0; do
TSVD_GRAM_SMEM=$gs timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_gs$gs.log 2>&1; echo bench=$? gram_smem=$gs
tail -1 gpurun_out/bench_gs$gs.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
