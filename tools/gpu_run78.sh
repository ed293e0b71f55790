# balanced K-chunk split for the structured core products: tests, bench with CK variants
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?; tail -2 gpurun_out/pytest_gpu.log
for ck in 256 0 128 512; do
TSVD_GEMM_CK=$ck timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ck$ck.log 2>&1; echo bench=$? ck=$ck
tail -1 gpurun_out/bench_ck$ck.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
