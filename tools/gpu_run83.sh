# balanced split chunk length sweep
for ck in 160 192 224 256 320; do
TSVD_GEMM_CK=$ck timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_ck$ck.log 2>&1
tail -1 gpurun_out/bench_ck$ck.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ck=$ck', round(d['value']), round(d['ms_per_step'],3), round(d['kernels']['dgemm_dmma']['ms_per_step'],3))"
done
