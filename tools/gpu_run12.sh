mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q --timeout 300 > gpurun_out/pytest_k.log 2>&1; echo k=$?
tail -15 gpurun_out/pytest_k.log
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_c2.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']); print(json.dumps(d['kernels'], indent=0))"
