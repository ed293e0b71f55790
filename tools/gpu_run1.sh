mkdir -p gpurun_out
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python tools/probe_fp64.py > gpurun_out/probe.log 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
tail -3 gpurun_out/pytest_gpu.log; tail -c 3000 gpurun_out/bench_c2.log
