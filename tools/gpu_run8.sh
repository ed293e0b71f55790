mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -25 gpurun_out/pytest_gpu.log
TSVD_TRACE=1 timeout 600 python tools/probe_c2.py c2 1 > gpurun_out/probe_c2.log 2>&1; echo c2=$?
grep -v "^\[jacobi\]" gpurun_out/probe_c2.log | tail -6
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
tail -c 2500 gpurun_out/bench_c2.log
