mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "chol or core_svd or jacobi or trsm" > gpurun_out/pytest_k.log 2>&1; echo k=$?
tail -15 gpurun_out/pytest_k.log
TSVD_TRACE=1 timeout 600 python tools/probe_c2.py c2 1 > gpurun_out/probe_c2.log 2>&1; echo c2=$?
grep -v "^\[jacobi\]" gpurun_out/probe_c2.log | tail -12
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
tail -c 3000 gpurun_out/bench_c2.log
