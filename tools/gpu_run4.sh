mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "core_svd or jacobi" > gpurun_out/pytest_core.log 2>&1; echo core=$?
tail -30 gpurun_out/pytest_core.log
TSVD_TRACE=1 timeout 600 python tools/probe_c2.py c2 1 > gpurun_out/probe_c2.log 2>&1; echo c2=$?
grep -v "^\[jacobi\]" gpurun_out/probe_c2.log | tail -12
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -5 gpurun_out/pytest_gpu.log
