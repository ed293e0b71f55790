mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -x -k "cholqr or core_svd" > gpurun_out/pytest_k.log 2>&1; echo k=$?; tail -3 gpurun_out/pytest_k.log
timeout 300 python tools/micro_cholqr.py 3345 128
bash tools/gpu_run14.sh
