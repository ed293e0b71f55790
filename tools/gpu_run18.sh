mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -k "cholqr or chol_deflate or core_svd" > gpurun_out/pytest_k.log 2>&1; echo k=$?; tail -3 gpurun_out/pytest_k.log
timeout 300 python tools/micro_cholqr.py 3345 128; timeout 300 python tools/micro_cholqr.py 3345 96; timeout 300 python tools/micro_cholqr.py 3345 200
timeout 300 python tools/micro_cholqr.py 3345 128 > gpurun_out/micro.log 2>&1 && timeout 300 ncu --set full --import-source on --clock-control none -k regex:chol_inv_small -s 5 -c 1 -o gpurun_out/prof_ci2 python tools/micro_cholqr.py 3345 128 > /dev/null 2>&1; echo ncu=$?
