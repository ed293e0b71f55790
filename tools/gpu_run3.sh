mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "variants" > gpurun_out/pytest_variants.log 2>&1; echo variants=$?
tail -40 gpurun_out/pytest_variants.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -5 gpurun_out/pytest_gpu.log
