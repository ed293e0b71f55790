mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -k "fullsize" > gpurun_out/pytest_fullsize.log 2>&1; echo fullsize=$?
tail -15 gpurun_out/pytest_fullsize.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
tail -c 4000 gpurun_out/bench_c2.log
