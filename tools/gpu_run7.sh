mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -5 gpurun_out/pytest_gpu.log
TSVD_TRACE=1 timeout 600 python tools/probe_c2.py c2 1 > gpurun_out/probe_c2.log 2>&1; echo c2=$?
grep -v "^\[jacobi\]" gpurun_out/probe_c2.log | tail -6
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
tail -c 3000 gpurun_out/bench_c2.log
timeout 900 python bench.py --steps 2 --warmup 3 > gpurun_out/bench_small.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ncu_launch.log 2>&1; echo ncu=$?
ls -la gpurun_out/
