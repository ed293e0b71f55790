# Evidence run: tests, bench (N=1, default K/W), ncu launch list of the bench command, one
# ncu --set full capture each of the two dominant kernels (tile-DAG Cholesky, core GEMM).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -2 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench_default.log 2>&1; echo bench=$?
tail -1 gpurun_out/bench_default.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], json.dumps(d['roofline'])); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.log 2>&1 && \
timeout 1800 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo ncu_list=$?
python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/launches_summary.txt | head -20
timeout 300 python tools/probe_c2.py c2 1 > gpurun_out/probe_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"chol_dag|trsm_dag" -c 2 -o gpurun_out/prof_chol python tools/probe_c2.py c2 1 > gpurun_out/ncu_full_chol.log 2>&1; echo ncu_full_chol=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"dgemm_v2" -s 20 -c 2 -o gpurun_out/prof_gemm python tools/probe_c2.py c2 1 > gpurun_out/ncu_full_gemm.log 2>&1; echo ncu_full_gemm=$?
for f in prof_chol prof_gemm; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; done
python tools/ncu_traffic.py gpurun_out/traffic.json gpurun_out/prof_chol_raw.csv gpurun_out/prof_gemm_raw.csv
ls -la gpurun_out | head -30
