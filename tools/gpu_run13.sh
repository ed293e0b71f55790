mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_c2.log 2>&1; echo bench=$?
python -c "
import json; d=json.loads(open('gpurun_out/bench_c2.log').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['kernel'], d['roofline']['frac']); print({k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()}, {k: v['launches_per_step'] for k,v in d['kernels'].items()})"
timeout 300 python tools/probe_c2.py c2 1 > gpurun_out/probe_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"jacobi_cta" -c 1 -o gpurun_out/prof_k7b python tools/probe_c2.py c2 1 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
