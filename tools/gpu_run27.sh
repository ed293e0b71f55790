for x in 32 64 96; do
  TSVD_CORE_EXTRA=$x timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_x$x.log 2>&1
  echo extra=$x; tail -1 gpurun_out/bench_x$x.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_step'], {k: round(v['ms_per_step'],2) for k,v in d['kernels'].items()})"
done
