# strip width A/B (prebuilt libraries)
cp paper_2401_09703_b200/libtsvd.so /tmp/lib4.so
for v in 3 6 4; do
  if [ $v = 4 ]; then cp /tmp/lib4.so paper_2401_09703_b200/libtsvd.so; else cp tools/scratch/libs/libtsvd_strip$v.so paper_2401_09703_b200/libtsvd.so; fi
  timeout 600 python bench.py --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('strip=$v', round(d['value']), round(d['kernels']['chol_panel']['ms_per_step'],3))"
done
