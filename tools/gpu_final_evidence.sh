# End-of-session evidence on one B200: full-stream parity of the default config, the other
# configs' bench lines (c5 at full size).  Writes gpurun_out/fin_*.
set -x
timeout 1500 python tools/stream_parity.py --config c4 --batches 10 --oracle-batches 10 --out gpurun_out/fin_parity_c4.json > gpurun_out/fin_parity_c4.log 2>&1
for c in c1 c2 c3; do timeout 300 python bench.py --config $c > gpurun_out/fin_bench_$c.json 2> gpurun_out/fin_bench_$c.err; done
timeout 900 python bench.py --config c5 > gpurun_out/fin_bench_c5.json 2> gpurun_out/fin_bench_c5.err
