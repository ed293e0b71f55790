set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s16_pytest.log 2>&1; echo pytest=$? >> gpurun_out/s16_pytest.log
timeout 300 python bench.py > gpurun_out/s16_bench.json 2> gpurun_out/s16_bench.err
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s16_traffic_c4.csv python tools/profile_one.py c4 > gpurun_out/s16_traffic.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/s16_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/s16_ncu_bench.log 2>&1
gzip -f gpurun_out/s16_launches.csv
