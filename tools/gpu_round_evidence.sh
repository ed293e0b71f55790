# Round evidence on one B200 (run with gpurun): the GPU tests, the default bench line, the
# one-update DRAM traffic of the GEMM class (bench.py's roofline.traffic), the ncu launch list of
# the default bench, and one `ncu --set full` capture of the dominant kernel's largest launches.
set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/ev_pytest.log 2>&1; echo pytest=$? >> gpurun_out/ev_pytest.log
timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/ev_traffic_c4.csv python tools/profile_one.py c4 > gpurun_out/ev_traffic.log 2>&1
python tools/ncu_traffic.py c4 gpurun_out/ev_traffic_c4.csv > gpurun_out/ev_traffic_json.log 2>&1
timeout 300 python bench.py > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/ev_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/ev_ncu_bench.log 2>&1
gzip -f gpurun_out/ev_launches.csv
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:dgemm_v2_kernel --launch-skip 20 -c 3 -o gpurun_out/ev_dgemm_full python tools/profile_one.py c4 > gpurun_out/ev_ncu_full.log 2>&1
