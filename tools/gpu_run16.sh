mkdir -p gpurun_out
timeout 300 python tools/probe_c2.py c2 1 > gpurun_out/probe_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"chol_inv_small" -s 2 -c 1 -o gpurun_out/prof_ci python tools/probe_c2.py c2 1 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
