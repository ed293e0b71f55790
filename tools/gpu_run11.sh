mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo all=$?
tail -4 gpurun_out/pytest_gpu.log
timeout 300 python tools/probe_c2.py c2 1 > gpurun_out/probe_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"jacobi_cta|dgemm_kernel|chol_panel_factor" -s 20 -c 6 -o gpurun_out/prof_k7 python tools/probe_c2.py c2 1 > gpurun_out/ncu_full.log 2>&1; echo ncu=$?
tail -3 gpurun_out/ncu_full.log
