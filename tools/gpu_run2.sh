mkdir -p gpurun_out
TSVD_TRACE=1 timeout 600 python tools/probe_c2.py c2 1 > gpurun_out/probe_c2.log 2>&1; echo c2=$?
TSVD_TRACE=1 timeout 600 python tools/probe_c2.py c3 1 > gpurun_out/probe_c3.log 2>&1; echo c3=$?
grep -v "^\[jacobi\]" gpurun_out/probe_c2.log gpurun_out/probe_c3.log | tail -8
