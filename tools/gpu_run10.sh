mkdir -p gpurun_out
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,BOOTSTRAP timeout 120 python tools/probe_nccl.py > gpurun_out/nccl_a.log 2>&1; echo a=$?
grep -E "uid|created|Bootstrap|bootstrap|WARN|NCCL INFO (NET|Using)" gpurun_out/nccl_a.log | head -20
NCCL_DEBUG=INFO NCCL_DEBUG_SUBSYS=INIT,BOOTSTRAP timeout 120 python tools/probe_nccl.py dist > gpurun_out/nccl_b.log 2>&1; echo b=$?
grep -E "uid|created|Bootstrap|bootstrap|WARN" gpurun_out/nccl_b.log | head -20
