mkdir -p gpurun_out
NCCL_DEBUG=WARN timeout 300 python -m pytest tests/test_gpu_shard.py -x -q -k nccl > gpurun_out/pytest_nccl.log 2>&1; echo nccl=$?
grep -E "NCCL|Error|error|E_NCCL|passed|failed" gpurun_out/pytest_nccl.log | head -30
