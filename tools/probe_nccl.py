"""Probe: NCCL-mode context creation in one process (1-rank communicator)."""
import os, sys, socket
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2401_09703_b200 as P
with socket.socket() as s:
    s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]
use_dist = len(sys.argv) > 1 and sys.argv[1] == "dist"
if use_dist:
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1)
torch.cuda.set_device(0)
uid = P.nccl_unique_id()
print("uid", uid[:24].hex(), flush=True)
t = P.TSVD(4, 10, 10, shard=dict(world=1, rank=0, nccl_id=uid))
print("created", flush=True)
