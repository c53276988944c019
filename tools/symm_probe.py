"""Probe: DistComm.alloc / peer_ptrs (CUDA symmetric memory) in a 1-rank NCCL group."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
from paper_1901_05423_b200.sharded import DistComm
c = DistComm()
buf = c.alloc(1 << 20, torch.device("cuda", 0))
ptrs = c.peer_ptrs(buf)
print("symmetric memory ok:", len(ptrs), hex(ptrs[0]), hex(buf.data_ptr()), ptrs[0] == buf.data_ptr())
dist.destroy_process_group()
