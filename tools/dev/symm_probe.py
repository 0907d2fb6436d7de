"""Probe: CUDA symmetric memory at world size 1 (rendezvous, get_buffer, barrier)."""
import os, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
t = symm.empty((16, 2), dtype=torch.int32, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD)
v = h.get_buffer(0, (16, 2), torch.int32)
v[3:5] = 7
h.barrier()
torch.cuda.synchronize()
print("ok", t[3].tolist(), h.world_size, h.rank, v.data_ptr() == t.data_ptr())
dist.destroy_process_group()
