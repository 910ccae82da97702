"""torch symmetric memory on one GPU: does rendezvous give a multicast (NVLS) pointer?"""
import os
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm
try:
    print("has_multicast_support", symm.has_multicast_support if hasattr(symm, "has_multicast_support") else "n/a")
except Exception as e:
    print("hms err", e)
t = symm.empty(1 << 20, dtype=torch.uint8, device="cuda")
h = symm.rendezvous(t, dist.group.WORLD.group_name)
print("buffer_ptrs", [hex(p) for p in h.buffer_ptrs])
print("multicast_ptr", hex(h.multicast_ptr) if getattr(h, "multicast_ptr", 0) else h.multicast_ptr)
print([a for a in dir(h) if not a.startswith("_")])
dist.destroy_process_group()
