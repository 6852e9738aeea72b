"""Does this box expose NVLS multicast to torch symmetric memory?  (One rank:
prints buffer_ptrs and multicast_ptr; 0 = no multicast object could be
created.)  Round-2 result on the one-GPU gpurun boxes: "fail to export
multicast handle ... invalid argument", multicast_ptr 0."""
import os, torch, torch.distributed as dist
os.environ.setdefault("MASTER_ADDR","127.0.0.1"); os.environ.setdefault("MASTER_PORT","29512")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda",0))
import torch.distributed._symmetric_memory as symm_mem
t = symm_mem.empty(1<<20, dtype=torch.uint8, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print("buffer_ptrs", h.buffer_ptrs)
for a in ("multicast_ptr","has_multicast_support"):
    try:
        v = getattr(h, a); print(a, v() if callable(v) else v)
    except Exception as e: print(a, "ERR", e)
try:
    print("has_multicast_support", symm_mem.has_multicast_support(torch.device("cuda",0).type, 0) if hasattr(symm_mem,'has_multicast_support') else 'n/a')
except Exception as e: print('hms', e)
dist.destroy_process_group()
