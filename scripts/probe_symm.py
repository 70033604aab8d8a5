import os, socket, torch, torch.distributed as dist
import torch.distributed._symmetric_memory as symm_mem
s=socket.socket(); s.bind(("127.0.0.1",0)); port=s.getsockname()[1]; s.close()
torch.cuda.set_device(0)
store=dist.TCPStore("127.0.0.1", port, 1, True)
dist.init_process_group("nccl", store=store, rank=0, world_size=1, device_id=torch.device("cuda",0))
from torch._C._distributed_c10d import _SymmetricMemory
print("has_multicast_support", _SymmetricMemory.has_multicast_support(torch._C._autograd.DeviceType.CUDA if hasattr(torch._C._autograd,'DeviceType') else None, 0) if False else "skip")
try:
    print("mc support:", _SymmetricMemory.has_multicast_support(symm_mem.DeviceType.CUDA, 0))
except Exception as e: print("mc err", e)
print("backend", symm_mem.get_backend(torch.device("cuda",0)) if hasattr(symm_mem,'get_backend') else None)
t = symm_mem.empty(1024, dtype=torch.float32, device="cuda")
h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
print("rank", h.rank, "world", h.world_size)
for a in ("multicast_ptr","buffer_ptrs","signal_pad_ptrs","buffer_size","signal_pad_size","buffer_ptrs_dev"):
    try: print(a, getattr(h,a))
    except Exception as e: print(a, "ERR", e)
print("t ptr", t.data_ptr())
print(torch.cuda.get_device_properties(0))
import subprocess; print(subprocess.run(["nvidia-smi","-q","-d","FABRIC"],capture_output=True,text=True).stdout[-1500:])
dist.destroy_process_group()
