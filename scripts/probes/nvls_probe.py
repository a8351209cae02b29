"""Does this box expose NVLS multicast to one process?  torch SymmetricMemory
rendezvous on a 1-rank NCCL group, then the multicast pointer; and the CUDA
driver's multicast support attribute."""
import os
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
try:
    from cuda.bindings import driver as cu
except ImportError:
    from cuda import cuda as cu
err, dev = cu.cuDeviceGet(0)
err, mc = cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev)
print("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED:", mc, err)
try:
    import torch.distributed._symmetric_memory as symm_mem
    t = symm_mem.empty(4096, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("symmetric memory ok; world", h.world_size, "multicast_ptr", hex(h.multicast_ptr), "buffer_ptrs", [hex(p) for p in h.buffer_ptrs])
except Exception as e:  # noqa
    print("symmetric memory failed:", type(e).__name__, e)
dist.destroy_process_group()
