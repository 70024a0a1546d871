"""Probe: NVLS multicast support on the box (driver attribute, torch symmetric memory at world 1)."""
import os
import torch
import torch.distributed as dist

print("torch", torch.__version__, "cuda", torch.version.cuda)
try:
    from cuda.bindings import driver as drv
except Exception:
    from cuda import cuda as drv
err, = drv.cuInit(0)
err, dev = drv.cuDeviceGet(0)
for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
             "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
    a = getattr(drv.CUdevice_attribute, name, None)
    if a is not None:
        print(name, drv.cuDeviceGetAttribute(a, dev))
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda:0"))
try:
    import torch.distributed._symmetric_memory as symm_mem
    print("symm backends:", getattr(symm_mem, "get_backend", lambda *a: "?")(torch.device("cuda")))
    t = symm_mem.empty(1 << 20, dtype=torch.float32, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    print("multicast_ptr", hex(h.multicast_ptr), "buffer_ptrs", [hex(p) for p in h.buffer_ptrs])
    print("has barrier", hasattr(h, "barrier"), "signal_pad_ptrs", hasattr(h, "signal_pad_ptrs"))
except Exception as e:
    import traceback; traceback.print_exc()
dist.destroy_process_group()
