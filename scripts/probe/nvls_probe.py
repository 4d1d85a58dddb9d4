"""Probe: does this box support NVLink SHARP (multicast objects, multimem.*) for one GPU?"""
import ctypes as C
import json
import os
import socket

import torch

out = {}
cu = C.CDLL("libcuda.so.1")
cu.cuInit(0)
dev = C.c_int()
cu.cuDeviceGet(C.byref(dev), 0)
for name, attr in (("multicast", 132), ("fabric_handle", 128), ("posix_fd", 103), ("vmm", 102)):
    v = C.c_int(-1)
    r = cu.cuDeviceGetAttribute(C.byref(v), attr, dev)
    out[name] = (r, v.value)
out["device_count"] = torch.cuda.device_count()
try:
    import torch.distributed as dist
    import torch.distributed._symmetric_memory as symm_mem
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    t = symm_mem.empty(1 << 20, dtype=torch.bfloat16, device="cuda")
    h = symm_mem.rendezvous(t, dist.group.WORLD.group_name)
    out["symm_backend"] = str(symm_mem.get_backend(torch.device("cuda")))
    out["multicast_ptr"] = int(h.multicast_ptr)
    out["buffer_ptrs"] = [int(p) for p in h.buffer_ptrs]
    out["world"] = h.world_size
    dist.destroy_process_group()
except Exception as exc:  # noqa: BLE001
    out["symm_error"] = repr(exc)[:500]
print(json.dumps(out))
