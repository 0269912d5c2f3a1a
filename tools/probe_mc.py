"""Probe the box for the fused wgrad + all-reduce prerequisites: multicast
(NVLS) support, P2P, torch symmetric memory with a 1-rank group."""
import json
import os
import socket

import torch
import torch.distributed as dist

out = {}
try:
    from cuda.bindings import driver as cu
    cu.cuInit(0)
    for name in ("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED", "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_FABRIC_SUPPORTED",
                 "CU_DEVICE_ATTRIBUTE_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR_SUPPORTED"):
        try:
            err, v = cu.cuDeviceGetAttribute(getattr(cu.CUdevice_attribute, name), 0)
            out[name] = [str(err), v]
        except Exception as e:
            out[name] = repr(e)
except Exception as e:
    out["cuda_bindings"] = repr(e)
out["device_count"] = torch.cuda.device_count()
s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0, world_size=1,
                        device_id=torch.device("cuda", 0))
try:
    import torch.distributed._symmetric_memory as symm
    t = symm.empty(1024, dtype=torch.float32, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD)
    out["symm_mem"] = {"mc_ptr": int(getattr(h, "multicast_ptr", 0) or 0), "world": h.world_size,
                       "buffer_ptrs": [int(p) for p in h.buffer_ptrs], "signal_pad_ptrs": [int(p) for p in h.signal_pad_ptrs]}
except Exception as e:
    out["symm_mem"] = repr(e)[:400]
dist.destroy_process_group()
print(json.dumps(out, indent=1))
