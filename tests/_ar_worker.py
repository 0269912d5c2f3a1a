"""Worker of tests/test_gpu_allreduce.py::test_fused_wgrad_allreduce_two_processes_ipc:
one rank of a 2-process group on cuda:0 (gloo for the CUDA IPC handle
exchange), running cks_dilated_wgrad_allreduce on its batch shard of each
layer; saves its dW to $AR_OUT."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from cks_synth import make_layer_inputs  # noqa: E402
from paper_2306_15951_b200 import _lib as L  # noqa: E402
from paper_2306_15951_b200.dist import FusedWgradAllReduce, shard_range  # noqa: E402
from test_gpu_allreduce import LAYERS  # noqa: E402
from test_gpu_parity import dev  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    d = torch.device("cuda", 0)
    torch.cuda.set_device(d)
    dt = L.CKS_BF16
    geoms, xs, dws, wss = [], [], [], []
    for i, l in enumerate(LAYERS):
        a = make_layer_inputs(l, 31, i, "bf16")
        lo, hi = shard_range(l.N, world, rank)
        X, G = dev(torch, a["X"][lo:hi], "bf16"), dev(torch, a["dY"][lo:hi], "bf16")
        g = L.make_geom(hi - lo, l.C, l.H, l.W, l.OC, l.FH, l.FW, l.sh, l.sw, l.ph, l.pw)
        geoms.append(g)
        xs.append((X, G))
        dws.append(torch.full((l.OC, l.FH, l.FW, l.C), float("nan"), device=d))
        wss.append(torch.empty(max(L.cks_workspace_size(g, dt, L.CKS_OP_WGRAD_AR), 256), dtype=torch.uint8,
                               device=d))
    fused = FusedWgradAllReduce(geoms, dws, d)
    torch.cuda.synchronize()
    dist.barrier()
    st = torch.cuda.Stream()
    for i in range(len(LAYERS)):
        X, G = xs[i]
        L.cks_dilated_wgrad_allreduce(geoms[i], dt, X.data_ptr(), G.data_ptr(), dws[i].data_ptr(), 0,
                                      wss[i].data_ptr(), wss[i].numel(), fused.group(i), st.cuda_stream)
    torch.cuda.synchronize()
    assert fused.errors() == [0], "cross-rank wait timed out"
    np.savez(os.environ["AR_OUT"], **{f"l{i}": t.cpu().numpy() for i, t in enumerate(dws)})
    dist.barrier()
    fused.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
