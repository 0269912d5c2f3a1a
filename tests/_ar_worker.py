"""Worker of tests/test_gpu_allreduce.py::test_fused_wgrad_allreduce_two_processes_ipc:
one of two processes on cuda:0 (gloo for the CUDA IPC handle exchange).

Rank 1 owns its receive buffer, dW and signal words and exports them as CUDA
IPC handles; rank 0 imports them and runs BOTH ranks' Sk-dilated + fused
reduce with cks_dilated_wgrad_allreduce_emulated (one cooperative launch:
the cross-process P2P stores of an 8-GPU node, without kernels of two
processes waiting on one another on one GPU).  Both save their dW to $AR_OUT."""
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
from paper_2306_15951_b200.dist import shard_range  # noqa: E402
from test_gpu_allreduce import LAYERS  # noqa: E402
from test_gpu_parity import dev  # noqa: E402

WORLD = 2


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    assert dist.get_world_size() == WORLD
    d = torch.device("cuda", 0)
    torch.cuda.set_device(d)
    dt = L.CKS_BF16
    nl = len(LAYERS)
    full = [L.make_geom(l.N, l.C, l.H, l.W, l.OC, l.FH, l.FW, l.sh, l.sw, l.ph, l.pw) for l in LAYERS]
    recv_off, off = [], 0
    for g in full:
        recv_off.append(off)
        off += (L.cks_ar_recv_bytes(g, WORLD) + 255) // 256 * 256
    # this process's buffer set (rank r's receive buffer, dW per layer, signal words)
    recv = torch.empty(max(off, 256), dtype=torch.uint8, device=d)
    flags = torch.zeros(2 * nl, dtype=torch.int32, device=d)
    dws = [torch.full((l.OC, l.FH, l.FW, l.C), float("nan"), device=d) for l in LAYERS]
    torch.cuda.synchronize()
    mine = (L.cks_ipc_export(recv.data_ptr()), [L.cks_ipc_export(t.data_ptr()) for t in dws],
            L.cks_ipc_export(flags.data_ptr()))
    allh = [None] * WORLD
    dist.all_gather_object(allh, mine)
    mapped = []
    if rank == 0:
        hr, hd, hf = allh[1]
        pr, pf = L.cks_ipc_import(hr), L.cks_ipc_import(hf)
        pd = [L.cks_ipc_import(h) for h in hd]
        mapped = [pr, pf] + pd
        peers = [(recv.data_ptr(), [t.data_ptr() for t in dws], flags.data_ptr()), (pr, pd, pf)]
        counts = [torch.zeros(4 * nl, dtype=torch.int32, device=d) for _ in range(WORLD)]
        errs = [torch.zeros(1, dtype=torch.int32, device=d) for _ in range(WORLD)]
        st = torch.cuda.Stream()
        keep = []
        for i, l in enumerate(LAYERS):
            a = make_layer_inputs(l, 31, i, "bf16")
            geoms, xs, gs, wss, grps = [], [], [], [], []
            for r in range(WORLD):
                lo, hi = shard_range(l.N, WORLD, r)
                X, G = dev(torch, a["X"][lo:hi], "bf16"), dev(torch, a["dY"][lo:hi], "bf16")
                g = L.make_geom(hi - lo, l.C, l.H, l.W, l.OC, l.FH, l.FW, l.sh, l.sw, l.ph, l.pw)
                ws = torch.empty(max(L.cks_workspace_size(g, dt, L.CKS_OP_WGRAD_AR), 256), dtype=torch.uint8,
                                 device=d)
                grp = L.cks_ar_group()
                grp.world, grp.rank, grp.ctas = WORLD, r, 8
                for t, (p_r, p_d, p_f) in enumerate(peers):
                    grp.recv[t] = p_r + recv_off[i]
                    grp.out[t] = p_d[i]
                    grp.flag[t] = p_f + 8 * i
                grp.count = counts[r].data_ptr() + 16 * i
                grp.err = errs[r].data_ptr()
                geoms.append(g)
                xs.append(X.data_ptr())
                gs.append(G.data_ptr())
                wss.append(ws)
                grps.append(grp)
                keep += [X, G, ws]
            L.cks_dilated_wgrad_allreduce_emulated(geoms, dt, xs, gs, [p[1][i] for p in peers], 0,
                                                   [w.data_ptr() for w in wss], [w.numel() for w in wss], grps,
                                                   st.cuda_stream)
        torch.cuda.synchronize()
        assert [int(e.item()) for e in errs] == [0] * WORLD, "cross-rank wait timed out"
    dist.barrier()  # rank 0's kernels (and their IPC stores into rank 1's dW) are complete
    np.savez(os.environ["AR_OUT"], **{f"l{i}": t.cpu().numpy() for i, t in enumerate(dws)})
    dist.barrier()
    for p in mapped:
        L.cks_ipc_close(p)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
