"""GPU tests of the fused Sk-dilated + cross-rank all-reduce (KB-REDUCE-AR,
cks_dilated_wgrad_allreduce).  The batch is split into
W contiguous shards (dist.shard_range); each "rank" computes Sk-dilated on its
shard and one kernel per rank aggregates the G_Z segments and the ranks'
partials through peer memory (the paper's map-reduce over G_K = N*O_H*O_W,
P:210, with the shard as the outermost segment).  Every rank must hold the
full-batch dW of the fp64 oracle, bit-identical across ranks and repeats.

* virtual ranks: W buffer sets in one process, run by
  cks_dilated_wgrad_allreduce_emulated: every rank's Sk-dilated, then ONE
  cooperative KB-REDUCE-AR launch over all ranks (grid.y = rank).  Kernels that
  wait on one another are never separate launches on one GPU -- nothing
  guarantees they are co-scheduled (B200_PROFILING.md: Xid 109 with 2-4 such
  ranks as processes on one GPU);
* two processes: rank 1's receive buffer, dW and signal words are exported as
  CUDA IPC handles over a gloo group and imported by rank 0, which runs both
  ranks' reduce in its one cooperative launch -- the cross-process P2P stores
  and the handle exchange of an 8-GPU node, without cross-process waits.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

import oracle as O
from cks_synth import Layer, make_layer_inputs

from test_gpu_parity import check, dev, red_len, torch_cuda  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

LAYERS = [Layer("ar0", 131, 64, 14, 14, 128, 3, 3, 2, 2, 1, 1),    # G_Z partials (KB-REDUCE path)
          Layer("ar1", 131, 256, 7, 7, 256, 3, 3, 1, 1, 1, 1),     # in-cluster G_Z reduce plans
          Layer("ar2", 131, 3, 28, 28, 64, 7, 7, 2, 2, 3, 3),      # narrow-channel row kernel (stem-like)
          Layer("ar3", 131, 64, 9, 9, 64, 1, 1, 2, 2, 0, 0)]       # 1x1 s2, short reduction


def _run_virtual(torch, world, dtype, reps=2):
    from paper_2306_15951_b200 import _lib as L
    from paper_2306_15951_b200.dist import FusedWgradAllReduce, shard_range
    dt = L.CKS_BF16 if dtype == "bf16" else L.CKS_TF32
    ins = [make_layer_inputs(l, 31, i, dtype) for i, l in enumerate(LAYERS)]
    dev0 = torch.device("cuda", 0)
    shards, geoms = [], []
    for l, a in zip(LAYERS, ins):
        X, G = dev(torch, a["X"], dtype), dev(torch, a["dY"], dtype)
        per = []
        for r in range(world):
            lo, hi = shard_range(l.N, world, r)
            per.append((X[lo:hi].contiguous(), G[lo:hi].contiguous(), hi - lo))
        shards.append(per)
    dws = [[torch.full((l.OC, l.FH, l.FW, l.C), float("nan"), device=dev0) for l in LAYERS] for _ in range(world)]
    # one geometry per (layer): the shards differ in N by <= 1; the group's buffers
    # are sized from the largest shard's geometry (dW does not depend on N)
    for l in LAYERS:
        geoms.append(L.make_geom(shard_range(l.N, world, 0)[1], l.C, l.H, l.W, l.OC, l.FH, l.FW, l.sh, l.sw,
                                 l.ph, l.pw))
    fused = FusedWgradAllReduce(geoms, dws, dev0, virtual_world=world, ctas=8)
    stream = torch.cuda.Stream()
    wss = []
    for r in range(world):
        per = []
        for i, l in enumerate(LAYERS):
            g = L.make_geom(shards[i][r][2], l.C, l.H, l.W, l.OC, l.FH, l.FW, l.sh, l.sw, l.ph, l.pw)
            per.append(torch.empty(max(L.cks_workspace_size(g, dt, L.CKS_OP_WGRAD_AR, 2), 256), dtype=torch.uint8,
                                   device=dev0))
        wss.append(per)
    results = []
    for _ in range(reps):
        torch.cuda.synchronize()
        for i, l in enumerate(LAYERS):
            gs = [L.make_geom(shards[i][r][2], l.C, l.H, l.W, l.OC, l.FH, l.FW, l.sh, l.sw, l.ph, l.pw)
                  for r in range(world)]
            fused.run_emulated(i, gs, dt, [shards[i][r][0].data_ptr() for r in range(world)],
                               [shards[i][r][1].data_ptr() for r in range(world)], 2,
                               [wss[r][i] for r in range(world)], stream.cuda_stream)
        torch.cuda.synchronize()
        assert fused.errors() == [0] * world, "a cross-rank wait timed out"
        results.append([[d.cpu().numpy() for d in dws[r]] for r in range(world)])
    return ins, results


@pytest.mark.parametrize("world,dtype", [(2, "bf16"), (3, "tf32"), (4, "bf16")])
def test_fused_wgrad_allreduce_virtual_ranks(torch_cuda, world, dtype):
    ins, results = _run_virtual(torch_cuda, world, dtype)
    for i, (l, a) in enumerate(zip(LAYERS, ins)):
        ref = O.wgrad_ref(a["X"], a["dY"], l.FH, l.FW, l.sh, l.sw, l.ph, l.pw)
        got0 = results[0][0][i]
        check(got0, ref, dtype, f"{l.name} fused all-reduce dW (world {world})", red_len(l, "wgrad"))
        for rep in results:
            for r in range(world):  # bit-identical on every rank and every repeat (fixed order)
                assert np.array_equal(rep[r][i], got0), (l.name, r)


def test_fused_wgrad_allreduce_two_processes_ipc(torch_cuda, tmp_path):
    """Two processes on cuda:0, buffers shared by CUDA IPC handles over gloo."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    procs = []
    for r in range(2):
        env = dict(os.environ, RANK=str(r), WORLD_SIZE="2", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port),
                   AR_OUT=str(tmp_path / f"dw{r}.npz"))
        procs.append(subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "_ar_worker.py")], env=env,
                                      cwd=ROOT, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True))
    outs = [p.communicate(timeout=600)[0] for p in procs]
    for p, o in zip(procs, outs):
        assert p.returncode == 0, o[-3000:]
    d0, d1 = np.load(tmp_path / "dw0.npz"), np.load(tmp_path / "dw1.npz")
    for i, l in enumerate(LAYERS):
        a = make_layer_inputs(l, 31, i, "bf16")
        ref = O.wgrad_ref(a["X"], a["dY"], l.FH, l.FW, l.sh, l.sw, l.ph, l.pw)
        check(d0[f"l{i}"], ref, "bf16", f"{l.name} IPC fused all-reduce dW", red_len(l, "wgrad"))
        assert np.array_equal(d0[f"l{i}"], d1[f"l{i}"])
