"""GPU test of the data-parallel path's collective: a
1-rank NCCL process group, the per-layer Sk-dilated partial dW written into
one flat fp32 buffer (dist.FlatGrads), and the bucketed all_reduce captured
inside a CUDA graph behind the wgrad launches exactly as bench.py schedules
it -- the reduced dW is compared with the fp64 oracle.  With one rank the SUM
is the identity, so this pins the plumbing (NCCL in-graph capture, bucket
offsets, stream ordering); the cross-rank arithmetic is covered by the
world-2 gloo test (tests/test_dist_gloo.py).  The paper's map-reduce over
G_K = N*O_H*O_W is the operation the collective completes."""
import socket

import numpy as np
import pytest

import oracle as O
from cks_synth import Layer, make_layer_inputs

from test_gpu_parity import check, dev, red_len, torch_cuda  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dtype", ["bf16", "tf32"])
def test_nccl_bucketed_allreduce_in_graph(torch_cuda, dtype):
    torch = torch_cuda
    import torch.distributed as dist
    from paper_2306_15951_b200 import ops as K
    from paper_2306_15951_b200.dist import FlatGrads
    lays = [Layer("d0", 131, 64, 14, 14, 128, 3, 3, 2, 2, 1, 1),
            Layer("d1", 131, 128, 7, 7, 256, 3, 3, 1, 1, 1, 1),
            Layer("d2", 131, 3, 28, 28, 64, 7, 7, 2, 2, 3, 3)]
    dev0 = torch.device("cuda", 0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{_free_port()}", rank=0, world_size=1,
                            device_id=dev0)
    try:
        ins = [make_layer_inputs(l, 21, i, dtype) for i, l in enumerate(lays)]
        Xs = [dev(torch, a["X"], dtype) for a in ins]
        Gs = [dev(torch, a["dY"], dtype) for a in ins]
        fg = FlatGrads([(l.OC, l.FH, l.FW, l.C) for l in lays], dev0)
        fg.flat.fill_(float("nan"))  # every element must be overwritten by the wgrads
        main, side, comm = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
        # warm-up (communicator, smem attributes, workspaces) outside the capture
        with torch.cuda.stream(side):
            for i, l in enumerate(lays):
                K.dilated_wgrad(Xs[i], Gs[i], (l.FH, l.FW), (l.sh, l.sw), (l.ph, l.pw), out=fg.views[i],
                                stream=side)
        torch.cuda.synchronize()
        with torch.cuda.stream(comm):
            dist.all_reduce(fg.flat)
        torch.cuda.synchronize()
        fg.flat.fill_(float("nan"))
        torch.cuda.synchronize()
        sizes = [v.numel() for v in fg.views]
        offs = np.cumsum([0] + sizes)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=main):
            fork = torch.cuda.Event()
            fork.record(main)
            side.wait_event(fork)
            # backward order, wgrads on the side stream, one bucket per layer
            for i in reversed(range(len(lays))):
                l = lays[i]
                with torch.cuda.stream(side):
                    K.dilated_wgrad(Xs[i], Gs[i], (l.FH, l.FW), (l.sh, l.sw), (l.ph, l.pw), out=fg.views[i],
                                    stream=side)
                    done = torch.cuda.Event()
                    done.record(side)
                comm.wait_event(done)
                with torch.cuda.stream(comm):
                    dist.all_reduce(fg.flat[int(offs[i]):int(offs[i + 1])])
            for s in (side, comm):
                j = torch.cuda.Event()
                j.record(s)
                main.wait_event(j)
        for _ in range(2):  # replay twice: results independent of the previous contents
            g.replay()
        torch.cuda.synchronize()
        got = fg.flat.cpu().numpy()
        for i, (l, a) in enumerate(zip(lays, ins)):
            ref = O.wgrad_ref(a["X"], a["dY"], l.FH, l.FW, l.sh, l.sw, l.ph, l.pw)
            part = got[int(offs[i]):int(offs[i + 1])].reshape(ref.shape)
            check(part, ref, dtype, f"{l.name} NCCL-reduced dW", red_len(l, "wgrad"))
    finally:
        dist.destroy_process_group()
