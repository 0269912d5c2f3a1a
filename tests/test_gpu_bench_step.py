"""The benchmarked step computes the right thing: bench.measure() runs the
training-step schedule graph (forward chain, Stage1-free / split KS-deconv
chain, Sk-dilated on two side streams), the per-op graph and the evented
graph; afterwards every layer's Y, dX and dW buffers hold the results of the
last replay -- compared here with the fp64 oracle on the inputs the bench
generated (reduced batch, every C3 ResNet-18 layer, both precisions)."""
import argparse

import numpy as np
import pytest

import oracle as O

from test_gpu_parity import check, red_len, torch_cuda  # noqa: F401  (fixture)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["tf32", "bf16"])
def test_bench_step_results(torch_cuda, dtype):
    torch = torch_cuda
    import torch.distributed as dist
    import bench
    args = argparse.Namespace(config=2, batch=3, steps=2, warmup=1, layers=False, allreduce="nccl")
    m = bench.measure(args, torch, dist, torch.device("cuda", 0), 0, 0, 1, False, dtype)
    torch.cuda.synchronize()
    assert m["ms_per_step"] > 0 and m["roofline"]["busy_ms_per_step"] <= m["roofline"]["evented_step_ms"] + 1e-6
    for b in m["bufs"]:
        lay, a = b.lay, b.host
        s = (lay.sh, lay.sw, lay.ph, lay.pw)
        if "fwd" in lay.ops:
            check(b.Y.cpu().numpy(), O.conv_ref(a["X"], a["W"], *s), dtype, f"bench {lay.name} Y", red_len(lay, "fwd"))
        if "deconv" in lay.ops:
            check(b.dX.cpu().numpy(), O.deconv_ref(a["dY"], a["W"], lay.H, lay.W, *s), dtype, f"bench {lay.name} dX",
                  red_len(lay, "deconv"))
        if "wgrad" in lay.ops:
            check(b.dW.cpu().numpy(), O.wgrad_ref(a["X"], a["dY"], lay.FH, lay.FW, *s), dtype,
                  f"bench {lay.name} dW", red_len(lay, "wgrad"))
