"""Warm-L2 per-op timing of one (config, layer, op): CUDA events over R reps.
usage: python tools/time_op.py CONFIG OP LAYER[,LAYER...]|all [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import LayerBufs  # noqa: E402
from paper_2306_15951_b200 import build  # noqa: E402
from cks_synth import get_config  # noqa: E402


def main():
    cfg, op = int(sys.argv[1]), sys.argv[2]
    names = sys.argv[3].split(",") if sys.argv[3] != "all" else None
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 50
    build.build()  # libcks.so, or libcks_exp.so under CKS_EXPERIMENTS=1 (knob sweeps)
    desc, layers = get_config(cfg)
    s = torch.cuda.current_stream()
    for idx, lay in enumerate(layers):
        base = "deconv" if op in ("split", "deconv_only", "deconv_w", "deconv_free") else op
        if names and lay.name not in names or base not in lay.ops:
            continue
        b = LayerBufs(torch, lay, cfg, idx, 0, torch.device("cuda", 0), os.environ.get("CKS_DTYPE", "bf16"))
        b.dW = torch.empty((lay.OC, lay.FH, lay.FW, lay.C), dtype=torch.float32, device="cuda")
        for _ in range(3):
            b.run(op, s.cuda_stream)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                b.run(op, torch.cuda.current_stream().cuda_stream)
        for _ in range(int(os.environ.get("TIME_OP_WARM", "1"))):  # clock ramp-up
            g.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / reps
        print(f"{lay.name:22s} {op:6s} {us:8.2f} us  {b.flops / us / 1e6:8.1f} TFLOP/s  flags={os.environ.get('CKS_DEBUG_FLAGS', '0')}")


if __name__ == "__main__":
    main()
