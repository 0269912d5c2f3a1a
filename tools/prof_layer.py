"""Run one (config, layer, op) of the hot path a few times -- for ncu captures.
usage: python tools/prof_layer.py CONFIG LAYER_NAME OP [REPS]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from bench import LayerBufs  # noqa: E402
from paper_2306_15951_b200 import build  # noqa: E402
from cks_synth import get_config  # noqa: E402


def main():
    cfg, name, op = int(sys.argv[1]), sys.argv[2], sys.argv[3]
    reps = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    build.build()  # libcks.so, or libcks_exp.so under CKS_EXPERIMENTS=1 (knob sweeps)
    desc, layers = get_config(cfg, int(os.environ["CKS_BATCH"]) if os.environ.get("CKS_BATCH") else None)
    idx = [l.name for l in layers].index(name)
    b = LayerBufs(torch, layers[idx], cfg, idx, 0, torch.device("cuda", 0),
                  os.environ.get("CKS_DTYPE", "bf16"))
    b.dW = torch.empty((b.lay.OC, b.lay.FH, b.lay.FW, b.lay.C), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    for _ in range(reps):
        b.run(op, s)
    torch.cuda.synchronize()
    print("ok", name, op)


if __name__ == "__main__":
    main()
