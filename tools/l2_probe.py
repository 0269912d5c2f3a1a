"""Eager per-op launches of one config (one call per layer x op, in step order) for ncu metric
passes (L2 / DRAM / TMA bytes per launch).  usage: python tools/l2_probe.py CONFIG DTYPE [LAYERS|all]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import LayerBufs  # noqa: E402
from cks_synth import get_config  # noqa: E402
from paper_2306_15951_b200 import build  # noqa: E402

cfg, dt = int(sys.argv[1]), sys.argv[2]
names = None if len(sys.argv) < 4 or sys.argv[3] == "all" else sys.argv[3].split(",")
build.build()
desc, layers = get_config(cfg)
s = torch.cuda.current_stream().cuda_stream
for idx, lay in enumerate(layers):
    if names and lay.name not in names:
        continue
    b = LayerBufs(torch, lay, cfg, idx, 0, torch.device("cuda", 0), dt)
    b.dW = torch.empty((lay.OC, lay.FH, lay.FW, lay.C), dtype=torch.float32, device="cuda")
    for op in ("fwd", "deconv", "wgrad"):
        if op in lay.ops:
            b.run("deconv_w" if op == "deconv" else op, s)  # deconv: the library's policy for W given
    torch.cuda.synchronize()
    del b
print("ok")
