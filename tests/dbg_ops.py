"""Run fwd / deconv / wgrad of one layer separately with a sync after each (debug; test infrastructure: compares with the oracle).
usage: python tests/dbg_ops.py N C H W OC FH FW sh sw ph pw [ops]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))  # repo root
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
from cks_synth import Layer, bf16_bits, make_layer_inputs  # noqa: E402
from paper_2306_15951_b200 import ops as K  # noqa: E402

a = [int(v) for v in sys.argv[1:12]]
ops = sys.argv[12].split(",") if len(sys.argv) > 12 else ["fwd", "wgrad", "deconv"]
lay = Layer("dbg", *a)
inp = make_layer_inputs(lay, 0, 0, "bf16")
dev = {k: torch.from_numpy(bf16_bits(v).view(np.int16)).view(torch.bfloat16).cuda() for k, v in inp.items()}
s, p = (lay.sh, lay.sw), (lay.ph, lay.pw)
for op in ops:
    if op == "fwd":
        y = K.conv2d_fwd(dev["X"], dev["W"], s, p)
        torch.cuda.synchronize()
        ref = O.conv_ref(inp["X"], inp["W"], lay.sh, lay.sw, lay.ph, lay.pw)
    elif op == "wgrad":
        y = K.dilated_wgrad(dev["X"], dev["dY"], (lay.FH, lay.FW), s, p)
        torch.cuda.synchronize()
        ref = O.wgrad_ref(inp["X"], inp["dY"], lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    else:
        y = K.deconv2d(dev["dY"], dev["W"], (lay.H, lay.W), s, p)
        torch.cuda.synchronize()
        ref = O.deconv_ref(inp["dY"], inp["W"], lay.H, lay.W, lay.sh, lay.sw, lay.ph, lay.pw)
    g = y.cpu().numpy().astype(np.float64)
    e = np.linalg.norm(g - ref) / max(np.linalg.norm(ref), 1e-30)
    print(f"{op}: normwise err {e:.3e}", flush=True)
    if e > 1e-3:
        d = np.abs(g - ref)
        idx = np.unravel_index(np.argmax(d), d.shape)
        print("  worst at", idx, "got", g[idx], "ref", ref[idx])
