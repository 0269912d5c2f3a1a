"""Debug timeline of one igemm launch (CTAs 0..3): python tools/trace_op.py CONFIG LAYER OP"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CKS_EXPERIMENTS"] = "1"  # the debug timeline exists only in the experiments build
import torch  # noqa: E402

from paper_2306_15951_b200 import build  # noqa: E402

build.build()

from bench import LayerBufs  # noqa: E402
from cks_synth import get_config  # noqa: E402

cfg, name, op = int(sys.argv[1]), sys.argv[2], sys.argv[3]
desc, layers = get_config(cfg)
idx = [l.name for l in layers].index(name)
b = LayerBufs(torch, layers[idx], cfg, idx, 0, torch.device("cuda", 0), os.environ.get("CKS_DTYPE", "bf16"))
b.dW = torch.empty((b.lay.OC, b.lay.FH, b.lay.FW, b.lay.C), dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
b.run(op, s)
torch.cuda.synchronize()
tr = torch.zeros(4 * 5 * 1024 + 148 * 8, dtype=torch.int64, device="cuda")
os.environ["CKS_TRACE_PTR"] = hex(tr.data_ptr())
b.run(op, s)
torch.cuda.synchronize()
del os.environ["CKS_TRACE_PTR"]
full = tr.cpu().numpy()
t = full[:4 * 5 * 1024].reshape(4, 5, 1024)
g = full[4 * 5 * 1024:].reshape(148, 8)
names = {0: ["start", "Bissue", "Aissue"], 1: ["start", "Bready", "Aready", "accfree", "Adone"],
         2: ["start", "tfull", "drained", "atomic", "reduced"], 3: ["start", "Bissue", "Aissue"],
         4: ["start", "Bissue", "Aissue"]}
for cta in range(2):
    base = None
    for role in (0, 3, 4, 1, 2):
        ev = [(int(v) >> 56, int(v) & ((1 << 56) - 1)) for v in t[cta, role] if v != 0]
        if not ev:
            continue
        if base is None:
            base = min(e[1] for e in ev)
        line = " ".join(f"{names[role][c] if c < len(names[role]) else c}@{ts - base}" for c, ts in ev[:80])
        print(f"cta{cta} role{role} n={len(ev)}: {line}\n")

import numpy as np
act = g[g[:, 0] != 0]
t0 = act[:, 0].min()
names_g = ["entry", "setup", "pdlwait", "firstB", "lastmma", "exit"]
print("CTAs active:", len(act))
for k, nm in enumerate(names_g):
    col = act[:, k]
    col = col[col != 0]
    if len(col):
        print(f"{nm:8s} min {(col.min()-t0)/1e3:7.2f} us  med {(np.median(col)-t0)/1e3:7.2f} us  max {(col.max()-t0)/1e3:7.2f} us")
