"""Print the tile plan of every layer (host only: cks_plan_describe) --
python tools/plan_dump.py CONFIG OP [DTYPE]   (OP = fwd | deconv | wgrad, DTYPE = bf16 | tf32)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from cks_synth import get_config  # noqa: E402
from paper_2306_15951_b200 import _lib as L  # noqa: E402

cfg, op = int(sys.argv[1]), sys.argv[2]
dt = L.CKS_TF32 if len(sys.argv) > 3 and sys.argv[3] == "tf32" else L.CKS_BF16
code = {"fwd": L.CKS_OP_FWD, "deconv": L.CKS_OP_DECONV, "wgrad": L.CKS_OP_WGRAD}[op]
for lay in get_config(cfg)[1]:
    g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    print(lay.name)
    print("[cks plan]", L.cks_plan_describe(g, dt, code))
