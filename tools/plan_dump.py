"""Print the igemm tile plan of every layer (no GPU needed: plan only) --
python tools/plan_dump.py CONFIG OP   (OP = fwd | deconv)"""
import os
import sys
import ctypes

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["CKS_PLAN_DEBUG"] = "1"
os.environ["CUDA_VISIBLE_DEVICES"] = ""  # plan only: never launch on the fake pointers below, even on a GPU box
from cks_synth import get_config  # noqa: E402
from paper_2306_15951_b200 import _lib as L  # noqa: E402

cfg, op = int(sys.argv[1]), sys.argv[2]
for lay in get_config(cfg)[1]:
    g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
    print(lay.name, flush=True)
    # fake 16-byte aligned device pointers: the launch fails after the plan is printed
    try:
        if op == "fwd":
            L.lib().cks_conv2d_fwd(ctypes.byref(g), 1, 256, 256, 256, 256, 1 << 40, None)
        else:
            L.lib().cks_deconv2d(ctypes.byref(g), 1, 256, None, 256, 256, 256, 1 << 40, None)
    except Exception:
        pass
