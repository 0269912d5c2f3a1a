"""Probe: which CUDA-graph shapes of the step can ncu replay node by node?
usage: python tools/ncu_graph_probe.py VARIANT   (run under ncu)
  eager   one igemm op launched eagerly
  g1      a graph holding that single op
  g2      a graph: wgrad op (row kernel + G_Z reduce) then the igemm op
  g2ev    as g2 with timing-event nodes between the ops (bench's serialized graph)
  g3ev    three ops (stem fwd, stem wgrad, l1 fwd) with event nodes, after a flush fill
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import LayerBufs  # noqa: E402
from cks_synth import get_config  # noqa: E402
from paper_2306_15951_b200 import build  # noqa: E402

build.build()
v = sys.argv[1]
dtype = sys.argv[2] if len(sys.argv) > 2 else "tf32"
desc, layers = get_config(2)
dev = torch.device("cuda", 0)
b = LayerBufs(torch, layers[1], 2, 1, 0, dev, dtype)   # l1_0
b.dW = torch.empty((b.lay.OC, b.lay.FH, b.lay.FW, b.lay.C), dtype=torch.float32, device=dev)
s0 = LayerBufs(torch, layers[0], 2, 0, 0, dev, dtype)  # stem
s0.dW = torch.empty((s0.lay.OC, s0.lay.FH, s0.lay.FW, s0.lay.C), dtype=torch.float32, device=dev)
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    b.run("fwd", st.cuda_stream)
    s0.run("wgrad", st.cuda_stream)
torch.cuda.synchronize()
if v == "eager":
    with torch.cuda.stream(st):
        b.run("fwd", st.cuda_stream)
else:
    ev = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(4)]
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        sp = torch.cuda.current_stream().cuda_stream
        if v == "g3ev":
            ev[0].record()
            s0.run("fwd", sp)
        if v in ("g2", "g2ev", "g3ev"):
            if v != "g2":
                ev[1].record()
            s0.run("wgrad", sp)
        if v != "g2" and v != "g1":
            ev[2].record()
        b.run("fwd", sp)
        if v != "g2" and v != "g1":
            ev[3].record()
    with torch.cuda.stream(st):
        flush.fill_(1.0)
        g.replay()
torch.cuda.synchronize()
print("ok", v)
