"""One small call of every kernel family of libcks.so, for compute-sanitizer
(memcheck / racecheck / synccheck): python tools/sanitize_cases.py
(prints one line per case; results are not checked here -- parity lives in
tests/; this is the sanitizer workload)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2306_15951_b200 import _lib as L  # noqa: E402
from paper_2306_15951_b200 import build  # noqa: E402
from paper_2306_15951_b200 import ops as K  # noqa: E402

build.build()
dev = torch.device("cuda", 0)
torch.manual_seed(0)


def t(shape, dtype):
    return (torch.rand(shape, device=dev) * 2 - 1).to(torch.bfloat16 if dtype == "bf16" else torch.float32)


CASES = [
    # (name, N, C, H, W, OC, F, s, p)
    ("igemm_s1", 130, 64, 9, 9, 96, 3, 1, 1),        # unit-step N-merged programs, TMA-store epilogue
    ("igemm_s2", 130, 64, 10, 10, 128, 3, 2, 1),     # KS phases, split / W-direct
    ("pair", 260, 128, 7, 7, 256, 3, 1, 1),          # CTA pairs (bf16), 2-CTA TMEM / multicast commits
    ("zc_splitk", 100, 512, 4, 4, 256, 3, 2, 1),     # cluster split-K (DSMEM reduce)
    ("narrow", 70, 3, 20, 16, 64, 7, 2, 3),          # filter-row kernels (fwd_row / wgrad_row + reduce)
    ("rowtiles", 130, 64, 40, 40, 64, 3, 1, 1),      # Sk-dilated row tiles, A1 (O_C <= 64)
    ("pad", 9, 3, 12, 13, 5, 3, 2, 1),               # channel padding (KB-PAD), odd pitches
    ("pospairs", 130, 64, 28, 28, 64, 3, 1, 1),      # Sk-dilated position pairs + filter-row groups
    ("wide", 256, 64, 28, 28, 64, 3, 1, 1),          # wide pixel blocks (two A slots per row step)
    ("pair256", 260, 256, 14, 14, 256, 3, 1, 1),     # CTA pairs (both dtypes)
    ("rg32", 32, 64, 23, 19, 64, 3, 1, 1),           # row groups: 4 rows x 32 images, position chunks
    ("rg_s2", 20, 64, 17, 15, 128, 3, 2, 1),         # row groups, element-strided A box, KS phases
    ("rg64", 50, 128, 9, 11, 96, 3, 1, 1),           # row groups of 2 rows x 64 images
    ("rg_zc", 16, 512, 4, 4, 256, 3, 2, 1),          # row groups + cluster split-K, 16-image chunks
]

for dtype in ("bf16", "tf32"):
    for name, N, C, H, W, OC, F, s, p in CASES:
        if name == "pair" and dtype == "tf32":
            continue  # pair256 covers TF32 pairs
        X = t((N, H, W, C), dtype)
        Wt = t((OC, F, F, C), dtype)
        OH, OW = (H + 2 * p - F) // s + 1, (W + 2 * p - F) // s + 1
        G = t((N, OH, OW, OC), dtype)
        K.conv2d_fwd(X, Wt, s, p)
        K.deconv2d(G, Wt, (H, W), s, p, ks_mode="stage1")
        if (C * (2 if dtype == "bf16" else 4)) % 16 == 0:
            K.deconv2d(G, Wt, (H, W), s, p, ks_mode="stage1_free")
        K.dilated_wgrad(X, G, (F, F), s, p)
        K.dilated_wgrad(X, G, (F, F), s, p, gz=3)
        K.zins_conv2d_fwd(X, Wt, s, p)
        K.zins_deconv2d(G, Wt, (H, W), s, p)
        K.zins_wgrad(X, G, (F, F), s, p)
        torch.cuda.synchronize()
        print("ok", dtype, name, flush=True)
    # 3-D
    X = t((40, 6, 9, 10, 32), dtype)
    Wt = t((48, 3, 3, 3, 32), dtype)
    G = t((40, 3, 5, 5, 48), dtype)
    K.conv3d_fwd(X, Wt, 2, 1)
    K.deconv3d(G, Wt, (6, 9, 10), 2, 1)
    K.dilated_wgrad3d(X, G, (3, 3, 3), 2, 1)
    torch.cuda.synchronize()
    print("ok", dtype, "3d", flush=True)

# fused Sk-dilated + all-reduce, two virtual ranks in one cooperative reduce launch
from paper_2306_15951_b200.dist import FusedWgradAllReduce  # noqa: E402
g = L.make_geom(33, 64, 9, 9, 64, 3, 3, 2, 2, 1, 1)
dws = [[torch.empty((64, 3, 3, 64), device=dev)] for _ in range(2)]
fused = FusedWgradAllReduce([g], dws, dev, virtual_world=2, ctas=4)
Xs = [t((33, 9, 9, 64), "bf16") for _ in range(2)]
Gs = [t((33, 5, 5, 64), "bf16") for _ in range(2)]
wss = [torch.empty(L.cks_workspace_size(g, L.CKS_BF16, L.CKS_OP_WGRAD_AR, 2), dtype=torch.uint8, device=dev)
       for _ in range(2)]
fused.run_emulated(0, [g, g], L.CKS_BF16, [x.data_ptr() for x in Xs], [y.data_ptr() for y in Gs], 2, wss,
                   torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok allreduce errors", fused.errors(), flush=True)
