#!/usr/bin/env python
"""bench.py -- one JSON line: zero-free TFLOP/s and ms per op (fwd / deconv /
wgrad) of the C-K-S hot path on B200 (BASELINE.json metric).

A "step" is one pass of the whole hot path over one batch of the workload:
for every layer of the workload, ConvV2 forward, KS-deconv-V2 (Stage1 split
+ fused Stage2&3) and Sk-dilated-V2 weight gradient (+ G_Z reduce), as in a
conv-layer training step.  Default workload: configs[4], C5 --
the ResNet-18 conv-layer train step (the 20 conv layers of ResNet-18 @224),
N = 256 per GPU, the largest single-GPU configuration (2,521 zero-free GFLOP
per step); weak scaling, global batch 256 x n_gpus.  Headline precision:
fp32 inputs multiplied as TF32 (the paper computes in fp32), with the
same step in BF16 reported beside it.  With N > 1 GPUs every rank runs its
batch shard and the per-layer dW are summed with bucketed NCCL all_reduces
overlapping the backward (``--gpus N`` without torchrun launches the N ranks).

Timing: inputs resident in HBM; the step is one CUDA graph (the C-ABI calls
captured once) replayed K times after W warm-ups; L2 is flushed (256 MB
write) before every timed step, outside the timed events; the step time is
the max over ranks.  The roofline's kernel durations come from a copy of the
same schedule graph with events on each op's launching stream; per-op /
per-layer numbers follow the paper's per-op protocol (each op alone).
``e2e`` repeats the step through the public Python API without graphs, with
the step's inputs copied host->device from pinned memory and the results
copied back inside the timed region.
``--impl reference`` times the fp64 CPU oracle (oracle/) on a bounded
sample of the same workload on the host cores (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "zero-free TFLOP/s and ms per op (fwd/deconv/wgrad) at 1/2/4/8 B200"
_JSON_OUT = None  # original stdout when fd 1 is redirected (multi-rank runs)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1,
                    help="GPUs of this node; without torchrun, N > 1 launches N ranks itself (torch.distributed.run)")
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("cks", "reference"), default="cks")
    ap.add_argument("--config", type=int, default=4,
                    help="BASELINE configs index (default 4: C5, the ResNet-18 conv-layer train step, N=256 per GPU "
                         "-- the largest single-GPU workload; 1: C2 VGG sweep, 2: C3 layers, 3: C4 DCGAN, 5: C6 5x5)")
    ap.add_argument("--batch", type=int, default=None, help="override per-GPU batch")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0, help="seconds of oracle work for cpu_baseline")
    ap.add_argument("--layers", action="store_true", help="per-layer breakdown on stderr")
    ap.add_argument("--no-zins", action="store_true", help="skip the zero-inserted-formulation comparison")
    ap.add_argument("--dtype", choices=("bf16", "tf32"), default="tf32",
                    help="headline: fp32 inputs multiplied as TF32 (the paper computes in fp32, P:262), or bf16 "
                         "inputs; fp32 accumulate and outputs either way")
    ap.add_argument("--allreduce", choices=("nccl", "fused"), default="nccl",
                    help="N > 1: dW sum by bucketed NCCL all_reduce in the step graph, or fused into the Sk-dilated "
                         "G_Z reduce (KB-REDUCE-AR over NVLink peer memory, CUDA IPC)")
    ap.add_argument("--companion", choices=("bf16", "tf32", "none"), default="bf16",
                    help="also time the step in this input precision and report it beside the headline")
    return ap.parse_args()


def self_launch(args):
    """--gpus N without torchrun: run this script as N ranks (one per GPU) with
    torch.distributed.run on 127.0.0.1; rank 0 prints the JSON line."""
    import socket
    import subprocess
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# --------------------------------------------------------------------- oracle
def oracle_sample(layers, config, n_sub, budget_s=None):
    """Run the fp64 oracle (as it stands) over every layer of the workload with
    n_sub images; returns (seconds, zero-free flops, passes)."""
    import oracle as O
    from cks_synth import make_layer_inputs
    samples = []
    for i, lay in enumerate(layers):
        l1 = lay.with_batch(n_sub)
        samples.append((l1, make_layer_inputs(l1, config, i, "bf16")))
    flops_pass = 0
    for l1, _ in samples:
        f = O.op_counts(O.geom(**l1.geom()))["zero_free_flops"]
        flops_pass += f * len(l1.ops)
    t0 = time.perf_counter()
    passes = 0
    while True:
        for l1, a in samples:
            s = (l1.sh, l1.sw, l1.ph, l1.pw)
            if "fwd" in l1.ops:
                O.conv_ref(a["X"], a["W"], *s)
            if "deconv" in l1.ops:
                O.deconv_ref(a["dY"], a["W"], l1.H, l1.W, *s)
            if "wgrad" in l1.ops:
                O.wgrad_ref(a["X"], a["dY"], l1.FH, l1.FW, *s)
        passes += 1
        el = time.perf_counter() - t0
        if budget_s is None or el >= budget_s:
            return el, flops_pass * passes, passes


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max((d.get("num_threads", 1) for d in threadpool_info()), default=1)
    except Exception:
        return os.cpu_count() or 1


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    from cks_synth import get_config
    desc, layers = get_config(args.config, args.batch)
    n_sub = 1
    for _ in range(args.warmup):
        oracle_sample(layers, args.config, n_sub)
    times, flops = [], 0
    for _ in range(args.steps):
        el, f, _ = oracle_sample(layers, args.config, n_sub)
        times.append(el)
        flops = f
    ms = 1e3 * statistics.mean(times)
    value = flops / (ms / 1e3) / 1e12
    cores = blas_threads()
    sample = f"all {len(layers)} layers x ops of '{desc}' at N={n_sub} image per step (oracle cost is linear in N)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": desc, "per_gpu_batch": layers[0].N, "sample_batch": n_sub,
                   "parallelism": "host cores (oracle)"},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi sampling (every 50 ms) of SM clock and throttle reasons during
    the timed region -- the profiling recipe's clocks line."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.out = None

    def __enter__(self):
        import subprocess
        import tempfile
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=self.out,
                                         stderr=subprocess.DEVNULL)
            time.sleep(0.3)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            with open(self.out.name) as f:
                for line in f:
                    parts = [x.strip() for x in line.split(",")]
                    if len(parts) < 6:
                        continue
                    try:
                        sm.append(float(parts[0]))
                        mx = float(parts[1])
                    except ValueError:
                        continue
                    for nm, v in zip(names, parts[2:6]):
                        if v.lower() in ("active", "1"):
                            reasons.add(nm)
            os.unlink(self.out.name)
        except Exception:
            pass
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------- GPU arm
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return {"hbm": float(d["hbm_gbs"]), "bf16": float(d["bf16_tflops"]),
                "bf16_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])), "src": "measured"}
    except Exception:
        return {"hbm": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "src": "fallback"}


def load_traffic(kernel, config, dtype):
    """dram bytes per launch of a kernel family on this workload (config, dtype)
    from the committed ncu capture (tools/summarize_profiles.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(f"config{config}/{dtype}", {}).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


class LayerBufs:
    """Device buffers + the C-ABI calls of one layer (argument marshalling only)."""

    def __init__(self, torch, lay, config, idx, rank, device, dtype="bf16"):
        import numpy as np
        from cks_synth import bf16_bits, make_layer_inputs
        from paper_2306_15951_b200 import _lib as L
        self.lay, self.L = lay, L
        self.dt = L.CKS_BF16 if dtype == "bf16" else L.CKS_TF32
        a = make_layer_inputs(lay, config + 100 * rank, idx, dtype)

        def dev(x):
            if dtype == "tf32":
                return torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).to(device)
            return torch.from_numpy(bf16_bits(x).view(np.int16)).view(torch.bfloat16).to(device)
        self.host = {k: v for k, v in a.items()}
        self.X, self.W, self.G = dev(a["X"]), dev(a["W"]), dev(a["dY"])
        OH, OW = lay.out_hw()
        f32 = dict(dtype=torch.float32, device=device)
        self.Y = torch.empty((lay.N, OH, OW, lay.OC), **f32)
        self.dX = torch.empty((lay.N, lay.H, lay.W, lay.C), **f32)
        self.dW = None  # view into the flat allreduce buffer, set by the caller
        g = L.make_geom(lay.N, lay.C, lay.H, lay.W, lay.OC, lay.FH, lay.FW, lay.sh, lay.sw, lay.ph, lay.pw)
        self.g = g
        cnt = L.cks_op_counts(g)
        self.flops = 2 * cnt["zero_free_macs"]
        # algorithmic bytes (read inputs once, write the fp32 output once)
        eb = 2 if dtype == "bf16" else 4
        xb, wb, gb = lay.N * lay.H * lay.W * lay.C * eb, lay.OC * lay.FH * lay.FW * lay.C * eb, lay.N * OH * OW * lay.OC * eb
        self.algo_bytes = {"fwd": xb + wb + (gb // eb) * 4,
                           "deconv": gb + wb + (xb // eb) * 4, "wgrad": xb + gb + (wb // eb) * 4, "split": 2 * wb}
        self.cp = torch.empty(L.cks_ks_split_size(g, self.dt) // eb, dtype=self.X.dtype, device=device)
        self.ws = {}
        for op, code in (("fwd", L.CKS_OP_FWD), ("deconv", L.CKS_OP_DECONV), ("wgrad", L.CKS_OP_WGRAD)):
            n = L.cks_workspace_size(g, self.dt, code)
            self.ws[op] = torch.empty(max(n, 256), dtype=torch.uint8, device=device)
        self.launches = {
            "fwd": L.cks_launch_count(g, self.dt, L.CKS_OP_FWD),
            "split": 1,
            "deconv": L.cks_launch_count(g, self.dt, L.CKS_OP_DECONV, c_packed_given=True),
            "deconv_w": L.cks_launch_count(g, self.dt, L.CKS_OP_DECONV),
            "wgrad": L.cks_launch_count(g, self.dt, L.CKS_OP_WGRAD),
        }
        # KS-deconv without Stage1 (the GEMM reads W directly) where the library's
        # policy takes it; eligible: W rows of a 16-byte multiple, sw <= 8
        pd = L.plan_dict(g, self.dt, L.CKS_OP_DECONV) if "deconv" in lay.ops else {}
        # W given: Stage1-free, or (narrow outputs) the multi-phase tile -- no separate Stage1 either way
        self.direct = pd.get("ks_direct") == "1" or pd.get("ks_mp") == "1"
        self.direct_ok = "deconv" in lay.ops and (lay.C * eb) % 16 == 0 and lay.sw <= 8

    def run_split(self, stream_ptr):
        self.L.cks_ks_split(self.g, self.dt, self.W.data_ptr(), self.cp.data_ptr(), stream_ptr)

    def run(self, op, stream_ptr):
        L, g = self.L, self.g
        if op == "split":  # Stage1 alone
            L.cks_ks_split(g, self.dt, self.W.data_ptr(), self.cp.data_ptr(), stream_ptr)
            return
        if op in ("deconv_w", "deconv_free"):  # W given: library policy / forced Stage1-free
            ws = self.ws["deconv"]
            L.cks_deconv2d_ex(g, self.dt, self.G.data_ptr(), self.W.data_ptr(), None, self.dX.data_ptr(),
                              ws.data_ptr(), ws.numel(), stream_ptr,
                              L.CKS_KS_AUTO if op == "deconv_w" else L.CKS_KS_STAGE1_FREE)
            return
        if op == "wgrad_ar":  # Sk-dilated + G_Z and cross-rank reduce in one kernel (KB-REDUCE-AR)
            ws = self.ws["wgrad_ar"]
            L.cks_dilated_wgrad_allreduce(g, self.dt, self.X.data_ptr(), self.G.data_ptr(), self.dW.data_ptr(), 0,
                                          ws.data_ptr(), ws.numel(), self.ar_grp, stream_ptr)
            return
        if op == "deconv_only":  # Stage2&3 from the already split sub-filters
            ws = self.ws["deconv"]
            L.cks_deconv2d(g, self.dt, self.G.data_ptr(), None, self.cp.data_ptr(), self.dX.data_ptr(),
                           ws.data_ptr(), ws.numel(), stream_ptr)
            return
        ws = self.ws[op]
        if op == "fwd":
            L.cks_conv2d_fwd(g, self.dt, self.X.data_ptr(), self.W.data_ptr(), self.Y.data_ptr(), ws.data_ptr(),
                             ws.numel(), stream_ptr)
        elif op == "deconv":  # Stage1 (W changes every training step) + fused Stage2&3
            L.cks_ks_split(g, self.dt, self.W.data_ptr(), self.cp.data_ptr(), stream_ptr)
            L.cks_deconv2d(g, self.dt, self.G.data_ptr(), None, self.cp.data_ptr(), self.dX.data_ptr(),
                           ws.data_ptr(), ws.numel(), stream_ptr)
        else:
            L.cks_dilated_wgrad(g, self.dt, self.X.data_ptr(), self.G.data_ptr(), self.dW.data_ptr(), 0,
                                ws.data_ptr(), ws.numel(), stream_ptr)


KIND_KERNEL = {"igemm": "igemm_kernel", "row_fwd": "fwd_row_kernel", "row_wgrad": "wgrad_row_kernel",
               "wgrad": "wgrad_kernel"}


def op_kernel(b, op):
    """Kernel family an op of the step launches (its plan's main kernel; the
    op's time includes its staging kernels: G_Z reduce, channel padding)."""
    if op == "split":
        return "ks_split_kernel"
    code = {"fwd": 0, "deconv_only": 1, "deconv": 1, "deconv_w": 1, "deconv_free": 1, "wgrad": 2, "wgrad_ar": 2}[op]
    kind = b.L.plan_dict(b.g, b.dt, code)["kind"]
    return KIND_KERNEL.get(kind, kind)


def union_ms(iv):
    """Length of the union of intervals [(s, e)] (ms)."""
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in sorted(iv):
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def measure(args, torch, dist, device, rank, local, n_gpus, use_dist, dtype, headline=True):
    """Build one workload in `dtype` and time it.  Returns the bench fields."""
    from cks_synth import get_config
    desc, layers = get_config(args.config, args.batch)
    bufs = [LayerBufs(torch, lay, args.config, i, rank, device, dtype) for i, lay in enumerate(layers)]
    # flat dW buffer: the bucketed NCCL all_reduce works on slices of it
    sizes = [b.lay.OC * b.lay.FH * b.lay.FW * b.lay.C for b in bufs]
    flat = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
    off = 0
    for b, s in zip(bufs, sizes):
        b.dW = flat[off:off + s].view(b.lay.OC, b.lay.FH, b.lay.FW, b.lay.C)
        off += s
    fused_ar = use_dist and args.allreduce == "fused"
    if fused_ar:  # per-layer KB-REDUCE-AR groups: peers' buffers mapped over CUDA IPC
        from paper_2306_15951_b200.dist import FusedWgradAllReduce
        far = FusedWgradAllReduce([b.g for b in bufs], [b.dW for b in bufs], device)
        for i, b in enumerate(bufs):
            b.ar_grp = far.group(i)
            n = b.L.cks_workspace_size(b.g, b.dt, b.L.CKS_OP_WGRAD_AR)
            b.ws["wgrad_ar"] = torch.empty(max(n, 256), dtype=torch.uint8, device=device)
            b.launches["wgrad_ar"] = b.L.cks_launch_count(b.g, b.dt, b.L.CKS_OP_WGRAD_AR)
    ops_seq = []
    for i, b in enumerate(bufs):
        for op in ("fwd", "deconv", "wgrad"):
            if op in b.lay.ops:
                if op == "wgrad" and fused_ar:
                    ops_seq.append((i, "wgrad_ar"))
                    continue
                if op == "deconv" and b.direct:  # Stage1-free KS-deconv (no split)
                    ops_seq.append((i, "deconv_w"))
                    continue
                if op == "deconv":
                    ops_seq.append((i, "split"))
                ops_seq.append((i, "deconv_only" if op == "deconv" else op))
    OPF = {"fwd": "fwd", "deconv_only": "deconv", "deconv_w": "deconv", "wgrad": "wgrad", "wgrad_ar": "wgrad",
           "split": "split"}
    LKEY = {"fwd": "fwd", "deconv_only": "deconv", "deconv_w": "deconv_w", "wgrad": "wgrad", "wgrad_ar": "wgrad_ar",
            "split": "split"}
    flops_step = sum(bufs[i].flops for i, op in ops_seq if op != "split")
    launches_step = sum(bufs[i].launches[LKEY[op]] for i, op in ops_seq)
    kern = {(i, op): op_kernel(bufs[i], op) for i, op in ops_seq}
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device)  # 256 MB > 126 MB L2
    peaks = load_peaks()
    # dense TF32 = 1/2 BF16 (the guide's nominal ratio).  Burst peak for ops timed alone (per-op
    # protocol), sustained peak for the family timed inside the repeated step schedule (roofline)
    tc_peak = peaks["bf16"] if dtype == "bf16" else peaks["bf16"] / 2
    tc_peak_sus = peaks["bf16_sustained"] if dtype == "bf16" else peaks["bf16_sustained"] / 2

    stream = torch.cuda.Stream(device)
    with torch.cuda.stream(stream):
        for i, op in ops_seq:  # eager warm-up (sets smem attributes, checks errors)
            bufs[i].run(op, stream.cuda_stream)
    torch.cuda.synchronize()

    # ---- (2) the step as a training-step schedule (one CUDA graph): forward
    # chain on the main stream with the weight-only KS Stage1 splits on a side
    # stream; then the backward chain in reverse layer order (KS-deconv on the
    # main stream) with each layer's Sk-dilated wgrad on one of two alternating
    # side streams, released when the layer above finished its deconv.
    s1, s3 = torch.cuda.Stream(device), torch.cuda.Stream(device)
    nws = max(1, int(os.environ.get("CKS_BENCH_WSTREAMS", "2")))  # measured: 2 best (C2 0.624 -> 0.597 ms)
    wst = [torch.cuda.Stream(device) for _ in range(nws)]
    # data-parallel: the flat dW is all-reduced in buckets of layers, each
    # launched (on s3, NCCL) as soon as the bucket's wgrads are done, so the
    # communication overlaps the rest of the backward chain
    order = list(reversed(range(len(bufs))))  # backward order
    cuts = []
    nbuck = int(os.environ.get("CKS_BENCH_BUCKETS", "3"))
    if use_dist and nbuck > 1:
        tot, acc = sum(sizes), 0
        for k, i in enumerate(order):
            acc += sizes[i]
            if acc >= tot / nbuck * (len(cuts) + 1) - 1 and k < len(order) - 1:
                cuts.append(k)
    cuts.append(len(order) - 1)
    offs = [0]
    for sz in sizes:
        offs.append(offs[-1] + sz)
    buckets, k0 = [], 0
    for k1 in cuts:
        layers_k = order[k0:k1 + 1]
        buckets.append((offs[min(layers_k)], offs[max(layers_k) + 1]))
        k0 = k1 + 1
    last_of_bucket = {order[k1]: bi for bi, k1 in enumerate(cuts)}
    ar_in_graph = os.environ.get("CKS_BENCH_AR_GRAPH", "1") == "1" or fused_ar
    if use_dist and not fused_ar:
        s3.wait_stream(stream)
        with torch.cuda.stream(s3):  # communicator warm-up on the capture-side stream
            dist.all_reduce(flat)
        stream.wait_stream(s3)
        torch.cuda.synchronize()

    def capture(ar_graph, timed):
        """timed: an event on the launching stream before and after every op
        (the in-schedule kernel durations for the roofline)."""
        tev = {}
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            main = torch.cuda.current_stream()
            if timed:
                t0 = torch.cuda.Event(enable_timing=True, external=True)
                t0.record(main)
                tev["t0"] = t0

            def run(i, op, s):
                if timed:
                    a, z = (torch.cuda.Event(enable_timing=True, external=True) for _ in range(2))
                    a.record(s)
                    bufs[i].run(op, s.cuda_stream)
                    z.record(s)
                    tev[(i, op)] = (a, z)
                else:
                    bufs[i].run(op, s.cuda_stream)

            fork = torch.cuda.Event()
            fork.record(main)
            s1.wait_event(fork)
            for w in wst:
                w.wait_event(fork)
            with torch.cuda.stream(s1):
                for i, b in enumerate(bufs):
                    if "deconv" in b.lay.ops and not b.direct:
                        run(i, "split", s1)
                split_done = torch.cuda.Event()
                split_done.record(s1)
            for i, b in enumerate(bufs):
                if "fwd" in b.lay.ops:
                    run(i, "fwd", main)
            main.wait_event(split_done)
            for k, i in enumerate(order):
                b = bufs[i]
                ev = torch.cuda.Event()
                ev.record(main)
                ws_k = wst[k % nws]
                if "wgrad" in b.lay.ops:
                    ws_k.wait_event(ev)
                    with torch.cuda.stream(ws_k):
                        run(i, "wgrad_ar" if fused_ar else "wgrad", ws_k)
                if use_dist and not fused_ar and ar_graph and i in last_of_bucket:
                    for w in wst:  # this bucket's dW is complete: NCCL all_reduce on s3
                        done = torch.cuda.Event()
                        done.record(w)
                        s3.wait_event(done)
                    lo, hi = buckets[last_of_bucket[i]]
                    with torch.cuda.stream(s3):
                        dist.all_reduce(flat[lo:hi])
                if "deconv" in b.lay.ops:
                    run(i, "deconv_w" if b.direct else "deconv_only", main)
            for w in wst + ([s3] if use_dist and not fused_ar and ar_graph else []):
                join = torch.cuda.Event()
                join.record(w)
                main.wait_event(join)
            if timed:
                t1 = torch.cuda.Event(enable_timing=True, external=True)
                t1.record(main)
                tev["t1"] = t1
        return g, tev

    try:
        graph2, _ = capture(ar_in_graph, False)
    except Exception as exc:  # NCCL capture unavailable: reduce after the graph instead
        if not (use_dist and ar_in_graph):
            raise
        print(f"[bench] NCCL graph capture failed ({exc}); all_reduce after the step graph", file=sys.stderr)
        torch.cuda.synchronize()
        ar_in_graph = False
        graph2, _ = capture(False, False)

    def replay(g):
        g.replay()
        if use_dist and not fused_ar and not ar_in_graph:  # fallback: one all_reduce after the step
            dist.all_reduce(flat)

    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    noev = []
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            flush.fill_(2.0)
            replay(graph2)
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clk:
            for k in range(args.steps):
                flush.fill_(float(k))
                t_start.record(stream)
                replay(graph2)
                t_end.record(stream)
                stream.synchronize()
                noev.append(t_start.elapsed_time(t_end))
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    total_ms = sum(noev)
    if use_dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    value = flops_step * n_gpus / (ms_per_step / 1e3) / 1e12
    del graph2

    # ---- (1) per-op protocol (each op timed on its own; run after the
    # headline, so the timed step comes first): the ops serialized in one graph
    # with event nodes between them, L2 flushed
    evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(ops_seq) + 1)]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        sp = torch.cuda.current_stream().cuda_stream
        for k, (i, op) in enumerate(ops_seq):
            evs[k].record()
            bufs[i].run(op, sp)
        evs[-1].record()
    nser = max(3, min(args.steps, 20))
    per_op_ms = [0.0] * len(ops_seq)
    with torch.cuda.stream(stream):
        for it in range(nser + 2):
            flush.fill_(float(it))
            graph.replay()
            stream.synchronize()
            if it >= 2:
                for k in range(len(ops_seq)):
                    per_op_ms[k] += evs[k].elapsed_time(evs[k + 1]) / nser
    del graph

    # ---- (3) the same schedule with an event before and after every op on
    # its launching stream: in-step kernel durations (roofline), per kernel
    # family the union of its launches' intervals, so it fits in the step
    graph3, tev = capture(ar_in_graph, True)
    nt = max(3, min(args.steps, 20))
    fam_iv = {}
    fam_busy = {}
    step3 = 0.0
    with torch.cuda.stream(stream):
        for it in range(nt + 2):
            flush.fill_(float(it))
            replay(graph3)
            stream.synchronize()
            if it < 2:
                continue
            t0 = tev["t0"]
            step3 += t0.elapsed_time(tev["t1"]) / nt
            iv = {}
            for key, ev in tev.items():
                if key in ("t0", "t1"):
                    continue
                a, z = ev
                iv.setdefault(kern[key], []).append((t0.elapsed_time(a), t0.elapsed_time(z)))
                fam_iv.setdefault(kern[key], {}).setdefault(key, 0.0)
                fam_iv[kern[key]][key] += (t0.elapsed_time(z) - t0.elapsed_time(a)) / nt
            for kname, v in iv.items():
                fam_busy[kname] = fam_busy.get(kname, 0.0) + union_ms(v) / nt
    del graph3
    torch.cuda.synchronize()

    # ---- roofline of the dominant kernel family (largest in-step busy time)
    kname = max(fam_busy, key=fam_busy.get)
    keys = [k for k in fam_iv[kname]]
    kfl = sum(bufs[i].flops for i, op in keys if op != "split")
    kby = sum(bufs[i].algo_bytes[OPF[op]] for i, op in keys)
    busy = fam_busy[kname]
    t_tc = kfl / (tc_peak_sus * 1e12)
    t_hbm = kby / (peaks["hbm"] * 1e9)
    bound = "tensor" if t_tc >= t_hbm else "hbm"
    ach_tc = kfl / (busy / 1e3) / 1e12
    ach_hbm = kby / (busy / 1e3) / 1e9
    tc_frac, hbm_frac = ach_tc / tc_peak_sus, ach_hbm / peaks["hbm"]
    roofline = {"bound": bound, "kernel": kname,
                "achieved": round(ach_tc if bound == "tensor" else ach_hbm, 2),
                "peak": round(tc_peak_sus if bound == "tensor" else peaks["hbm"], 1),
                "unit": "TFLOP/s" if bound == "tensor" else "GB/s",
                "frac": round(tc_frac if bound == "tensor" else hbm_frac, 4),
                "traffic": load_traffic(kname, args.config, dtype),
                "tc_frac": round(tc_frac, 4), "hbm_frac": round(hbm_frac, 4),
                "tc_frac_vs_burst_peak": round(ach_tc / tc_peak, 4),
                "launches_per_step": len(keys),
                "algorithmic_flops_per_launch": round(kfl / len(keys)),
                "algorithmic_bytes_per_launch": round(kby / len(keys)),
                "busy_ms_per_step": round(busy, 5), "evented_step_ms": round(step3, 5),
                "share_of_step": round(busy / step3, 4),
                "peak_src": (f"{peaks['src']} bf16 SUSTAINED (MEASURED_PEAKS.json bf16_tflops_sustained: the family "
                             f"is timed inside the repeated step)" if dtype == "bf16" else
                             f"{peaks['src']} bf16 SUSTAINED x 1/2 (nominal TF32:BF16; the family is timed inside "
                             f"the repeated step)") + f"; HBM {peaks['hbm']} GB/s",
                "timing": "CUDA events on each op's launching stream inside the step schedule graph (a copy of the "
                          "headline graph with event nodes); busy = union of the family's launch intervals per step",
                "traffic_src": "profiles/ncu_traffic.json: ncu dram__bytes_read+write per launch (cold-cache replay)"}
    fams = {k: {"busy_ms": round(v, 5), "share": round(v / step3, 4)} for k, v in sorted(fam_busy.items(),
                                                                                         key=lambda kv: -kv[1])}

    # ---- per-op families and the per-layer table (per-op protocol)
    fam = {"fwd": [0.0, 0], "split": [0.0, 0], "deconv": [0.0, 0], "wgrad": [0.0, 0]}
    rows = []
    for k, (i, op) in enumerate(ops_seq):
        f = OPF[op]
        b = bufs[i]
        ms = per_op_ms[k]
        fam[f][0] += ms
        fl = b.flops if f != "split" else 0
        fam[f][1] += fl
        by = b.algo_bytes[f]
        tc = fl / (ms / 1e3) / 1e12 / tc_peak
        hb = by / (ms / 1e3) / 1e9 / peaks["hbm"]
        lb = "tensor" if fl / (tc_peak * 1e12) >= by / (peaks["hbm"] * 1e9) else "hbm"
        rows.append({"layer": b.lay.name, "op": f, "kernel": kern[(i, op)], "us": round(ms * 1e3, 2),
                     "tflops": round(fl / (ms / 1e3) / 1e12, 1) if fl else None, "bound": lb,
                     "tc_frac": round(tc, 3), "hbm_frac": round(hb, 3),
                     "frac": round(tc if lb == "tensor" else hb, 3)})
    per_op = {op: {"ms": round(v[0], 5), "tflops": round(v[1] / (v[0] / 1e3) / 1e12, 2) if v[1] else None}
              for op, v in fam.items() if v[0]}
    out = {"desc": desc, "layers": layers, "bufs": bufs, "ops_seq": ops_seq, "flops_step": flops_step, "flush": flush,
           "value": value, "ms_per_step": ms_per_step, "per_op": per_op, "roofline": roofline, "families": fams,
           "per_layer": rows, "gpu_launches": launches_step * args.steps, "clocks": clk.summary(), "nws": nws,
           "buckets": len(buckets), "ar_in_graph": ar_in_graph, "serialized_ms": sum(per_op_ms),
           "fam_ms": {"fwd": fam["fwd"][0], "deconv": fam["deconv"][0] + fam["split"][0], "wgrad": fam["wgrad"][0]}}
    if args.layers and rank == 0:
        for r in rows:
            print(f"  {r['layer']:22s} {r['op']:7s} {r['kernel']:17s} {r['us']:9.2f} us  "
                  f"{(r['tflops'] or 0):8.1f} TFLOP/s  {r['bound']:6s} tc {r['tc_frac']:.3f} hbm {r['hbm_frac']:.3f}",
                  file=sys.stderr)
    return out


def run_gpu(args):
    import torch
    import torch.distributed as dist
    from paper_2306_15951_b200 import build

    ws_, rank, local = dist_env()
    if args.gpus != ws_:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE {ws_}: running {ws_} rank(s)", file=sys.stderr)
    n_gpus = ws_
    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    # the data-parallel path (NCCL dW all_reduce) runs for N > 1; CKS_BENCH_DIST=1
    # exercises it with a single rank under torchrun (testing on one GPU)
    use_dist = n_gpus > 1 or (os.environ.get("CKS_BENCH_DIST") == "1" and "RANK" in os.environ)
    if use_dist:
        # keep stdout to the one JSON line: library output written to fd 1 (NCCL's
        # version banner under NCCL_DEBUG=VERSION) is sent to stderr; the line goes
        # to the original stdout
        global _JSON_OUT
        _JSON_OUT = os.fdopen(os.dup(1), "w")
        sys.stdout.flush()
        os.dup2(2, 1)
        dist.init_process_group("nccl", device_id=device)
    if local == 0:
        build.build()
    if use_dist:
        dist.barrier()
    build.build()  # loads the library (up to date now)
    m = measure(args, torch, dist, device, rank, local, n_gpus, use_dist, args.dtype)
    desc, layers, bufs = m["desc"], m["layers"], m["bufs"]
    line = {
        "metric": METRIC, "value": round(m["value"], 3), "unit": "TFLOP/s", "n_gpus": n_gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(m["ms_per_step"], 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype,
        "data": "synthetic (seeded U[-1,1) X/dY, kaiming-uniform W)" +
                ("; fp32 inputs multiplied as TF32, fp32 accumulate and outputs" if args.dtype == "tf32" else
                 "; bf16 inputs, fp32 accumulate and outputs"),
        "config": {"workload": desc, "layers": len(layers), "per_gpu_batch": layers[0].N,
                   "global_batch": layers[0].N * n_gpus, "ops_per_step": len(m["ops_seq"]),
                   "zero_free_gflop_per_gpu_step": round(m["flops_step"] / 1e9, 3),
                   "l2": "flushed (256 MB write) before every timed step, outside the timed events",
                   "parallelism": f"dp{n_gpus}",
                   "schedule": "fwd chain || KS Stage1 splits; reverse deconv chain || per-layer wgrad on %d "
                               "alternating streams (CUDA graph)" % m["nws"]
                               + (("; dW summed across ranks inside each layer's Sk-dilated G_Z reduce "
                                   "(KB-REDUCE-AR, NVLink P2P, CUDA IPC)") if use_dist and args.allreduce == "fused" else
                                  ("; dW all_reduce in %d buckets overlapping the backward (NCCL in the graph)"
                                   % m["buckets"] if m["ar_in_graph"] else "; dW all_reduce after the step graph")
                                  if use_dist else ""),
                   "serialized_step_ms_per_op_protocol": round(m["serialized_ms"], 5)},
        "per_op": m["per_op"], "roofline": m["roofline"], "kernel_families_in_step": m["families"],
        "gpu_launches": m["gpu_launches"], "clocks": m["clocks"],
    }
    # ---- the zero-inserted / zero-padded formulation on the same kernels
    if not args.no_zins and n_gpus == 1:
        line["zins"] = run_zins(torch, bufs, max(3, min(args.steps, 20)), device, m["flush"], m["fam_ms"], args.layers)
    # ---- Stage1-free vs Stage1 KS-deconv on every eligible layer
    if not args.no_zins and n_gpus == 1:
        line["ks_stage1_free"] = run_ks_compare(torch, bufs, max(3, min(args.steps, 20)), device, m["flush"],
                                                args.layers)
    # ---- e2e through the public API with host buffers
    if not args.no_e2e:
        line["e2e"] = run_e2e(torch, dist, bufs, m["ops_seq"], m["flops_step"], n_gpus, max(2, min(args.steps, 10)),
                              device)
    line["per_layer"] = m["per_layer"]
    del m, bufs
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    # ---- the other input precision beside the headline (same workload)
    if args.companion and args.companion != args.dtype:
        c = measure(args, torch, dist, device, rank, local, n_gpus, use_dist, args.companion)
        line[args.companion] = {"value": round(c["value"], 3), "ms_per_step": round(c["ms_per_step"], 5),
                                "per_op": c["per_op"], "roofline": c["roofline"],
                                "kernel_families_in_step": c["families"], "gpu_launches": c["gpu_launches"],
                                "clocks": c["clocks"],
                                "per_layer": [{k: r[k] for k in ("layer", "op", "us", "tflops", "frac")}
                                              for r in c["per_layer"]]}
        if not args.no_zins and n_gpus == 1:
            line[args.companion]["ks_stage1_free"] = run_ks_compare(torch, c["bufs"], max(3, min(args.steps, 20)),
                                                                    device, c["flush"], args.layers)
        del c
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
    # ---- CPU oracle baseline (rank 0, N=1 only)
    if rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        el, f, passes = oracle_sample(layers, args.config, 1, budget_s=args.cpu_budget)
        line["cpu_baseline"] = {"value": f / el / 1e12, "unit": "TFLOP/s", "cores": blas_threads(), "kind": "oracle",
                                "sample": f"{passes} passes over all {len(layers)} layers x ops at N=1 image "
                                          f"({el:.1f} s; oracle cost is linear in N)"}
    if rank == 0:
        print(json.dumps(line), file=_JSON_OUT or sys.stdout, flush=True)
    if use_dist:
        dist.destroy_process_group()
    return 0


def run_ks_compare(torch, bufs, steps, device, flush, per_layer):
    """Stage1-free KS-deconv (the GEMM reads W directly)
    against KB-SPLIT + KB-KS (Stage1 every step, then Stage2&3), per eligible
    layer: one serialized graph with event nodes, L2 flushed per replay."""
    seq = []
    for i, b in enumerate(bufs):
        if b.direct_ok:
            seq += [(i, "split"), (i, "deconv_only"), (i, "deconv_free")]
    if not seq:
        return None
    stream = torch.cuda.Stream(device)
    with torch.cuda.stream(stream):
        for i, op in seq:
            bufs[i].run(op, stream.cuda_stream)
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(seq) + 1)]
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        sp = torch.cuda.current_stream().cuda_stream
        for k, (i, op) in enumerate(seq):
            evs[k].record()
            bufs[i].run(op, sp)
        evs[-1].record()
    acc = [0.0] * len(seq)
    with torch.cuda.stream(stream):
        for it in range(steps + 2):
            flush.fill_(float(it))
            graph.replay()
            stream.synchronize()
            if it >= 2:
                for k in range(len(seq)):
                    acc[k] += evs[k].elapsed_time(evs[k + 1]) / steps
    rows, tot_s1, tot_free = [], 0.0, 0.0
    for k in range(0, len(seq), 3):
        i = seq[k][0]
        s1 = acc[k] + acc[k + 1]
        fr = acc[k + 2]
        tot_s1 += s1
        tot_free += fr
        rows.append({"layer": bufs[i].lay.name, "stage1_plus_ks_us": round(s1 * 1e3, 2),
                     "split_us": round(acc[k] * 1e3, 2), "stage1_free_us": round(fr * 1e3, 2),
                     "policy": "stage1_free" if bufs[i].direct else "stage1"})
        if per_layer:
            print(f"  ks {bufs[i].lay.name:22s} split+ks {s1 * 1e3:8.2f} us  stage1-free {fr * 1e3:8.2f} us"
                  f"  ({rows[-1]['policy']})", file=sys.stderr)
    return {"what": "KS-deconv with Stage1 (KB-SPLIT + KB-KS) vs Stage1-free (W read directly by the GEMM), "
                    "serialized graph, L2 flushed", "ms_stage1_plus_ks": round(tot_s1, 5),
            "ms_stage1_free": round(tot_free, 5), "layers": rows, "steps": steps}


def run_zins(torch, bufs, steps, device, flush, cks_ms, per_layer):
    """Time cks_zins_* (KB-ZINS: the operands materialised with every padded and
    inserted zero, then the same tensor-core kernels with nothing left to
    trim) exactly like the serialized C-K-S ops: one CUDA graph with event
    nodes between the ops, L2 flushed before every replay.  Reports the time
    ratio next to the nominal (Table III) / zero-free FLOP ratio."""
    from paper_2306_15951_b200 import _lib as L
    seq = []
    for i, b in enumerate(bufs):
        for op in ("fwd", "deconv", "wgrad"):
            if op in b.lay.ops:
                seq.append((i, op))
    code = {"fwd": L.CKS_OP_FWD, "deconv": L.CKS_OP_DECONV, "wgrad": L.CKS_OP_WGRAD}
    need = max(L.cks_zins_workspace_size(bufs[i].g, bufs[i].dt, code[op]) for i, op in seq)
    ws = torch.empty(max(need, 256), dtype=torch.uint8, device=device)
    dw = torch.empty(max(b.dW.numel() for b in bufs), dtype=torch.float32, device=device)

    def run(i, op, sp):
        b = bufs[i]
        if op == "fwd":
            L.cks_zins_conv2d_fwd(b.g, b.dt, b.X.data_ptr(), b.W.data_ptr(), b.Y.data_ptr(), ws.data_ptr(),
                                  ws.numel(), sp)
        elif op == "deconv":
            L.cks_zins_deconv2d(b.g, b.dt, b.G.data_ptr(), b.W.data_ptr(), b.dX.data_ptr(), ws.data_ptr(),
                                ws.numel(), sp)
        else:
            L.cks_zins_wgrad(b.g, b.dt, b.X.data_ptr(), b.G.data_ptr(), dw.data_ptr(), ws.data_ptr(),
                             ws.numel(), sp)

    stream = torch.cuda.Stream(device)
    evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(seq) + 1)]
    with torch.cuda.stream(stream):
        for i, op in seq:
            run(i, op, stream.cuda_stream)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        sp = torch.cuda.current_stream().cuda_stream
        for k, (i, op) in enumerate(seq):
            evs[k].record()
            run(i, op, sp)
        evs[-1].record()
    acc = [0.0] * len(seq)
    with torch.cuda.stream(stream):
        for it in range(steps + 2):
            flush.fill_(float(it))
            graph.replay()
            stream.synchronize()
            if it >= 2:
                for k in range(len(seq)):
                    acc[k] += evs[k].elapsed_time(evs[k + 1]) / steps
    ms = {"fwd": 0.0, "deconv": 0.0, "wgrad": 0.0}
    nominal = {"fwd": 0, "deconv": 0, "wgrad": 0}
    zf = {"fwd": 0, "deconv": 0, "wgrad": 0}
    tkey = {"fwd": "T_conv", "deconv": "T_deconv", "wgrad": "T_dilated"}
    for k, (i, op) in enumerate(seq):
        ms[op] += acc[k]
        cnt = L.cks_op_counts(bufs[i].g)
        nominal[op] += cnt[tkey[op]]
        zf[op] += bufs[i].flops
        if per_layer:
            print(f"  zins {bufs[i].lay.name:22s} {op:7s} {acc[k] * 1e3:9.2f} us", file=sys.stderr)
    return {"what": "cks_zins_*: zero-padded (fwd) / zero-inserted (deconv, wgrad) operands materialised in HBM "
                    "(P:114, Eqs (1)-(3) as written) + the same tcgen05 kernels; serialized graph, L2 flushed",
            "ms": {k: round(v, 5) for k, v in ms.items() if v},
            "cks_ms": {k: round(v, 5) for k, v in cks_ms.items() if v},
            "time_ratio_zins_over_cks": {k: round(ms[k] / cks_ms[k], 3) for k in ms if ms[k] and cks_ms.get(k)},
            "nominal_over_zero_free_flops": {k: round(nominal[k] / zf[k], 3) for k in ms if zf[k]},
            "steps": steps}


def run_e2e(torch, dist, bufs, ops_seq, flops_step, n_gpus, steps, device):
    """The same step through the public torch API (paper_2306_15951_b200.ops):
    pinned host inputs -> device, the three operators, results -> host, every
    byte of every layer every step (copies overlapped with compute)."""
    from paper_2306_15951_b200 import ops as K
    host_in, host_out = [], []
    for b in bufs:
        host_in.append({k: getattr(b, k).cpu().pin_memory() for k in ("X", "W", "G")})
        host_out.append({k: torch.empty(getattr(b, k).shape, dtype=torch.float32).pin_memory()
                         for k in ("Y", "dX", "dW")})
    h2d = sum(t.numel() * t.element_size() for d in host_in for t in d.values())
    d2h = 0
    for b, d in zip(bufs, host_out):
        for k in ("Y", "dX", "dW"):
            opname = {"Y": "fwd", "dX": "deconv", "dW": "wgrad"}[k]
            if opname in b.lay.ops:
                d2h += d[k].numel() * 4
    # three streams: H2D copies, the C-K-S ops, D2H copies -- PCIe traffic in
    # both directions overlaps the compute of other layers (copy engines run
    # concurrently with the SMs); per-layer events carry the dependencies, and
    # the device buffers of a layer are reused across steps behind its events
    s_in, s_comp, s_out = (torch.cuda.Stream(device) for _ in range(3))
    dev_in = [{k: torch.empty_like(getattr(b, k)) for k in ("X", "W", "G")} for b in bufs]
    dev_out = []
    for b in bufs:
        lay = b.lay
        OH, OW = lay.out_hw()
        f32 = dict(dtype=torch.float32, device=device)
        dev_out.append({"Y": torch.empty((lay.N, OH, OW, lay.OC), **f32),
                        "dX": torch.empty((lay.N, lay.H, lay.W, lay.C), **f32),
                        "dW": torch.empty((lay.OC, lay.FH, lay.FW, lay.C), **f32)})
    nl = len(bufs)
    ev_in = [torch.cuda.Event() for _ in range(nl)]
    ev_comp = [torch.cuda.Event() for _ in range(nl)]
    ev_out = [torch.cuda.Event() for _ in range(nl)]
    started = [False] * nl

    def one():
        for i, (b, hi, ho) in enumerate(zip(bufs, host_in, host_out)):
            lay = b.lay
            di, do = dev_in[i], dev_out[i]
            with torch.cuda.stream(s_in):
                if started[i]:
                    s_in.wait_event(ev_comp[i])  # the previous step's ops of this layer read these buffers
                for k in ("X", "W", "G"):
                    di[k].copy_(hi[k], non_blocking=True)
                ev_in[i].record(s_in)
            with torch.cuda.stream(s_comp):
                s_comp.wait_event(ev_in[i])
                if started[i]:
                    s_comp.wait_event(ev_out[i])  # the previous step's results were copied out
                st, pd = (lay.sh, lay.sw), (lay.ph, lay.pw)
                X, W, G = di["X"], di["W"], di["G"]
                if "fwd" in lay.ops:
                    K.conv2d_fwd(X, W, st, pd, out=do["Y"], stream=s_comp)
                if "deconv" in lay.ops:
                    K.deconv2d(G, W, (lay.H, lay.W), st, pd, out=do["dX"], stream=s_comp)
                if "wgrad" in lay.ops:
                    K.dilated_wgrad(X, G, (lay.FH, lay.FW), st, pd, out=do["dW"], stream=s_comp)
                    if n_gpus > 1:
                        dist.all_reduce(do["dW"])
                ev_comp[i].record(s_comp)
            with torch.cuda.stream(s_out):
                s_out.wait_event(ev_comp[i])
                for k, opname in (("Y", "fwd"), ("dX", "deconv"), ("dW", "wgrad")):
                    if opname in lay.ops:
                        ho[k].copy_(do[k], non_blocking=True)
                ev_out[i].record(s_out)
            started[i] = True

    one()
    torch.cuda.synchronize()
    if n_gpus > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s_in)
    s_comp.wait_event(e0)
    s_out.wait_event(e0)
    for _ in range(steps):
        one()
    s_out.wait_stream(s_in)
    s_out.wait_stream(s_comp)
    e1.record(s_out)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if n_gpus > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"value": round(flops_step * n_gpus / (ms / 1e3) / 1e12, 3), "unit": "TFLOP/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": round(ms, 4), "steps": steps}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    if args.companion == "none":
        args.companion = None
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
