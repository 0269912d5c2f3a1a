"""Multi-process (world_size 2, gloo, CPU) checks of the batch-sharded path.

The per-rank compute here is the fp64 oracle standing in for the CUDA kernels
(no GPU in this container); what is under test is the host logic of
paper_2306_15951_b200.dist: the contiguous batch partition and the bucketed
FlatGrads SUM all_reduce that completes the Sk-dilated map-reduce
across ranks.  The rank-sharded forward/deconv outputs concatenate to the
full-batch result and the all-reduced partial dW equals the full-batch dW.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as O
from paper_2306_15951_b200.dist import FlatGrads, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


LAYERS = [dict(N=5, C=3, H=7, W=6, OC=4, FH=3, FW=3, sh=2, sw=1, ph=1, pw=1),
          dict(N=5, C=2, H=5, W=5, OC=3, FH=1, FW=2, sh=1, sw=2, ph=0, pw=1)]


def _inputs(i, g):
    rng = np.random.default_rng(100 + i)
    X = rng.uniform(-1, 1, (g.N, g.H, g.W, g.C))
    W = rng.uniform(-1, 1, (g.OC, g.FH, g.FW, g.C))
    G = rng.uniform(-1, 1, (g.N, g.OH, g.OW, g.OC))
    return X, W, G


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        geoms = [O.geom(**l) for l in LAYERS]
        fg = FlatGrads([(g.OC, g.FH, g.FW, g.C) for g in geoms], "cpu")
        outs = []
        for i, g in enumerate(geoms):
            X, W, G = _inputs(i, g)
            a, b = shard_range(g.N, world, rank)
            s = (g.sh, g.sw, g.ph, g.pw)
            Y = O.conv_ref(X[a:b], W, *s)
            dX = O.deconv_ref(G[a:b], W, g.H, g.W, *s)
            dW = O.wgrad_ref(X[a:b], G[a:b], g.FH, g.FW, *s)
            fg.views[i].copy_(torch.from_numpy(dW).float())
            outs.append((a, b, Y, dX))
        fg.all_reduce()
        q.put((rank, outs, [v.numpy().copy() for v in fg.views]))
    finally:
        dist.destroy_process_group()


def test_shard_range_partition():
    for n in range(0, 20):
        for world in range(1, 9):
            rs = [shard_range(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


def test_world2_gloo_sharded_step():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, outs, dws = q.get(timeout=120)
        res[rank] = (outs, dws)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    geoms = [O.geom(**l) for l in LAYERS]
    for i, g in enumerate(geoms):
        X, W, G = _inputs(i, g)
        s = (g.sh, g.sw, g.ph, g.pw)
        Yf = O.conv_ref(X, W, *s)
        dXf = O.deconv_ref(G, W, g.H, g.W, *s)
        dWf = O.wgrad_ref(X, G, g.FH, g.FW, *s)
        Y = np.concatenate([res[r][0][i][2] for r in range(world)])
        dX = np.concatenate([res[r][0][i][3] for r in range(world)])
        np.testing.assert_allclose(Y, Yf, atol=1e-12)
        np.testing.assert_allclose(dX, dXf, atol=1e-12)
        for r in range(world):  # every rank holds the complete dW after the all_reduce
            np.testing.assert_allclose(res[r][1][i], dWf, rtol=1e-5, atol=1e-5)
