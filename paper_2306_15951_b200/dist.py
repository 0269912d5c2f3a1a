"""Batch-sharded multi-GPU C-K-S conv-layer step (one process per GPU).

Partitioning: ConvV2 forward and KS-deconv are independent
per batch image, so each rank owns a contiguous slice of the batch and the
filters are replicated; the Sk-dilated weight gradient is the paper's
map-reduce over G_K = N*O_H*O_W with the batch shard as the OUTERMOST
segment -- every rank computes its partial dW with cks_dilated_wgrad, then ONE
fp32 SUM all_reduce (NCCL over NVLink/NVSwitch) completes it.  That is the
only cross-GPU exchange on the path.

The collective is bucketed: all layers' dW live in one flat fp32 buffer, so a
step issues a single all_reduce (or one per bucket when overlapped with the
remaining backward).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous batch slice [start, stop) of `rank`; sizes differ by <= 1."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


class FlatGrads:
    """One flat fp32 buffer holding the dW of several layers (views), so the
    cross-rank reduction is a single bucketed all_reduce."""

    def __init__(self, shapes, device):
        sizes = [int(torch.Size(s).numel()) for s in shapes]
        self.flat = torch.zeros(sum(sizes), dtype=torch.float32, device=device)
        self.views = []
        off = 0
        for s, n in zip(shapes, sizes):
            self.views.append(self.flat[off:off + n].view(*s))
            off += n

    def all_reduce(self, group=None, async_op=False):
        """SUM the partial dW of all ranks (no-op without a process group)."""
        if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
            return None
        return dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def sharded_layer_step(x_local, w, dy_local, stride, padding, grads_view, stream=None):
    """One conv-layer training step on this rank's batch shard with the CUDA
    path: Y_local = ConvV2(X_local, W); dX_local = KS-deconv(dY_local, W);
    partial dW (Sk-dilated) into `grads_view` -- the caller all-reduces the
    FlatGrads buffer once all layers are done."""
    from . import ops as K
    y = K.conv2d_fwd(x_local, w, stride, padding, stream=stream)
    dx = K.deconv2d(dy_local, w, tuple(x_local.shape[1:3]), stride, padding, stream=stream)
    K.dilated_wgrad(x_local, dy_local, tuple(w.shape[1:3]), stride, padding, out=grads_view, stream=stream)
    return y, dx


class FusedWgradAllReduce:
    """Per-layer Sk-dilated + cross-rank dW sum in one kernel over peer memory
    (cks_dilated_wgrad_allreduce, KB-REDUCE-AR): the
    G_Z segments and the ranks' batch shards are reduced together in fixed
    order, every rank receives the bit-identical dW, no NCCL call on the path.

    Buffers per layer (allocated here, one flat tensor each): the receive
    buffer (world x slice float4), two signal words, and three counter words
    (CTA arrivals + the device-side call sequence number: the calls may be
    captured in a CUDA graph and replayed).
    Peers' buffers are mapped with CUDA IPC (handles exchanged over the
    process group: gloo or NCCL), or, with ``virtual_world`` on ONE process,
    the "ranks" are this process's own buffer sets, run together by
    ``run_emulated`` (every rank's Sk-dilated, then ONE cooperative reduce
    launch over all ranks: kernels that wait on one another must never be
    separate launches on one GPU).
    """

    def __init__(self, geoms, dws, device, group=None, virtual_world=None, ctas=0):
        from . import _lib as L
        self.L = L
        self.geoms = list(geoms)
        self.device = device
        self.ctas = int(ctas)
        if virtual_world is not None:
            self.world, self.ranks = int(virtual_world), list(range(int(virtual_world)))
        else:
            self.world = dist.get_world_size(group) if dist.is_initialized() else 1
            self.ranks = [dist.get_rank(group) if dist.is_initialized() else 0]
        if not 1 <= self.world <= L.CKS_AR_MAX_RANKS:
            raise ValueError("world size out of range for the fused all-reduce")
        nl = len(self.geoms)
        self.recv_off, off = [], 0
        for g in self.geoms:
            self.recv_off.append(off)
            off += (L.cks_ar_recv_bytes(g, self.world) + 255) // 256 * 256
        self.recv_bytes = max(off, 256)
        # one buffer set per local rank (virtual ranks: several on this process)
        self.sets = []
        for r in self.ranks:
            self.sets.append({
                "recv": torch.empty(self.recv_bytes, dtype=torch.uint8, device=device),
                "flags": torch.zeros(2 * nl, dtype=torch.int32, device=device),
                "count": torch.zeros(4 * nl, dtype=torch.int32, device=device),
                "err": torch.zeros(1, dtype=torch.int32, device=device),
                "dws": dws[r] if virtual_world is not None else dws,
            })
        self._mapped = []
        if virtual_world is not None:
            peers = [(s["recv"].data_ptr(), [d.data_ptr() for d in s["dws"]], s["flags"].data_ptr())
                     for s in self.sets]
        else:
            s = self.sets[0]
            mine = (L.cks_ipc_export(s["recv"].data_ptr()), [L.cks_ipc_export(d.data_ptr()) for d in s["dws"]],
                    L.cks_ipc_export(s["flags"].data_ptr()))
            allh = [None] * self.world
            dist.all_gather_object(allh, mine, group=group)
            peers = []
            for t, (hr, hd, hf) in enumerate(allh):
                if t == self.ranks[0]:
                    peers.append((s["recv"].data_ptr(), [d.data_ptr() for d in s["dws"]], s["flags"].data_ptr()))
                    continue
                pr, pf = L.cks_ipc_import(hr), L.cks_ipc_import(hf)
                pd = [L.cks_ipc_import(h) for h in hd]
                self._mapped += [pr, pf] + pd
                peers.append((pr, pd, pf))
        self.peers = peers

    def group(self, layer, local=0):
        """cks_ar_group of `layer` for local buffer set `local`."""
        L = self.L
        s = self.sets[local]
        grp = L.cks_ar_group()
        grp.world, grp.rank, grp.ctas = self.world, self.ranks[local], self.ctas
        for t, (pr, pd, pf) in enumerate(self.peers):
            grp.recv[t] = pr + self.recv_off[layer]
            grp.out[t] = pd[layer]
            grp.flag[t] = pf + 8 * layer
        grp.count = s["count"].data_ptr() + 16 * layer
        grp.err = s["err"].data_ptr()
        return grp

    def run_emulated(self, layer, geoms, dtype, xs, dys, gz, wss, stream):
        """Virtual ranks: Sk-dilated of every rank's shard (geoms[r], xs[r], dys[r]: device pointers,
        wss[r]: workspace tensors) + the fused G_Z / cross-rank reduce in one cooperative launch."""
        grps = [self.group(layer, r) for r in range(self.world)]
        dw = [self.sets[r]["dws"][layer].data_ptr() for r in range(self.world)]
        self.L.cks_dilated_wgrad_allreduce_emulated(list(geoms), dtype, list(xs), list(dys), dw, gz,
                                                    [w.data_ptr() for w in wss], [w.numel() for w in wss], grps,
                                                    stream)

    def errors(self):
        return [int(s["err"].item()) for s in self.sets]

    def close(self):
        for p in self._mapped:
            self.L.cks_ipc_close(p)
        self._mapped = []
