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
