"""Seeded synthetic inputs and workload shapes shared by the oracle tests, the
GPU parity tests, ``bench.py`` and ``__graft_entry__.smoke()``.

This module holds NONE of the method's arithmetic: it only draws random
numbers, rounds them to the storage precision the GPU path consumes, and lists
the layer shapes of the workloads.  Both sides of
every parity check (``oracle/`` and the CUDA path) take their inputs from here.

Value distributions follow the paper's workloads:
  * X  ~ U[-1, 1)   -- "pixel values ... linearly scaled between -1 and +1"
                       (§V.B.1)
  * W  ~ U[-1/sqrt(fan_in), 1/sqrt(fan_in)), fan_in = F_H*F_W*I_C
                    -- "initialized using kaiming-uniform"
  * dY ~ U[-1, 1)
Seeds: ``1000*config + 10*layer + {1: X, 2: W, 3: dY}``.
"""
from __future__ import annotations

import numpy as np

from .configs import CONFIGS, Layer, get_config  # noqa: F401

__all__ = ["CONFIGS", "Layer", "get_config", "round_bf16", "bf16_bits",
           "make_layer_inputs", "seeds_for"]


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round float32 values to the nearest bfloat16 (ties to even) and return
    them widened back to float32.  Storage-precision preparation only."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    lsb = (u >> np.uint32(16)) & np.uint32(1)
    r = (u + np.uint32(0x7FFF) + lsb) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """uint16 bit patterns of already-bf16-representable float32 values."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    if np.any(u & np.uint32(0xFFFF)):
        raise ValueError("values are not bf16-representable; call round_bf16 first")
    return (u >> np.uint32(16)).astype(np.uint16)


def seeds_for(config: int, layer: int) -> dict:
    base = 1000 * config + 10 * layer
    return {"X": base + 1, "W": base + 2, "dY": base + 3}


def make_layer_inputs(layer: "Layer", config: int = 0, layer_idx: int = 0,
                      dtype: str = "bf16", n: int | None = None,
                      which=("X", "W", "dY")) -> dict:
    """Draw X (N,I_H,I_W,I_C), W (O_C,F_H,F_W,I_C), dY (N,O_H,O_W,O_C) as
    float32 arrays.  For dtype 'bf16' the values are rounded to bf16 once, so
    the oracle and the GPU see identical numbers.  ``n`` overrides the batch
    (bounded samples for the CPU baseline)."""
    N = layer.N if n is None else n
    seeds = seeds_for(config, layer_idx)
    OH, OW = layer.out_hw()
    out = {}
    if "X" in which:
        rng = np.random.default_rng(seeds["X"])
        out["X"] = rng.uniform(-1.0, 1.0, size=(N, layer.H, layer.W, layer.C)).astype(np.float32)
    if "W" in which:
        rng = np.random.default_rng(seeds["W"])
        bound = 1.0 / np.sqrt(layer.FH * layer.FW * layer.C)
        out["W"] = rng.uniform(-bound, bound, size=(layer.OC, layer.FH, layer.FW, layer.C)).astype(np.float32)
    if "dY" in which:
        rng = np.random.default_rng(seeds["dY"])
        out["dY"] = rng.uniform(-1.0, 1.0, size=(N, OH, OW, layer.OC)).astype(np.float32)
    if dtype == "bf16":
        out = {k: round_bf16(v) for k, v in out.items()}
    elif dtype != "tf32":
        raise ValueError(f"unknown dtype {dtype!r}")
    return out
