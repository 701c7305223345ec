"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds NONE of the method's arithmetic: only random numbers with the
shapes, dtypes and distributions of the paper's workloads (DESIGN.md "Input
recipe").  numpy's PCG64 generator; every array is a function of its seed.
"""
from __future__ import annotations

import numpy as np

# Llama-3-8B linear layer shapes (F_out, F_in) per block, in model order:
# q, k, v, o, gate, up, down (public config: hidden 4096, 8 KV heads x 128,
# intermediate 14336).  The paper's E2E model.
LLAMA3_8B_LAYERS = [
    ("q_proj", 4096, 4096), ("k_proj", 1024, 4096), ("v_proj", 1024, 4096),
    ("o_proj", 4096, 4096), ("gate_proj", 14336, 4096), ("up_proj", 14336, 4096),
    ("down_proj", 4096, 14336),
]
LLAMA3_8B_BLOCKS = 32
LLAMA3_8B_SHAPES = [(4096, 4096), (14336, 4096), (4096, 14336)]   # configs[1]


def rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


def weight(F_out: int, F_in: int, seed: int = 0, std: float = 0.02) -> np.ndarray:
    """fp16 [F_out][F_in] ~ N(0, std^2) (HF Llama initializer_range 0.02)."""
    return rng(seed).normal(0.0, std, size=(F_out, F_in)).astype(np.float16)


def activation(B: int, F_in: int, seed: int = 1, std: float = 1.0) -> np.ndarray:
    """fp16 [B][F_in] ~ N(0, std^2)."""
    return rng(seed).normal(0.0, std, size=(B, F_in)).astype(np.float16)


def structured_weight(F_out: int, F_in: int, d: int, n_distinct: int, group: int = 1,
                      seed: int = 0) -> np.ndarray:
    """fp16 W whose every codebook (``group`` consecutive width-d subspaces)
    draws its sub-vectors from at most ``n_distinct`` distinct fp16 vectors
    (the saturation case of SPEC S:85/S:133)."""
    g = rng(seed)
    N_ss = F_in // d
    N_cb = N_ss // group
    W = np.empty((F_out, F_in), np.float16)
    for cb in range(N_cb):
        alphabet = g.normal(0.0, 0.02, size=(n_distinct, d)).astype(np.float16)
        for s in range(group):
            ss = cb * group + s
            pick = g.integers(0, n_distinct, size=F_out)
            W[:, ss * d:(ss + 1) * d] = alphabet[pick]
    return W


def random_layer(F_out: int, F_in: int, d: int, C: int, group: int = 1, seed: int = 0,
                 std: float | None = None):
    """Logical PQ layer with uniform-random indices (worst-case locality) and
    fp16 N(0, std^2) codebooks; std defaults to 1/sqrt(F_in) so that a chain of
    layers keeps activations O(1).  Returns (codebooks [N_cb][C][d] fp16,
    indices [N_ss][F_out] uint8, uint16 when C > 256)."""
    g = rng(seed)
    N_ss = F_in // d
    N_cb = N_ss // group
    if std is None:
        std = 1.0 / np.sqrt(F_in)
    cb = g.normal(0.0, std, size=(N_cb, C, d)).astype(np.float16)
    idx = g.integers(0, C, size=(N_ss, F_out), dtype=np.uint8 if C <= 256 else np.uint16)
    return cb, idx


def torch_random_layer(F_out: int, F_in: int, d: int, C: int, group: int = 1, seed: int = 0,
                       device: str = "cuda", std: float | None = None):
    """Same recipe as :func:`random_layer` drawn with torch's generator on
    ``device`` (fast for the full-size bench model; different stream of
    random numbers than the numpy version)."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    N_ss = F_in // d
    N_cb = N_ss // group
    if std is None:
        std = 1.0 / float(np.sqrt(F_in))
    cb = (torch.randn((N_cb, C, d), generator=g, device=device) * std).to(torch.float16)
    idx = torch.randint(0, C, (N_ss, F_out), generator=g, device=device, dtype=torch.int32)
    idx = idx.to(torch.uint8) if C <= 256 else idx.to(torch.int16)   # int16 holds 0..1023 (uint16 bits)
    return cb, idx


def torch_activation(B: int, F_in: int, seed: int = 1, device: str = "cuda", std: float = 1.0):
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return (torch.randn((B, F_in), generator=g, device=device) * std).to(torch.float16)
