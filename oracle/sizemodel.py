"""FASQ size model -- TEST INFRASTRUCTURE ONLY (closed forms, plain Python).

Eq. 4, Eq. 5, #W and the Alg. 2 split-K
planner formula, plus the storage actually used by this build
(uint8 indices, fp16 codebooks, readings R9/R10) and the fitted
"paper accounting" formula that reproduces the paper's
printed Size% values.
"""
from __future__ import annotations

import math
from dataclasses import dataclass


def eff_bits(d: int, C: int) -> float:
    """#W = ceil(log2 K_s) / SZ_ss, codebook excluded."""
    return math.ceil(math.log2(C)) / d if C > 1 else 0.0


def eq4_layer_bits(K_s: int, dim_ss: int, N_ss: int, dim_dp: int) -> int:
    """Eq. 4: 16*K_s*dim_ss + ceil(log2 K_s)*N_ss*dim_dp bits."""
    lg = math.ceil(math.log2(K_s)) if K_s > 1 else 0
    return 16 * K_s * dim_ss + lg * N_ss * dim_dp


def stored_bytes(F_out: int, F_in: int, d: int, C: int, group: int = 1) -> dict:
    """Bytes this build stores for one layer: uint8 index per (subspace,
    output row) and fp16 codebooks [N_cb][C][d] (reading R9/R10)."""
    N_ss = F_in // d
    N_cb = N_ss // group
    idx = N_ss * F_out
    cb = N_cb * C * d * 2
    return {"index_bytes": idx, "codebook_bytes": cb, "total_bytes": idx + cb}


def bits_per_weight(F_out: int, F_in: int, d: int, C: int, group: int = 1) -> float:
    """Closed form of stored_bytes per weight: 8/d + 16*C/(group*F_out)."""
    return 8.0 / d + 16.0 * C / (group * F_out)


@dataclass(frozen=True)
class Arch:
    name: str
    hidden: int
    layers: int
    q_out: int
    kv_out: int
    ffn: int
    vocab: int
    tied: bool = False

    def linears(self):
        h = self.hidden
        return [(self.q_out, h), (self.kv_out, h), (self.kv_out, h), (h, self.q_out),
                (self.ffn, h), (self.ffn, h), (h, self.ffn)]

    def aux_params(self) -> int:
        # embeddings + lm_head + 2 RMSNorms per block + final norm
        emb = self.vocab * self.hidden * (1 if self.tied else 2)
        return emb + (2 * self.layers + 1) * self.hidden

    def linear_params(self) -> int:
        return self.layers * sum(o * i for o, i in self.linears())

    def fp16_bytes(self) -> int:
        return 2 * (self.aux_params() + self.linear_params())


# Public model configurations (hidden, blocks, q width, kv width, ffn, vocab).
LLAMA3_8B = Arch("Llama-3-8B", 4096, 32, 4096, 1024, 14336, 128256)
LLAMA2_7B = Arch("LLaMA-2-7B", 4096, 32, 4096, 4096, 11008, 32000)
LLAMA2_13B = Arch("LLaMA-2-13B", 5120, 40, 5120, 5120, 13824, 32000)
QWEN3_8B = Arch("Qwen3-8B", 4096, 36, 4096, 1024, 12288, 151936)


def model_size_percent_ours(arch: Arch, d: int, C: int, group: int = 1) -> float:
    """Eq. 5 with this build's storage: every linear layer packed
    (input-axis subspaces, uint8 indices, fp16 codebooks), aux kept FP16."""
    comp = 0
    for (o, i) in arch.linears():
        comp += stored_bytes(o, i, d, C, group)["total_bytes"]
    size = comp * arch.layers + 2 * arch.aux_params()
    return 100.0 * size / arch.fp16_bytes()


def model_size_percent_paper_fit(arch: Arch, d: int, C: int) -> float:
    """the accounting that reproduces the printed Size%:
    output-axis subspaces (N_ss = F_out/SZ, P:444 dim=0), ceil(log2 K)-bit
    packed indices and 2 bytes per centroid; aux at FP16."""
    lg = math.ceil(math.log2(C))
    comp = 0.0
    for (o, i) in arch.linears():
        comp += lg * (o * i / d) / 8.0 + 2.0 * C * (o / d)
    size = comp * arch.layers + 2 * arch.aux_params()
    return 100.0 * size / arch.fp16_bytes()


def paper_split_k(n_sm: int, blocks_per_sm: int, batch: int, f_out: int, n_ss: int | None = None) -> int:
    """Alg. 2 auto-tuner: ceil(N_SM*8 / (B_s * ceil(F_out/128))),
    clamped to N_ss (SPEC plan_splits)."""
    k = math.ceil(n_sm * blocks_per_sm / (batch * math.ceil(f_out / 128)))
    if n_ss is not None:
        k = min(k, n_ss)
    return max(1, k)


def gemv_algorithmic_bytes(F_out: int, F_in: int, d: int, C: int, group: int = 1, B: int = 1,
                           y_bytes: int = 4) -> int:
    """Bytes the GEMV must move: indices + codebooks + x + y."""
    sb = stored_bytes(F_out, F_in, d, C, group)
    return sb["index_bytes"] + sb["codebook_bytes"] + B * F_in * 2 + B * F_out * y_bytes
