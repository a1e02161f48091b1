"""Seeded synthetic inputs for REFT snapshot-and-protect -- shared by the oracle side
and the CUDA side (tests, smoke, bench).  Holds NONE of the method's arithmetic: no
packing, no parity, no rebuild.  Two things live here:

* ``fill``: the counter-based generator (SplitMix64 finaliser, SURVEY.md 8(c)
  "Generator").  The oracle has its own C copy
  (oracle/reft_oracle.c) and the GPU harness its own CUDA copy
  (paper_2310_12670_b200/csrc/synth_fill.cu); a test pins all three to each other
  and to the published SplitMix64 output sequence.
* ``llama_layout``: per-rank tensor lists (name, dtype, numel) for the
  BASELINE.json configs, from public Llama-2 shapes.
  bf16 param + fp32 master + fp32 exp_avg + fp32 exp_avg_sq per model tensor
  (Adam's "triple extra parameters", PAPER.md P.671; Q8), role-major (Q6).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

SEED = 12670
_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def _sm(x):
    with np.errstate(over="ignore"):
        z = np.asarray(x, dtype=np.uint64) + _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def splitmix64(x: int) -> int:
    return int(_sm(np.uint64(x)))


def tensor_base(seed: int, rank: int, tensor: int) -> int:
    return int(_sm(_sm(_sm(np.uint64(seed)) ^ np.uint64(rank)) ^ np.uint64(tensor)))


def fill(seed: int, rank: int, tensor: int, nbytes: int) -> np.ndarray:
    """Bytes of tensor ``tensor`` of rank ``rank``: word w = sm(base ^ w), little-endian."""
    nwords = (nbytes + 7) // 8
    base = np.uint64(tensor_base(seed, rank, tensor))
    w = _sm(base ^ np.arange(nwords, dtype=np.uint64))
    return w.astype("<u8").view(np.uint8)[:nbytes].copy()


# ---------------------------------------------------------------------------------------
# Llama-2 layouts (public shapes [ext])
# ---------------------------------------------------------------------------------------
@dataclass(frozen=True)
class LlamaShape:
    name: str
    vocab: int
    hidden: int
    layers: int
    ffn: int
    heads: int
    kv_heads: int


LLAMA = {
    "7b": LlamaShape("Llama-2-7B", 32000, 4096, 32, 11008, 32, 32),
    "13b": LlamaShape("Llama-2-13B", 32000, 5120, 40, 13824, 40, 40),
    # Q16: "Llama-2-34B" was never released; CodeLlama-34B shape (GQA, 8 KV heads).
    "34b": LlamaShape("Llama-2-34B", 32000, 8192, 48, 22016, 64, 8),
}

ROLES = (("param", "bf16", 2), ("master", "fp32", 4), ("exp_avg", "fp32", 4), ("exp_avg_sq", "fp32", 4))


@dataclass(frozen=True)
class TensorSpec:
    name: str
    dtype: str  # "bf16" | "fp32"
    numel: int
    role: str

    @property
    def nbytes(self) -> int:
        return self.numel * (2 if self.dtype == "bf16" else 4)


def _model_tensors(s: LlamaShape, tp: int, layer_range, first: bool, last: bool):
    """(name, numel) of one TP shard of the given layers (Q17/Q18 sharding rules)."""
    h, f, hd = s.hidden, s.ffn, s.hidden // s.heads
    kv = s.kv_heads * hd
    out = []
    if first:
        out.append(("embed_tokens", (s.vocab // tp) * h))
    for i in layer_range:
        p = f"layers.{i}."
        out += [
            (p + "q_proj", (h // tp) * h),
            (p + "k_proj", (kv // tp) * h),
            (p + "v_proj", (kv // tp) * h),
            (p + "o_proj", h * (h // tp)),
            (p + "gate_proj", (f // tp) * h),
            (p + "up_proj", (f // tp) * h),
            (p + "down_proj", h * (f // tp)),
            (p + "input_layernorm", h),
            (p + "post_attention_layernorm", h),
        ]
    if last:
        out += [("norm", h), ("lm_head", (s.vocab // tp) * h)]
    return out


def rank_tensors(model: str, tp: int, pp: int, pp_rank: int):
    """Role-major list of TensorSpec for the TP shard of PP stage ``pp_rank``."""
    s = LLAMA[model]
    per = s.layers // pp
    lr = range(pp_rank * per, (pp_rank + 1) * per)
    mt = _model_tensors(s, tp, lr, pp_rank == 0, pp_rank == pp - 1)
    return [TensorSpec(f"{n}.{role}", dt, numel, role) for role, dt, _ in ROLES for n, numel in mt]


# BASELINE.json configs -> (description, per-rank tensor list builder, group size m)
CONFIGS = {
    "c1_16mb_fp32_m8": "8-rank RAIM5 XOR-parity encode + rebuild, 16 MiB seeded fp32 shard per rank",
    "c2_7b_tp8": "Llama-2-7B bf16 params + fp32 Adam state, TP=8, full snapshot+protect",
    "c3_13b_tp4pp2": "Llama-2-13B TP=4 PP=2 layout, bucket sweep, D2H overlap with GEMM",
    "c4_34b_tp8_stage0": "Llama-2-34B TP=8 per-node state (PP stage 0 of 4)",
    "c5_13b_drill": "Failure drill: Llama-2-13B TP4 PP2, lose rank k, rebuild + load",
}


def config_tensors(config: str, rank: int):
    """Per-rank tensor list of a BASELINE.json config (rank = local rank in the node)."""
    if config.startswith("c1"):
        return [TensorSpec("shard", "fp32", 4 * 1024 * 1024, "param")]
    if config.startswith("c2"):
        return rank_tensors("7b", 8, 1, 0)
    if config.startswith("c3") or config.startswith("c5"):
        return rank_tensors("13b", 4, 2, (rank // 4) % 2)
    if config.startswith("c4"):
        return rank_tensors("34b", 8, 4, 0)
    if config.startswith("tiny"):
        # small ragged layout for parity tests: odd sizes, both dtypes
        rng = np.random.default_rng(1000 + rank)
        out = []
        for i in range(int(config.split("_")[1]) if "_" in config else 7):
            numel = int(rng.integers(1, 40000))
            out.append(TensorSpec(f"t{i}", "bf16" if i % 2 == 0 else "fp32", numel, "param"))
        return out
    raise KeyError(config)
