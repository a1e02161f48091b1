"""GPU side of the synthetic-state harness: allocate a rank's tensors as SEPARATE
device allocations (the scattered worst case) and fill them with the
seeded generator through the CUDA copy of it (libreft_synth, include/reft_synth.h).
No method arithmetic here."""
from __future__ import annotations

import torch

from . import SEED, TensorSpec, config_tensors
from paper_2310_12670_b200 import ckpt as C

_ROLE = {"param": C.CKPT_ROLE_PARAM, "master": C.CKPT_ROLE_MASTER, "exp_avg": C.CKPT_ROLE_EXP_AVG,
         "exp_avg_sq": C.CKPT_ROLE_EXP_AVG_SQ}
_DT = {"bf16": torch.bfloat16, "fp32": torch.float32}


def alloc_state(specs, device, misalign: int = 0):
    """One torch allocation per tensor.  misalign > 0 makes every odd tensor a view that
    starts `misalign` elements into a larger allocation (unaligned-view case)."""
    out = []
    for i, s in enumerate(specs):
        dt = _DT[s.dtype]
        if misalign and i % 2 == 1:
            base = torch.empty(s.numel + misalign, dtype=dt, device=device)
            out.append(base[misalign:])
        else:
            out.append(torch.empty(s.numel, dtype=dt, device=device))
    return out


def fill_state(tensors, rank: int, seed: int = SEED, xor_mode: int = 0, stream=None):
    for t_idx, t in enumerate(tensors):
        C.reft_synth_fill(t.data_ptr(), t.numel() * t.element_size(), seed, rank, t_idx, xor_mode, stream)


def descriptors(tensors, specs):
    return [C.tensor_desc(t, _ROLE.get(s.role, C.CKPT_ROLE_OTHER),
                          C.CKPT_TENSOR_REPLICATED if "layernorm" in s.name or s.name.startswith("norm") else 0,
                          s.name)
            for t, s in zip(tensors, specs)]


def make_rank_state(config: str, rank: int, device, seed: int = SEED, misalign: int = 0):
    specs = config_tensors(config, rank)
    ts = alloc_state(specs, device, misalign)
    fill_state(ts, rank, seed)
    return specs, ts
