"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the CPU oracle.

This module draws random numbers and lays them out; it holds NONE of the method's arithmetic (no
softmax, no lattice, no loss).  Both sides receive the same tensors: the oracle never sees values
produced by the CUDA path, and the CUDA path never sees values produced by the oracle.

Input recipe (DESIGN.md §"Input recipe"):
  * logits  z[b] ~ i.i.d. N(0,1) fp32 of shape [Tmax, Umax+1, V], one generator per GLOBAL utterance
    id b seeded with ``logit_seed + b`` (so a shard's data never depends on rank or world size);
    padded cells are drawn too (or overwritten with ``pad_value``).  ``scale`` > 1 gives the "peaky"
    numerics variant (occupancies near 1).
  * lengths  T_b ~ U{t_lo..Tmax}, U_b ~ U{u_lo..Umax} from numpy seed ``len_seed`` over the global batch,
    b=0 pinned to (Tmax, Umax); fixed-length configs use T_b = Tmax, U_b = Umax.
  * targets  uniform over [0, V) minus the blank id, numpy seed ``tgt_seed + b``; padding entries are
    ``pad_target``.  c4 truncates longer transcripts at both ends (§4.1: "We discarded 20%
    and 50% of the words from each training utterance in a random left-right proportion").
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    B: int
    Tmax: int
    Umax: int
    V: int
    blank: int = 0
    variant: str = "rnnt"            # rnnt | force_final | allow_ignore
    variable_lengths: bool = False
    t_lo: int = 1
    u_lo: int = 0
    logit_seed: int = 0
    len_seed: int = 1
    tgt_seed: int = 7
    drop: tuple = ()                 # c4: word-drop fractions, cycled over b
    drop_seed: int = 3
    fixed_targets: tuple = ()        # c1: explicit transcript
    per_gpu: int = 0                 # utterances per GPU when B is a multi-GPU global batch (c5); 0 = B

    @property
    def B_per_gpu(self) -> int:
        return self.per_gpu or self.B

    @property
    def cells_per_utt(self) -> int:
        return self.Tmax * (self.Umax + 1)

    @property
    def logits_bytes(self) -> int:
        return self.B * self.cells_per_utt * self.V * 4


# BASELINE.json "configs", in order.
CONFIGS = {
    # Fig.1 toy: four frames, "A C" over vocabulary {<b>, A, B, C}.
    "c1": Config("fig1_toy", B=1, Tmax=4, Umax=2, V=4, blank=0, fixed_targets=(1, 3)),
    "c2": Config("B16_T200_U50_V256_var", B=16, Tmax=200, Umax=50, V=256, variable_lengths=True,
                 t_lo=100, u_lo=25, logit_seed=1000, len_seed=1),
    "c3": Config("B32_T500_U100_V1024", B=32, Tmax=500, Umax=100, V=1024, logit_seed=2000),
    "c4": Config("B32_T500_U100_V1024_wrnnt", B=32, Tmax=500, Umax=100, V=1024, logit_seed=2000,
                 variant="force_final", drop=(0.2, 0.5)),
    "c5": Config("B256_T1000_U200_V4096", B=256, Tmax=1000, Umax=200, V=4096, logit_seed=5000, per_gpu=32),
}
# Not a BASELINE config: the paper's own loss benchmark (§4.1, read per DESIGN.md c15): batch 30,
# vocabulary 500, time 101..433 and units 73..92 across the batch; with Encoder/Predictor embeddings of 512 it
# is the fused joint's natural workload (bench --mode joint --config p124).
EXTRA_CONFIGS = {
    "p124": Config("B30_T433_U92_V500_var", B=30, Tmax=433, Umax=92, V=500, variable_lengths=True, t_lo=101,
                   u_lo=73, logit_seed=1240, len_seed=124),
}


def lengths(cfg: Config):
    """(T_b, U_b) int32 arrays over the GLOBAL batch."""
    if not cfg.variable_lengths:
        return (np.full(cfg.B, cfg.Tmax, np.int32), np.full(cfg.B, cfg.Umax, np.int32))
    rs = np.random.RandomState(cfg.len_seed)
    T = rs.randint(cfg.t_lo, cfg.Tmax + 1, size=cfg.B).astype(np.int32)
    U = rs.randint(cfg.u_lo, cfg.Umax + 1, size=cfg.B).astype(np.int32)
    T[0], U[0] = cfg.Tmax, cfg.Umax
    return T, U


def _draw_units(rng, n, V, blank):
    v = rng.integers(0, V - 1, size=n)
    return np.where(v >= blank, v + 1, v).astype(np.int32)   # uniform over [0,V) \ {blank}


def targets(cfg: Config, U_b, b_ids=None, pad_target: int = 0):
    """int32 [len(b_ids), max(Umax,1)] targets; row i belongs to global utterance b_ids[i]."""
    b_ids = range(cfg.B) if b_ids is None else b_ids
    out = np.full((len(b_ids), max(cfg.Umax, 1)), pad_target, np.int32)
    for i, b in enumerate(b_ids):
        n = int(U_b[b])
        if cfg.fixed_targets:
            out[i, :n] = np.asarray(cfg.fixed_targets[:n], np.int32)
            continue
        rng = np.random.default_rng(cfg.tgt_seed + b)
        if cfg.drop:
            p = cfg.drop[b % len(cfg.drop)]
            n_orig = int(round(n / (1.0 - p)))
            full = _draw_units(rng, n_orig, cfg.V, cfg.blank)
            r = np.random.default_rng(cfg.drop_seed * 100003 + b).random()
            left = int(math.floor((n_orig - n) * r))
            out[i, :n] = full[left:left + n]
        else:
            out[i, :n] = _draw_units(rng, n, cfg.V, cfg.blank)
    return out[:, :cfg.Umax] if cfg.Umax > 0 else out[:, :0]


def fill_logits(out: torch.Tensor, cfg: Config, b_ids, scale: float = 1.0):
    """Fill ``out`` [len(b_ids), Tmax, Umax+1, V] (fp32, any device) with N(0,1)*scale per global id."""
    assert out.shape == (len(b_ids), cfg.Tmax, cfg.Umax + 1, cfg.V), out.shape
    for i, b in enumerate(b_ids):
        g = torch.Generator(device=out.device)
        g.manual_seed(cfg.logit_seed + int(b))
        out[i].normal_(0.0, 1.0, generator=g)
        if scale != 1.0:
            out[i].mul_(scale)
    return out


def pad_cells(logits: torch.Tensor, T_b, U_b, value: float):
    """Overwrite every padded cell (t >= T_b or u > U_b) with ``value`` (e.g. NaN for padding tests)."""
    for i in range(logits.shape[0]):
        logits[i, int(T_b[i]):] = value
        logits[i, :, int(U_b[i]) + 1:] = value
    return logits


def problem(cfg: Config, b_ids=None, device="cpu", scale: float = 1.0, pad_value=None,
            pad_target: int = 0):
    """Everything one call needs for the utterances ``b_ids`` (default: the whole global batch)."""
    b_ids = list(range(cfg.B)) if b_ids is None else list(b_ids)
    T_all, U_all = lengths(cfg)
    y = targets(cfg, U_all, b_ids, pad_target)
    T_b = T_all[b_ids].copy()
    U_b = U_all[b_ids].copy()
    z = torch.empty((len(b_ids), cfg.Tmax, cfg.Umax + 1, cfg.V), dtype=torch.float32, device=device)
    fill_logits(z, cfg, b_ids, scale)
    if pad_value is not None:
        pad_cells(z, T_b, U_b, pad_value)
    return {"logits": z, "targets": y, "logit_lens": T_b, "target_lens": U_b,
            "blank": cfg.blank, "variant": cfg.variant, "cfg": cfg, "b_ids": b_ids}


def random_config(B, Tmax, Umax, V, seed, blank=0, variant="rnnt", variable=True):
    """A small random configuration for parity/property tests (lengths variable unless told otherwise)."""
    return Config(f"rand_B{B}_T{Tmax}_U{Umax}_V{V}_s{seed}", B=B, Tmax=Tmax, Umax=Umax, V=V, blank=blank,
                  variant=variant, variable_lengths=variable, t_lo=1, u_lo=0, logit_seed=10_000 * seed,
                  len_seed=seed, tgt_seed=77 * seed + 5)


def joint_inputs(B, Tmax, Umax, H, V, seed, device="cpu"):
    """Seeded inputs of the fused joint network (NEXT-4, §4.1: Encoder / Predictor embeddings
    of size H = 512): enc [B,Tmax,H] and pred [B,Umax+1,H] ~ N(0, 1/2) each (so enc + pred ~ N(0, 1), the
    pre-activation range of a trained joiner), weight [V,H] ~ N(0, 1/H), all rounded to bf16; bias [V] ~
    N(0, 0.1^2) fp32.  Per-utterance streams (seed, b) as for the logits, so a shard is a slice."""
    gen = torch.Generator().manual_seed(7_000_003 * seed + 11)
    weight = (torch.randn(V, H, generator=gen) / math.sqrt(H)).to(torch.bfloat16)
    bias = torch.randn(V, generator=gen) * 0.1
    enc = torch.empty(B, Tmax, H, dtype=torch.bfloat16)
    pred = torch.empty(B, Umax + 1, H, dtype=torch.bfloat16)
    for b in range(B):
        gb = torch.Generator().manual_seed(7_000_003 * seed + 1_000 + b)
        enc[b] = (torch.randn(Tmax, H, generator=gb) * math.sqrt(0.5)).to(torch.bfloat16)
        pred[b] = (torch.randn(Umax + 1, H, generator=gb) * math.sqrt(0.5)).to(torch.bfloat16)
    return enc.to(device), pred.to(device), weight.to(device), bias.to(device)
