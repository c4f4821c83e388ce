"""Oracle for the fused joint network + loss (rnnt_joint_loss).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

PAPER.md §4.1: the loss is fed by a joint network over Encoder and Predictor embeddings (size 512);
P:58 / P:64: the log-probabilities tensor comes from that network.  The paper does not spell the joint out;
DESIGN.md reading R22 takes the standard transducer joiner in bf16 mixed precision:

    h(b,t,u,:) = bf16( tanh( f(b,t,:) + g(b,u,:) ) )
    z(b,t,u,v) = sum_k h(b,t,u,k) W(v,k) + bias(v)

Here: f, g, W are the bf16 inputs widened exactly to float64; tanh and the sum are float64 (numpy); h is
rounded to the nearest bf16 (ties to even) from the float32 rounding of the float64 tanh; z is handed to the
loss oracle (``oracle.batch``) as float32, the storage type of the loss path's logits.  Plain numpy, one
expression per line of the definition above.
"""
from __future__ import annotations

import numpy as np

from . import batch as _loss_batch


def bf16_round(x):
    """Round to the nearest bfloat16 (ties to even), returned as float64.  Via float32: exact unless the
    float32 rounding lands on a bf16 halfway point (probability ~2^-16 per element)."""
    x32 = np.ascontiguousarray(x, dtype=np.float32)
    bits = x32.view(np.uint32).astype(np.uint64)
    rounded = (bits + 0x7FFF + ((bits >> 16) & 1)) & 0xFFFF0000
    out = rounded.astype(np.uint32).view(np.float32).astype(np.float64)
    nan = np.isnan(x32)
    out[nan] = np.nan
    return out


def joint_logits(f, g, W, bias=None):
    """f [B,Tmax,H], g [B,Umax+1,H], W [V,H] (bf16 values as any float array), bias [V] or None ->
    z float64 [B, Tmax, Umax+1, V]."""
    f = np.asarray(f, np.float64)
    g = np.asarray(g, np.float64)
    W = np.asarray(W, np.float64)
    h = bf16_round(np.tanh(f[:, :, None, :] + g[:, None, :, :]))
    z = h @ W.T
    if bias is not None:
        z = z + np.asarray(bias, np.float64)
    return z


def joint_loss(f, g, W, bias, y, T_b, U_b, blank=0, variant="rnnt"):
    """Per-utterance losses (float64 [B]) of the loss oracle on the joint logits."""
    z = joint_logits(f, g, W, bias)
    losses, _ = _loss_batch(z.astype(np.float32), y, T_b, U_b, blank, variant, grad=False)
    return losses


def joint_loss_and_grads(f, g, W, bias, y, T_b, U_b, blank=0, variant="rnnt", round_bf16=True):
    """Losses and the gradients of their sum w.r.t. (f, g, W, bias) -- the chain rule of the joint above,
    line by line (reading R23: the backward uses the stored bf16 h for tanh' = 1 - h^2, dz is
    rounded to bf16 before the two backward matrix products and dh = dz W is stored in bf16, as a bf16
    training graph stores them).  round_bf16=False drops the roundings (h, dz, dh): the plain real-valued
    chain rule (for pinning).

    Returns (losses [B], d_f [B,Tmax,H], d_g [B,Umax+1,H], d_W [V,H], d_bias [V]), float64."""
    f = np.asarray(f, np.float64)
    g = np.asarray(g, np.float64)
    W = np.asarray(W, np.float64)
    rnd = bf16_round if round_bf16 else (lambda x: np.asarray(x, np.float64))
    h = rnd(np.tanh(f[:, :, None, :] + g[:, None, :, :]))          # [B, T, U+1, H]
    z = h @ W.T
    if bias is not None:
        z = z + np.asarray(bias, np.float64)
    losses, dz = _loss_batch(z.astype(np.float32), y, T_b, U_b, blank, variant, grad=True)
    dz = rnd(dz)                                                     # d sum(loss) / d z, zero on padding
    dh = rnd(dz @ W)                                                 # [B, T, U+1, H], stored in bf16
    d_W = np.einsum("btuv,btuh->vh", dz, h)
    d_bias = dz.sum(axis=(0, 1, 2))
    dpre = dh * (1.0 - h * h)                                        # through tanh
    d_f = dpre.sum(axis=2)                                           # enc(b,t) feeds every u
    d_g = dpre.sum(axis=1)                                           # pred(b,u) feeds every t
    return losses, d_f, d_g, d_W, d_bias
