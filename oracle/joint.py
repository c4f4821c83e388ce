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
expression per line of the definition above.  The backward (reading R23) is that bf16 graph's chain rule in
real arithmetic (``rounding="forward"``, pinned to torch float64 autograd through torch's own bf16 rounding
and aten's tanh backward in tests/test_joint_oracle.py).
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


def joint_loss_and_grads(f, g, W, bias, y, T_b, U_b, blank=0, variant="rnnt", rounding="forward"):
    """Losses and the gradients of their sum w.r.t. (f, g, W, bias) -- the chain rule of the joint above,
    line by line (reading R23).

    rounding = "forward" (the parity reference): the forward is R22's bf16 graph -- h = bf16(tanh(f + g)) --
        and the backward is that graph's chain rule in real arithmetic: tanh' = 1 - h^2 from the stored h (the
        saved output of tanh, as autograd's tanh backward uses it), dW = dz^T h with the same h; no rounding of
        dz or dh.
    rounding = "none": no rounding at all (h = tanh(f + g)): the plain real-valued chain rule.
    rounding = "storage": "forward" plus dz rounded to bf16 before the two backward products and dh = dz W
        stored in bf16 -- the kernel's own storage points (a diagnostic, not a parity reference).

    Returns (losses [B], d_f [B,Tmax,H], d_g [B,Umax+1,H], d_W [V,H], d_bias [V]), float64."""
    if rounding not in ("forward", "none", "storage"):
        raise ValueError(rounding)
    f = np.asarray(f, np.float64)
    g = np.asarray(g, np.float64)
    W = np.asarray(W, np.float64)
    keep = lambda x: np.asarray(x, np.float64)                        # noqa: E731
    rnd_h = keep if rounding == "none" else bf16_round
    rnd_back = bf16_round if rounding == "storage" else keep
    h = rnd_h(np.tanh(f[:, :, None, :] + g[:, None, :, :]))          # [B, T, U+1, H]
    z = h @ W.T
    if bias is not None:
        z = z + np.asarray(bias, np.float64)
    losses, dz = _loss_batch(z.astype(np.float32), y, T_b, U_b, blank, variant, grad=True)
    dz = rnd_back(dz)                                                # d sum(loss) / d z, zero on padding
    dh = rnd_back(dz @ W)                                            # [B, T, U+1, H]
    d_W = np.einsum("btuv,btuh->vh", dz, h)
    d_bias = dz.sum(axis=(0, 1, 2))
    dpre = dh * (1.0 - h * h)                                        # through tanh
    d_f = dpre.sum(axis=2)                                           # enc(b,t) feeds every u
    d_g = dpre.sum(axis=1)                                           # pred(b,u) feeds every t
    return losses, d_f, d_g, d_W, d_bias


def joint_grad_magnitudes(f, g, W, bias, y, T_b, U_b, blank=0, variant="rnnt"):
    """Sums of absolute terms of each gradient of the "forward" chain rule, for rounding-error bounds (R23):
    with D = |dz| (zero on padding), A_W = D^T |h|, A_bias = sum D, A_h = D |W|, A_f = sum_u A_h (1 - h^2),
    A_g = sum_t A_h (1 - h^2); and the same sums with D = 1 on every valid cell (A1_*, for absolute errors of
    dz).  Returns two dicts keyed "d_f", "d_g", "d_W", "d_bias"."""
    f = np.asarray(f, np.float64)
    g = np.asarray(g, np.float64)
    W = np.asarray(W, np.float64)
    h = bf16_round(np.tanh(f[:, :, None, :] + g[:, None, :, :]))
    z = h @ W.T
    if bias is not None:
        z = z + np.asarray(bias, np.float64)
    _, dz = _loss_batch(z.astype(np.float32), y, T_b, U_b, blank, variant, grad=True)
    B, T, U1, _ = h.shape
    valid = np.zeros((B, T, U1, 1))
    for b in range(B):
        Tb, Ub = int(T_b[b]), int(U_b[b])
        if 1 <= Tb <= T and 0 <= Ub < U1:
            valid[b, :Tb, :Ub + 1] = 1.0

    def sums(D):
        Ah = D @ np.abs(W)
        tp = Ah * (1.0 - h * h)
        return {"d_f": tp.sum(axis=2), "d_g": tp.sum(axis=1),
                "d_W": np.einsum("btuv,btuh->vh", D, np.abs(h)), "d_bias": D.sum(axis=(0, 1, 2))}
    return sums(np.abs(dz)), sums(np.broadcast_to(valid, dz.shape))


BF16_U = 2.0 ** -8      # bf16 unit roundoff (8 significant bits, round to nearest)
DZ_ABS_ERR = 1e-5       # fp32 pipeline error of one dz element (fp32 z / lse / exp; fp64 alpha, beta)


def r23_bounds(f, g, W, bias, y, T_b, U_b, blank=0, variant="rnnt"):
    """Elementwise parity bounds for the fused joint's gradients against ``rounding="forward"`` (R23):
    |gpu - ref| <= 4 u A + DZ_ABS_ERR A1, u = 2^-8.  Derivation: dz stored in bf16 moves every term of dW,
    dbias and dh by <= u |term| (u A); dh = dz W stored in bf16 adds <= u |dh| <= u A_h, passed through tanh' to
    d enc / d pred (total 2u A, the kernel's storage points; checked on the oracle's own "storage" variant in
    tests/test_joint_oracle.py); the GPU's tanh (~2e-7 absolute) can land on the other side of a bf16 rounding
    boundary than float64 tanh, moving that h by one bf16 ulp <= 2u |h| (<= 2u A on the terms it feeds); and
    the fp32 path that produces dz differs from the float64 oracle by <= DZ_ABS_ERR per element (A1 counts the
    valid cells each gradient element sums over, weighted like A).  Returns a dict name -> bound array."""
    A, A1 = joint_grad_magnitudes(f, g, W, bias, y, T_b, U_b, blank, variant)
    return {k: 4 * BF16_U * A[k] + DZ_ABS_ERR * A1[k] for k in A}
