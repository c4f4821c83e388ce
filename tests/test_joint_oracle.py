"""Pins for the fused-joint oracle (oracle/joint.py, NEXT-4) against things other than itself: torch's own
bf16 rounding and tanh (library routines), the uniform-logits closed form of the loss, and torchaudio's RNN-T
loss on torch-built joint logits."""
import math

import numpy as np
import pytest
import torch

import workloads
from oracle import joint as oj


def test_bf16_round_matches_torch():
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.standard_normal(100_000) * s for s in (1e-3, 1.0, 1e3)] + [[0.0, -0.0, 1.0, -2.5]])
    ref = torch.from_numpy(x.astype(np.float32)).to(torch.bfloat16).double().numpy()
    assert np.array_equal(oj.bf16_round(x), ref)


def test_joint_logits_identity_weight_is_rounded_tanh():
    """W = I (exact in bf16), bias = 0, f = 0: z(t,u,v) = bf16(tanh(g(u,v))) independently of t."""
    B, T, U, H = 2, 3, 4, 128
    enc = torch.zeros(B, T, H, dtype=torch.bfloat16)
    pred = (torch.randn(B, U + 1, H, generator=torch.Generator().manual_seed(5)) * 2).to(torch.bfloat16)
    W = torch.eye(H, dtype=torch.bfloat16)
    z = oj.joint_logits(enc.double().numpy(), pred.double().numpy(), W.double().numpy())
    ref = torch.tanh(pred.double()).to(torch.bfloat16).double().numpy()
    for t in range(T):
        assert np.array_equal(z[:, t], ref)


def test_joint_loss_uniform_closed_form():
    """f + g = 0 and bias = 0 give z = 0: uniform logits, loss = (T+U) ln V - ln C(T-1+U, U)."""
    B, T, U, H, V = 1, 6, 3, 128, 16
    enc = np.zeros((B, T, H))
    pred = np.zeros((B, U + 1, H))
    W = torch.randn(V, H, generator=torch.Generator().manual_seed(1)).to(torch.bfloat16).double().numpy()
    y = np.array([[1, 2, 3]], np.int32)
    l = oj.joint_loss(enc, pred, W, None, y, [T], [U], 0, "rnnt")
    assert abs(l[0] - ((T + U) * math.log(V) - math.log(math.comb(T - 1 + U, U)))) < 1e-9


@pytest.mark.parametrize("variant", ["rnnt"])
def test_joint_loss_matches_torchaudio_on_torch_joint(variant):
    ta = pytest.importorskip("torchaudio")
    B, T, U, H, V = 2, 12, 5, 128, 32
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=9)
    y = torch.randint(1, V, (B, U), generator=torch.Generator().manual_seed(2), dtype=torch.int32)
    T_b = torch.tensor([T, T - 3], dtype=torch.int32)
    U_b = torch.tensor([U, U - 2], dtype=torch.int32)
    # the joint written with torch ops (independent of oracle/joint.py's numpy)
    h = torch.tanh(enc.double()[:, :, None, :] + pred.double()[:, None, :, :]).float().to(torch.bfloat16)
    z = (h.double() @ W.double().T + bias.double()).float()
    ref = ta.functional.rnnt_loss(z, y, T_b, U_b, blank=0, reduction="none", clamp=-1).double().numpy()
    l = oj.joint_loss(enc.double().numpy(), pred.double().numpy(), W.double().numpy(), bias.double().numpy(),
                      y.numpy(), T_b.numpy(), U_b.numpy(), 0, variant)
    assert np.allclose(l, ref, rtol=2e-6, atol=0)


def test_joint_grads_chain_rule_matches_torch_autograd():
    """The oracle's hand-written chain rule (round_bf16=False) against torch autograd in float64 through the
    same joint, with the loss oracle's d loss / d z plugged in as the backward of the loss node."""
    import oracle
    B, T, U, H, V = 2, 6, 3, 128, 16
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=13)
    y = np.array([[1, 2, 3], [4, 5, 0]], np.int32)
    T_b, U_b = np.array([6, 4], np.int32), np.array([3, 2], np.int32)

    class Loss(torch.autograd.Function):
        @staticmethod
        def forward(ctx, z):
            l, dz = oracle.batch(z.detach().numpy().astype(np.float32), y, T_b, U_b, 0, "force_final")
            ctx.save_for_backward(torch.from_numpy(dz))
            return torch.tensor(l.sum(), dtype=torch.float64)

        @staticmethod
        def backward(ctx, go):
            (dz,) = ctx.saved_tensors
            return go * dz

    f = enc.double().requires_grad_()
    g = pred.double().requires_grad_()
    w = W.double().requires_grad_()
    b = bias.double().requires_grad_()
    z = torch.tanh(f[:, :, None, :] + g[:, None, :, :]) @ w.T + b
    Loss.apply(z).backward()
    l, d_f, d_g, d_W, d_b = oj.joint_loss_and_grads(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                                                     bias.double().numpy(), y, T_b, U_b, 0, "force_final",
                                                     round_bf16=False)
    for mine, ref in ((d_f, f.grad), (d_g, g.grad), (d_W, w.grad), (d_b, b.grad)):
        assert np.allclose(mine, ref.numpy(), rtol=1e-9, atol=1e-12)


def test_joint_grads_padding_and_rounding():
    """Padded frames / units get zero input gradients; the bf16 readings change the gradients only at the
    bf16 level (relative 2^-7 of the largest entry)."""
    B, T, U, H, V = 2, 7, 4, 128, 32
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=17)
    y = np.array([[1, 2, 3, 4], [5, 6, 0, 0]], np.int32)
    T_b, U_b = np.array([7, 5], np.int32), np.array([4, 2], np.int32)
    args = (enc.double().numpy(), pred.double().numpy(), W.double().numpy(), bias.double().numpy(), y, T_b, U_b)
    _, d_f, d_g, d_W, d_b = oj.joint_loss_and_grads(*args, 0, "rnnt")
    assert not d_f[1, 5:].any() and not d_g[1, 3:].any()
    _, d_f0, d_g0, d_W0, d_b0 = oj.joint_loss_and_grads(*args, 0, "rnnt", round_bf16=False)
    for a_, b_ in ((d_f, d_f0), (d_g, d_g0), (d_W, d_W0), (d_b, d_b0)):
        assert np.abs(a_ - b_).max() <= 2.0 ** -7 * np.abs(b_).max()
