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


def _torch_autograd_grads(enc, pred, W, bias, y, T_b, U_b, variant, rounded_forward):
    """torch float64 autograd through the joint, with the loss oracle's d loss / d z plugged in as the backward
    of the loss node.  rounded_forward: tanh's output is rounded to bf16 by torch's own conversion and its
    backward is aten's tanh_backward at that saved (rounded) output -- what a bf16 autograd graph does."""
    import oracle

    class Loss(torch.autograd.Function):
        @staticmethod
        def forward(ctx, z):
            l, dz = oracle.batch(z.detach().numpy().astype(np.float32), y, T_b, U_b, 0, variant)
            ctx.save_for_backward(torch.from_numpy(dz))
            return torch.tensor(l.sum(), dtype=torch.float64)

        @staticmethod
        def backward(ctx, go):
            (dz,) = ctx.saved_tensors
            return go * dz

    class Bf16Tanh(torch.autograd.Function):
        @staticmethod
        def forward(ctx, x):
            out = torch.tanh(x).float().to(torch.bfloat16).double()
            ctx.save_for_backward(out)
            return out

        @staticmethod
        def backward(ctx, go):
            (out,) = ctx.saved_tensors
            return torch.ops.aten.tanh_backward(go, out)

    f = enc.double().requires_grad_()
    g = pred.double().requires_grad_()
    w = W.double().requires_grad_()
    b = bias.double().requires_grad_()
    x = f[:, :, None, :] + g[:, None, :, :]
    h = Bf16Tanh.apply(x) if rounded_forward else torch.tanh(x)
    Loss.apply(h @ w.T + b).backward()
    return f.grad.numpy(), g.grad.numpy(), w.grad.numpy(), b.grad.numpy()


@pytest.mark.parametrize("rounding", ["none", "forward"])
def test_joint_grads_chain_rule_matches_torch_autograd(rounding):
    """The oracle's hand-written chain rule against torch autograd in float64 through the same joint: exact
    (rounding="none") and R22's bf16 forward graph (rounding="forward", the GPU parity reference, R23)."""
    B, T, U, H, V = 2, 6, 3, 128, 16
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=13)
    y = np.array([[1, 2, 3], [4, 5, 0]], np.int32)
    T_b, U_b = np.array([6, 4], np.int32), np.array([3, 2], np.int32)
    ref = _torch_autograd_grads(enc, pred, W, bias, y, T_b, U_b, "force_final", rounding == "forward")
    l, d_f, d_g, d_W, d_b = oj.joint_loss_and_grads(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                                                     bias.double().numpy(), y, T_b, U_b, 0, "force_final",
                                                     rounding=rounding)
    for mine, r in zip((d_f, d_g, d_W, d_b), ref):
        assert np.allclose(mine, r, rtol=1e-9, atol=1e-12)


def test_joint_forward_rounding_differs_from_exact():
    """The two references are not the same function: R22's bf16 h moves the gradients at the bf16 level, so a
    test against one cannot pass by accident against the other's arithmetic."""
    B, T, U, H, V = 1, 5, 2, 128, 16
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=21)
    args = (enc.double().numpy(), pred.double().numpy(), W.double().numpy(), bias.double().numpy(),
            np.array([[1, 2]], np.int32), np.array([5], np.int32), np.array([2], np.int32), 0, "rnnt")
    a = oj.joint_loss_and_grads(*args, rounding="forward")
    b = oj.joint_loss_and_grads(*args, rounding="none")
    assert np.abs(a[3] - b[3]).max() > 1e-6 * np.abs(b[3]).max()


def test_joint_grads_padding_and_rounding():
    """Padded frames / units get zero input gradients; the kernel's storage roundings (dz, dh in bf16) move
    each gradient element by at most 2u times its sum of absolute terms (u = 2^-8, bf16; R23's bound), and the
    bf16 forward moves them from the exact ones only at the bf16 level (2^-7 of the largest entry here)."""
    B, T, U, H, V = 2, 7, 4, 128, 32
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=17)
    y = np.array([[1, 2, 3, 4], [5, 6, 0, 0]], np.int32)
    T_b, U_b = np.array([7, 5], np.int32), np.array([4, 2], np.int32)
    args = (enc.double().numpy(), pred.double().numpy(), W.double().numpy(), bias.double().numpy(), y, T_b, U_b)
    ref = oj.joint_loss_and_grads(*args, 0, "rnnt", rounding="forward")
    assert not ref[1][1, 5:].any() and not ref[2][1, 3:].any()
    st = oj.joint_loss_and_grads(*args, 0, "rnnt", rounding="storage")
    A, _ = oj.joint_grad_magnitudes(*args, 0, "rnnt")
    u = 2.0 ** -8
    for name, a_, b_ in zip(("d_f", "d_g", "d_W", "d_bias"), st[1:], ref[1:]):
        assert (np.abs(a_ - b_) <= 2 * u * A[name] + 1e-15).all(), name
    ex = oj.joint_loss_and_grads(*args, 0, "rnnt", rounding="none")
    for a_, b_ in zip(ref[1:], ex[1:]):
        assert np.abs(a_ - b_).max() <= 2.0 ** -7 * np.abs(b_).max()


def test_joint_grad_magnitudes_bound_the_gradients():
    """|gradient| <= its sum of absolute terms, elementwise (triangle inequality) -- and the sums are tight for
    a one-term case: T = 1, U = 0 has one cell per utterance."""
    B, T, U, H, V = 1, 1, 0, 128, 8
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=23)
    args = (enc.double().numpy(), pred.double().numpy(), W.double().numpy(), bias.double().numpy(),
            np.zeros((1, 0), np.int32), np.array([1], np.int32), np.array([0], np.int32), 0, "rnnt")
    ref = oj.joint_loss_and_grads(*args, rounding="forward")
    A, A1 = oj.joint_grad_magnitudes(*args)
    for name, r in zip(("d_f", "d_g", "d_W", "d_bias"), ref[1:]):
        assert (np.abs(r) <= A[name] * (1 + 1e-12) + 1e-300).all(), name
    assert np.allclose(np.abs(ref[4]), A["d_bias"])          # one cell: |sum| = sum of |.|
    assert np.allclose(A1["d_bias"], 1.0)                     # one valid cell per vocabulary entry
