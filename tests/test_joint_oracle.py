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
