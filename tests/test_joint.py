"""GPU parity of the fused joint network + loss (rnnt_joint_loss, NEXT-4: tcgen05 GEMM with the log-softmax /
Populate epilogue, then K2) vs the oracle (oracle/joint.py, pinned in tests/test_joint_oracle.py).  Bar: loss
within 1e-5 relative (floor |L| >= 1), the loss path's bar; the GEMM accumulates in fp32 and h is rounded to
bf16 on both sides (reading R22)."""
import numpy as np
import pytest
import torch

import workloads
from oracle import joint as oj

pytestmark = pytest.mark.gpu
VARIANTS = ("rnnt", "force_final", "allow_ignore")


@pytest.fixture(scope="module")
def rb():
    import paper_2303_10384_b200
    return paper_2303_10384_b200


def _case(rb, B, T, U, H, V, seed, variant, blank=0, variable=True, bias=True):
    cfg = workloads.random_config(B, T, U, V, seed=seed, blank=blank, variant=variant, variable=variable)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=seed)
    if not bias:
        b = None
    losses = rb.rnnt_joint_loss(enc.cuda(), pred.cuda(), W.cuda(), None if b is None else b.cuda(), y, T_b, U_b,
                                blank, variant)
    torch.cuda.synchronize()
    ref = oj.joint_loss(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                        None if b is None else b.double().numpy(), y, T_b, U_b, blank, variant)
    l = losses.cpu().numpy().astype(np.float64)
    rel = np.abs(l - ref) / np.maximum(np.abs(ref), 1.0)
    assert rel.max() <= 1e-5, (rel.max(), l, ref)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("shape", [(2, 9, 4, 128, 128), (3, 37, 11, 256, 384), (2, 50, 20, 512, 1024),
                                   (2, 30, 9, 512, 500), (2, 11, 5, 128, 37)],
                         ids=lambda s: "B{}_T{}_U{}_H{}_V{}".format(*s))
def test_joint_loss_matches_oracle(rb, shape, variant):
    B, T, U, H, V = shape
    _case(rb, B, T, U, H, V, seed=sum(shape) % 97 + 3, variant=variant)


def test_joint_blank_last_no_bias_many_tiles(rb):
    # > 148 row tiles (every CTA loops), ragged last tile, blank = V-1, no bias
    _case(rb, 4, 120, 40, 384, 256, seed=17, variant="rnnt", blank=255, variable=False, bias=False)


def test_joint_matches_materialised_loss_path(rb):
    """Same utterances two ways on the GPU: the fused path, and the oracle-built logits through rnnt_loss."""
    B, T, U, H, V = 3, 60, 25, 512, 512
    cfg = workloads.random_config(B, T, U, V, seed=23, variant="allow_ignore")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=23)
    z = torch.from_numpy(oj.joint_logits(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                                         b.double().numpy()).astype(np.float32)).cuda()
    l_ref, _ = rb.wrnnt_loss(z, y, T_b, U_b, 0, "allow_ignore", grads=False)
    l = rb.rnnt_joint_loss(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "allow_ignore")
    torch.cuda.synchronize()
    assert torch.allclose(l, l_ref, rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("variant", ("rnnt", "allow_ignore"))
def test_joint_large_vocabulary(rb, variant):
    # V = 32003: 251 N tiles, ragged last tile; shared memory does not depend on V (bias read from global)
    _case(rb, 2, 6, 3, 128, 32003, seed=41, variant=variant)


def test_joint_grad_large_vocabulary(rb):
    B, T, U, H, V = 2, 5, 3, 128, 8195
    cfg = workloads.random_config(B, T, U, V, seed=43, variant="force_final")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=43)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "force_final")
    torch.cuda.synchronize()
    ref = oj.joint_loss_and_grads(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                                  b.double().numpy(), y, T_b, U_b, 0, "force_final")
    l = out[0].cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref[0]) / np.maximum(np.abs(ref[0]), 1.0)).max() <= 1e-5
    for name, mine, r in zip(("d_enc", "d_pred", "d_weight", "d_bias"), out[1:], ref[1:]):
        err = np.abs(mine.cpu().numpy().astype(np.float64) - r).max()
        assert err <= 2e-3 * np.abs(r).max(), (name, err, np.abs(r).max())


@pytest.mark.parametrize("scale", [2.0, 8.0])
def test_joint_large_preactivations(rb, scale):
    """enc, pred scaled up (|f + g| up to ~6 sigma * scale: saturated tanh, h = +-1 in bf16 for large |x|):
    loss and gradients still match the oracle's bf16(tanh(f + g)).  d enc / d pred bar 5e-3 of the largest
    entry: they sum dh (stored in bf16, reading R23) times tanh' = 1 - h^2 over up to U+1 / T terms, and a
    one-ulp difference in a bf16 dh (fp32 vs fp64 accumulation of dz W) shifts a term by 2^-8 of itself;
    measured 2.6e-3 at scale 2 (5e-6 at scale 8, where most tanh' vanish)."""
    B, T, U, H, V = 2, 17, 6, 256, 384
    cfg = workloads.random_config(B, T, U, V, seed=53, variant="allow_ignore")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=53)
    enc = (enc.float() * scale).to(torch.bfloat16)
    pred = (pred.float() * scale).to(torch.bfloat16)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "allow_ignore")
    l = rb.rnnt_joint_loss(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "allow_ignore")
    torch.cuda.synchronize()
    ref = oj.joint_loss_and_grads(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                                  b.double().numpy(), y, T_b, U_b, 0, "allow_ignore")
    for losses in (l, out[0]):
        lg = losses.cpu().numpy().astype(np.float64)
        assert (np.abs(lg - ref[0]) / np.maximum(np.abs(ref[0]), 1.0)).max() <= 1e-5, (lg, ref[0])
    for name, mine, r, bar in zip(("d_enc", "d_pred", "d_weight", "d_bias"), out[1:], ref[1:], (5e-3, 5e-3, 2e-3, 2e-3)):
        err = np.abs(mine.cpu().numpy().astype(np.float64) - r).max()
        assert err <= bar * np.abs(r).max(), (name, err, np.abs(r).max())


def test_joint_rejects_misaligned_bias(rb):
    enc, pred, W, b = workloads.joint_inputs(1, 4, 2, 128, 130, seed=5)
    bb = torch.zeros(131, device="cuda")[1:]  # 4-byte offset
    with pytest.raises(rb.RnntError):
        rb.rnnt_joint_loss(enc.cuda(), pred.cuda(), W.cuda(), bb, [[1, 2]], [4], [2])


def test_joint_rejects_unsupported_shapes(rb):
    enc = torch.zeros(1, 4, 96, dtype=torch.bfloat16, device="cuda")
    pred = torch.zeros(1, 3, 96, dtype=torch.bfloat16, device="cuda")
    W = torch.zeros(128, 96, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(rb.RnntError):
        rb.rnnt_joint_loss(enc, pred, W, None, [[1, 2]], [4], [2])


def test_joint_many_short_utterances(rb):
    # 300 utterances of a few cells each (variable lengths): the compact row map crosses many utterance
    # boundaries inside every 128-row tile
    _case(rb, 300, 5, 3, 128, 128, seed=29, variant="force_final")


@pytest.mark.parametrize("variant", VARIANTS)
def test_joint_viterbi_matches_oracle(rb, variant):
    """rnnt_joint_viterbi (K6 + K4) vs the Viterbi oracle on the oracle-built joint logits: same best score
    (1e-5 relative) and the same alignment (reading R21 tie-break; random logits have no ties)."""
    import oracle
    B, T, U, H, V = 3, 40, 12, 256, 256
    cfg = workloads.random_config(B, T, U, V, seed=31, variant=variant)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=31)
    best, frames, span = rb.rnnt_joint_viterbi(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, variant)
    torch.cuda.synchronize()
    z = oj.joint_logits(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                        b.double().numpy()).astype(np.float32)
    from tests.test_viterbi import _path_score
    for i in range(B):
        T, U = int(T_b[i]), int(U_b[i])
        ref_best, ref_frames, ref_span = oracle.viterbi(z[i], T, U, y[i][:U], 0, variant)
        assert abs(best[i].item() - ref_best) <= 1e-5 * max(abs(ref_best), 1.0)
        f = frames[i, :U].cpu().numpy()
        sp = tuple(span[i].cpu().numpy().tolist())
        if f.tolist() != list(ref_frames) or sp != tuple(ref_span):
            # a near-tie under the GPU's fp32 accumulation: its alignment must score as well, to rounding
            sg = _path_score(z[i], y[i], T, U, 0, f, sp, variant)
            assert abs(sg - ref_best) <= 1e-5 * max(abs(ref_best), 1.0)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("shape", [(2, 9, 4, 128, 128), (3, 30, 10, 256, 500), (2, 40, 16, 512, 1024)],
                         ids=lambda s: "B{}_T{}_U{}_H{}_V{}".format(*s))
def test_joint_loss_grad_matches_oracle(rb, shape, variant):
    """rnnt_joint_loss_grad (K6, K2, K6<grad>, cuBLAS, K7) vs the oracle's chain rule under reading R23.
    Bars: losses 1e-5 relative; each gradient within 2e-3 of its largest entry (bf16 dz: an element whose
    GPU value sits within ~1e-6 of a bf16 rounding boundary may round the other way; fp32 vs fp64 sums)."""
    B, T, U, H, V = shape
    cfg = workloads.random_config(B, T, U, V, seed=sum(shape) % 89 + 7, variant=variant)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=sum(shape) % 89 + 7)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, variant)
    torch.cuda.synchronize()
    ref = oj.joint_loss_and_grads(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                                  b.double().numpy(), y, T_b, U_b, 0, variant)
    l = out[0].cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref[0]) / np.maximum(np.abs(ref[0]), 1.0)).max() <= 1e-5
    for name, mine, r in zip(("d_enc", "d_pred", "d_weight", "d_bias"), out[1:], ref[1:]):
        err = np.abs(mine.cpu().numpy().astype(np.float64) - r).max()
        assert err <= 2e-3 * np.abs(r).max(), (name, err, np.abs(r).max())


def test_joint_edge_cases(rb):
    """T = 1, U = 0 and an invalid length in one batch; B = 0 is a no-op."""
    H, V = 128, 128
    enc, pred, W, b = workloads.joint_inputs(3, 5, 3, H, V, seed=37)
    y = np.array([[1, 2, 3], [4, 5, 6], [7, 8, 9]], np.int32)
    T_b = np.array([1, 5, 6], np.int32)   # utterance 2: T > Tmax -> NaN loss, zero gradients
    U_b = np.array([3, 0, 2], np.int32)
    l = rb.rnnt_joint_loss(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "allow_ignore")
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "allow_ignore")
    torch.cuda.synchronize()
    ref = oj.joint_loss_and_grads(enc[:2].double().numpy(), pred[:2].double().numpy(), W.double().numpy(),
                                  b.double().numpy(), y[:2], T_b[:2], U_b[:2], 0, "allow_ignore")
    lg = l.cpu().numpy().astype(np.float64)
    assert np.isnan(lg[2]) and np.isnan(out[0][2].item())
    assert (np.abs(lg[:2] - ref[0]) / np.maximum(np.abs(ref[0]), 1.0)).max() <= 1e-5
    assert not out[1][2].any() and not out[2][2].any()
    # the two valid utterances' gradients; W / bias gradients get nothing from the invalid one
    for mine, r in ((out[1][:2], ref[1]), (out[2][:2], ref[2]), (out[3], ref[3]), (out[4], ref[4])):
        assert np.abs(mine.cpu().numpy().astype(np.float64) - r).max() <= 2e-3 * np.abs(r).max()
    e = torch.zeros(0, 5, H, dtype=torch.bfloat16, device="cuda")
    p = torch.zeros(0, 4, H, dtype=torch.bfloat16, device="cuda")
    assert rb.rnnt_joint_loss(e, p, W.cuda(), b.cuda(), np.zeros((0, 3), np.int32), [], []).numel() == 0


def test_joint_grad_scale(rb):
    """grad_scale[b] scales utterance b's contribution: the gradients equal those of the oracle's sum of
    scaled losses (here: only the gradients change; the losses stay per utterance)."""
    B, T, U, H, V = 3, 20, 6, 128, 256
    cfg = workloads.random_config(B, T, U, V, seed=43)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=43)
    scale = torch.tensor([0.5, 2.0, 0.0])
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "rnnt",
                                  grad_scale=scale)
    torch.cuda.synchronize()
    refs = [oj.joint_loss_and_grads(enc[i:i + 1].double().numpy(), pred[i:i + 1].double().numpy(),
                                    W.double().numpy(), b.double().numpy(), y[i:i + 1], T_b[i:i + 1], U_b[i:i + 1],
                                    0, "rnnt") for i in range(B)]
    d_w = sum(float(scale[i]) * refs[i][3] for i in range(B))
    assert np.abs(out[3].cpu().numpy() - d_w).max() <= 2e-3 * np.abs(d_w).max()
    assert not out[1][2].any()  # scale 0: no gradient into utterance 2's encoder frames
    for i in range(2):
        r = float(scale[i]) * refs[i][1][0]
        assert np.abs(out[1][i].cpu().numpy() - r).max() <= 2e-3 * np.abs(r).max()


def test_joint_grad_valid_rows_paths(rb):
    """Host lengths (valid_rows hint: GEMMs over the valid cells) and device lengths (-1: every padded row, tail
    zeroed) give the same result; a wrong hint is a loud failure (NaN losses)."""
    B, T, U, H, V = 4, 23, 9, 128, 500
    cfg = workloads.random_config(B, T, U, V, seed=47, variant="rnnt")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=47)
    args = (enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y)
    n = rb.joint_valid_rows(T_b, U_b, T, U)
    assert n == int(sum(int(t) * (int(u) + 1) for t, u in zip(T_b, U_b))) and n < B * T * (U + 1)
    host = rb.rnnt_joint_loss_grad(*args, T_b, U_b, 0, "rnnt")
    dev = rb.rnnt_joint_loss_grad(*args, torch.from_numpy(T_b).cuda(), torch.from_numpy(U_b).cuda(), 0, "rnnt")
    torch.cuda.synchronize()
    assert torch.equal(host[0], dev[0])
    for a, c in zip(host[1:], dev[1:]):
        assert torch.allclose(a, c, rtol=1e-5, atol=1e-6 * c.abs().max().item())
    bad = rb.rnnt_joint_loss_grad(*args, T_b, U_b, 0, "rnnt", valid_rows=n - 1)
    torch.cuda.synchronize()
    assert torch.isnan(bad[0]).all()
    with pytest.raises(rb.RnntError):
        rb.rnnt_joint_loss_grad(*args, T_b, U_b, 0, "rnnt", valid_rows=B * T * (U + 1) + 1)
