"""Out-of-bounds guards (compute-sanitizer is closed on this GPU pool): every device buffer an
entry point touches is embedded between NaN / 0xFF canary regions of 1 MiB.  After the call the canaries must
be bit-identical (no out-of-bounds write) and the results must still match the oracle (an out-of-bounds read of
a NaN canary that reached any result would show up as a NaN)."""
import numpy as np
import pytest
import torch

import oracle
import workloads

pytestmark = pytest.mark.gpu
CANARY = 1 << 20  # bytes


@pytest.fixture(scope="module")
def rb():
    import paper_2303_10384_b200
    return paper_2303_10384_b200


class Guarded:
    """A device byte buffer with canaries on both sides; .view(dtype, shape) is the usable middle."""

    def __init__(self, nbytes):
        self.n = nbytes
        self.buf = torch.empty(nbytes + 2 * CANARY, dtype=torch.uint8, device="cuda")
        self.buf[:CANARY].fill_(0xFF)        # 0xFFFFFFFF is a NaN for fp32 / fp64
        self.buf[CANARY + nbytes:].fill_(0xFF)
        self.ref = torch.cat([self.buf[:CANARY], self.buf[CANARY + nbytes:]]).clone()

    def view(self, dtype, shape):
        esz = torch.empty(0, dtype=dtype).element_size()
        count = int(np.prod(shape)) if len(shape) else 1
        return self.buf[CANARY:CANARY + count * esz].view(dtype).view(shape)

    def intact(self):
        now = torch.cat([self.buf[:CANARY], self.buf[CANARY + self.n:]])
        return torch.equal(now, self.ref)


def _guarded_call(rb, cfg, variant, dtype=torch.float32, inplace=False):
    pb = workloads.problem(cfg)
    B, Tmax, Up1, V = pb["logits"].shape
    Umax = Up1 - 1
    esz = torch.empty(0, dtype=dtype).element_size()
    gz = Guarded(B * Tmax * Up1 * V * esz)
    z = gz.view(dtype, (B, Tmax, Up1, V))
    z.copy_(pb["logits"].to(dtype).cuda())
    gg = gz if inplace else Guarded(B * Tmax * Up1 * V * esz)
    g = z if inplace else gg.view(dtype, (B, Tmax, Up1, V))
    gw = Guarded(rb.rnnt_workspace_bytes(B, Tmax, Umax))
    gl = Guarded(4 * B)
    gt = Guarded(4 * max(B * Umax, 1))
    t = gt.view(torch.int32, (B, Umax))
    t.copy_(torch.from_numpy(pb["targets"]).cuda())
    zs = z.float().cpu().numpy()
    losses, grads = rb.loss(z, t, pb["logit_lens"], pb["target_lens"], cfg.blank, variant, grads=g,
                            losses=gl.view(torch.float32, (B,)), workspace=gw.view(torch.uint8, (gw.n,)))
    torch.cuda.synchronize()
    for guard in (gz, gg, gw, gl, gt):
        assert guard.intact()
    ref_l, ref_g = oracle.batch(zs, pb["targets"], pb["logit_lens"], pb["target_lens"], cfg.blank, variant)
    l = losses.cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1)).max() <= 1e-5
    tol = 1e-4 if dtype == torch.float32 else 1e-4 + 2.0 ** -8 * np.abs(ref_g)
    assert (np.abs(grads.float().cpu().numpy() - ref_g) <= tol).all()


@pytest.mark.parametrize("variant", ("rnnt", "force_final", "allow_ignore"))
def test_canaries_sequential_path(rb, variant):
    _guarded_call(rb, workloads.random_config(3, 40, 17, 100, seed=71, variant=variant), variant)


@pytest.mark.parametrize("variant", ("rnnt", "allow_ignore"))
def test_canaries_chunked_overlap_path_in_place(rb, variant):
    # >= 2^24 elements: 4 chunks on internal streams; first and last utterances exercise K2's padded prefetch
    _guarded_call(rb, workloads.random_config(4, 150, 30, 1024, seed=72, variant=variant), variant, inplace=True)


def test_canaries_bf16_grouped_rows(rb):
    _guarded_call(rb, workloads.random_config(5, 30, 12, 256, seed=73), "force_final", dtype=torch.bfloat16)


def test_canaries_viterbi_and_lattice(rb):
    from paper_2303_10384_b200 import lattice as rlat
    cfg = workloads.random_config(3, 30, 10, 64, seed=74, variant="force_final")
    pb = workloads.problem(cfg)
    B, Tmax, Up1, V = pb["logits"].shape
    gz = Guarded(pb["logits"].numel() * 4)
    z = gz.view(torch.float32, tuple(pb["logits"].shape))
    z.copy_(pb["logits"].cuda())
    gw = Guarded(rb.rnnt_workspace_bytes(B, Tmax, Up1 - 1))
    best, frames, span = rb.rnnt_viterbi(z, pb["targets"], pb["logit_lens"], pb["target_lens"], 0, "force_final",
                                         workspace=gw.view(torch.uint8, (gw.n,)))
    L = rlat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], 0, "force_final")
    losses, grads = rb.rnnt_lattice_loss(z, L, pb["logit_lens"], pb["target_lens"])
    torch.cuda.synchronize()
    assert gz.intact() and gw.intact()
    ref_l, _ = oracle.batch(pb["logits"].numpy(), pb["targets"], pb["logit_lens"], pb["target_lens"], 0,
                            "force_final", grad=False)
    assert np.allclose(losses.cpu().numpy(), ref_l, rtol=1e-5)
    assert np.isfinite(best.cpu().numpy()).all()


def test_canaries_fused_joint_forward_and_training_step(rb):
    """K6 / K6<grad> / K7 / cuBLAS: every input and output buffer of the fused joint between NaN canaries."""
    from oracle import joint as oj
    B, T, U, H, V = 3, 26, 9, 256, 500
    cfg = workloads.random_config(B, T, U, V, seed=75, variant="force_final")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, bias = workloads.joint_inputs(B, T, U, H, V, seed=75)

    def guarded_copy(x):
        g = Guarded(x.numel() * x.element_size())
        v = g.view(x.dtype, tuple(x.shape))
        v.copy_(x.cuda())
        return g, v

    ge, e = guarded_copy(enc)
    gp, p = guarded_copy(pred)
    gw, w = guarded_copy(W)
    gb, b = guarded_copy(bias)
    outs_g = [Guarded(4 * n) for n in (B, B * T * H, B * (U + 1) * H, V * H, V)]
    shapes = [(B,), (B, T, H), (B, U + 1, H), (V, H), (V,)]
    outs = tuple(g.view(torch.float32, sh) for g, sh in zip(outs_g, shapes))
    ws = Guarded(int(rb.library.rnnt_joint_grad_workspace_bytes(B, T, U, H, V)))
    out = rb.rnnt_joint_loss_grad(e, p, w, b, y, T_b, U_b, 0, "force_final", outputs=outs,
                                  workspace=ws.view(torch.uint8, (ws.n,)))
    lf = Guarded(4 * B)
    l = rb.rnnt_joint_loss(e, p, w, b, y, T_b, U_b, 0, "force_final", losses=lf.view(torch.float32, (B,)),
                           workspace=ws.view(torch.uint8, (ws.n,)))
    torch.cuda.synchronize()
    for g in (ge, gp, gw, gb, ws, lf, *outs_g):
        assert g.intact()
    ref = oj.joint_loss_and_grads(enc.double().numpy(), pred.double().numpy(), W.double().numpy(),
                                  bias.double().numpy(), y, T_b, U_b, 0, "force_final")
    bnd = oj.r23_bounds(enc.double().numpy(), pred.double().numpy(), W.double().numpy(), bias.double().numpy(),
                        y, T_b, U_b, 0, "force_final")
    assert np.allclose(l.cpu().numpy(), ref[0], rtol=1e-5) and np.allclose(out[0].cpu().numpy(), ref[0], rtol=1e-5)
    for mine, r, k in zip(out[1:], ref[1:], ("d_f", "d_g", "d_W", "d_bias")):
        assert (np.abs(mine.cpu().numpy().astype(np.float64) - r) <= bnd[k]).all(), k
