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


GRADS = ("d_enc", "d_pred", "d_weight", "d_bias")
_ORACLE = {"d_enc": "d_f", "d_pred": "d_g", "d_weight": "d_W", "d_bias": "d_bias"}


def _np(*ts):
    return [None if t is None else t.double().numpy() for t in ts]


def assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, blank, variant, scales=None, tag=""):
    """GPU training-step gradients vs the exact chain rule of R22's bf16 forward graph (oracle rounding=
    "forward", pinned to torch float64 autograd), elementwise within R23's derived bound (oracle/joint.py
    r23_bounds).  scales: optional per-utterance grad_scale (the reference is then sum_b s_b ref_b, the bound
    sum_b |s_b| bound_b).  Returns the worst err / bound per tensor (the margin; < 1 passes)."""
    args = _np(enc, pred, W, b)
    if scales is None:
        ref = oj.joint_loss_and_grads(*args, y, T_b, U_b, blank, variant)
        bnd = oj.r23_bounds(*args, y, T_b, U_b, blank, variant)
        refs, bnds = ref[1:], [bnd[_ORACLE[n]] for n in GRADS]
    else:
        B = len(scales)
        refs = [0.0] * 4
        bnds = [0.0] * 4
        for i in range(B):
            a = [None if x is None else x[i:i + 1] for x in args[:2]] + args[2:]
            r = oj.joint_loss_and_grads(*a, y[i:i + 1], T_b[i:i + 1], U_b[i:i + 1], blank, variant)
            bd = oj.r23_bounds(*a, y[i:i + 1], T_b[i:i + 1], U_b[i:i + 1], blank, variant)
            s = float(scales[i])
            for k, n in enumerate(GRADS):
                rr, bb = r[1 + k], bd[_ORACLE[n]]
                if k < 2:   # per-utterance tensors: place utterance i
                    full = np.zeros((B,) + rr.shape[1:]); full[i] = rr; rr = full
                    fb = np.zeros((B,) + bb.shape[1:]); fb[i] = bb; bb = fb
                refs[k] = refs[k] + s * rr
                bnds[k] = bnds[k] + abs(s) * bb
    margins = {}
    for n, mine, r, bd in zip(GRADS, out[1:], refs, bnds):
        m = mine.cpu().numpy().astype(np.float64)
        err = np.abs(m - r)
        ratio = err / np.maximum(bd, 1e-300)
        margins[n] = float(ratio.max()) if ratio.size else 0.0
        assert (err <= bd).all(), (tag, n, margins[n], float(err.max()), float(np.abs(r).max()))
    print(f"R23 margins {tag}: " + ", ".join(f"{k} {v:.3f}" for k, v in margins.items()))
    return margins


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


def test_joint_nan_input_propagates(rb):
    """A NaN in one encoder element makes the loss of exactly the utterance it belongs to NaN (R12),
    whichever of the 8 columns of a 16-byte item it sits in
    (the builders take tanh's reciprocal from MUFU for some of an item's words and from Newton steps for others:
    a clamp that dropped the NaN would give a finite, wrong loss); the other utterances' losses do not change."""
    B, T, U, H, V = 3, 12, 5, 256, 200
    cfg = workloads.random_config(B, T, U, V, seed=41, variant="rnnt", variable=False)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=41)
    ref = rb.rnnt_joint_loss(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "rnnt").cpu()
    for col in range(8):
        e = enc.clone()
        e[1, 3, 64 + col] = float("nan")
        l = rb.rnnt_joint_loss(e.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "rnnt").cpu()
        assert torch.isnan(l[1]), (col, l)
        assert torch.equal(l[[0, 2]], ref[[0, 2]]), col


def test_joint_grad_nan_input(rb):
    """The training step with a NaN in one encoder element: that utterance's loss is NaN, the other utterances'
    losses are bit-identical to the run without it."""
    B, T, U, H, V = 3, 12, 5, 256, 200
    cfg = workloads.random_config(B, T, U, V, seed=42, variant="rnnt", variable=False)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=42)
    ref = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "rnnt")[0].cpu()
    for col in (0, 7):
        e = enc.clone()
        e[1, 3, 64 + col] = float("nan")
        l = rb.rnnt_joint_loss_grad(e.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "rnnt")[0].cpu()
        assert torch.isnan(l[1]), (col, l)
        assert torch.equal(l[[0, 2]], ref[[0, 2]]), col


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
    ref_l = oj.joint_loss(*_np(enc, pred, W, b), y, T_b, U_b, 0, "force_final")
    l = out[0].cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5
    assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, 0, "force_final", tag="V8195")


@pytest.mark.parametrize("scale", [2.0, 8.0])
def test_joint_large_preactivations(rb, scale):
    """enc, pred scaled up (|f + g| up to ~6 sigma * scale: saturated tanh, h = +-1 in bf16 for large |x|):
    loss and gradients still match the oracle's bf16(tanh(f + g)) graph, within R23's bound."""
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
    ref_l = oj.joint_loss(*_np(enc, pred, W, b), y, T_b, U_b, 0, "allow_ignore")
    for losses in (l, out[0]):
        lg = losses.cpu().numpy().astype(np.float64)
        assert (np.abs(lg - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5, (lg, ref_l)
    assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, 0, "allow_ignore", tag=f"scale{scale}")


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
    """rnnt_joint_loss_grad vs the exact chain rule of R22's bf16 forward graph (oracle rounding="forward",
    pinned to torch float64 autograd).  Bars: losses 1e-5 relative; gradients elementwise within R23's derived
    bound (4u times each element's sum of absolute terms + the fp32 dz error)."""
    B, T, U, H, V = shape
    cfg = workloads.random_config(B, T, U, V, seed=sum(shape) % 89 + 7, variant=variant)
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=sum(shape) % 89 + 7)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, variant)
    torch.cuda.synchronize()
    ref_l = oj.joint_loss(*_np(enc, pred, W, b), y, T_b, U_b, 0, variant)
    l = out[0].cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5
    assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, 0, variant, tag=f"{shape} {variant}")


@pytest.mark.parametrize("shape", [(2, 11, 5, 384, 200), (3, 13, 4, 256, 37), (2, 17, 6, 512, 300),
                                   (5, 29, 9, 128, 130)],
                         ids=lambda s: "B{}_T{}_U{}_H{}_V{}".format(*s))
def test_joint_grad_backward_gemm_shapes(rb, shape):
    """The backward GEMMs' edge shapes: H = 384 (K8's N chunks 256 + 128, K9's 3 h boxes per CTA), V = 37 and
    V = 130 (one / three 128-v tiles: K9's pair with an idle odd CTA; K8's last K block partly past V), V = 300
    (Vp = 384), a row count that is not a multiple of K8's 256-row pair tile or K9's 64-row stage."""
    B, T, U, H, V = shape
    cfg = workloads.random_config(B, T, U, V, seed=sum(shape) % 83 + 5, variant="allow_ignore")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=sum(shape) % 83 + 5)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "allow_ignore")
    torch.cuda.synchronize()
    ref_l = oj.joint_loss(*_np(enc, pred, W, b), y, T_b, U_b, 0, "allow_ignore")
    l = out[0].cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5
    assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, 0, "allow_ignore", tag=f"gemm {shape}")


def test_joint_grad_many_tiles_per_cta(rb):
    """~61k valid rows (~480 row tiles, > 3 per CTA on 148 SMs): every CTA pair of K6's forward and k6_dz_2sm
    walks several row tiles, so the per-K-block A ring (h blocks refilled as the previous tile's last N tile
    frees them), the accumulator ring and the barrier phases wrap many times; Vp = 256 (2 N tiles), H = 256
    (4 K blocks)."""
    B, T, U, H, V = 40, 160, 48, 256, 130
    cfg = workloads.random_config(B, T, U, V, seed=71, variant="rnnt")
    T_b, U_b = workloads.lengths(cfg)
    assert rb.joint_valid_rows(T_b, U_b, T, U) >= 3 * 148 * 128
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=71)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "rnnt")
    torch.cuda.synchronize()
    ref_l = oj.joint_loss(*_np(enc, pred, W, b), y, T_b, U_b, 0, "rnnt")
    l = out[0].cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5
    assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, 0, "rnnt", tag="many tiles")


@pytest.mark.parametrize("env", [{"RNNT_K6_DZTMA": "0"}, {"RNNT_K6_HREUSE": "0"}, {"RNNT_K6_PAIR": "0"},
                                 {"RNNT_K8_SPLIT": "0"}],
                         ids=lambda e: ",".join(f"{k}={v}" for k, v in e.items()))
def test_joint_grad_ab_paths(rb, env, monkeypatch):
    """The training step's A/B switches (read per call) stay correct: k6_joint_lse<true> loading the forward's h into
    TMEM (DZTMA=0), recomputing h (HREUSE=0), per-CTA MMAs (PAIR=0), K8's single accumulator hand-over (SPLIT=0),
    each against the same exact chain rule (R23) as the default path."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    B, T, U, H, V = 3, 30, 10, 512, 500  # H = 512: K8's split hand-over applies
    cfg = workloads.random_config(B, T, U, V, seed=73, variant="allow_ignore")
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=73)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), y, T_b, U_b, 0, "allow_ignore")
    torch.cuda.synchronize()
    ref_l = oj.joint_loss(*_np(enc, pred, W, b), y, T_b, U_b, 0, "allow_ignore")
    l = out[0].cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5
    assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, 0, "allow_ignore", tag=f"ab {env}")


@pytest.mark.parametrize("name", ["p124", "c3"])
def test_joint_grad_full_size_properties(rb, name):
    """The training step at full size -- the paper's shapes (B = 30, T <= 433, U <= 92, V = 500) and c3's
    (B = 32, T = 500, U = 100, V = 1024), H = 512, the launch bench.py times -- checked by what holds at any size: (1) a sampled utterance's loss matches the oracle's R22 forward;
    (2) every row's dz sums to zero over v in real arithmetic (softmax mass gamma minus the two occupancies), so
    |sum_v d_bias(v)| is bounded by dz's bf16 rounding, u = 2^-8 of sum |dz| <= 2 sum_b (T_b + U_b) (each path
    scores T_b blanks and U_b labels: the occupancies sum to T_b + U_b); a dropped or mis-signed occupancy term
    would leave ~sum_b (T_b + U_b); (3) an utterance's d enc / d pred / loss from the whole batch equal bit for bit
    those of a one-utterance call (row-independent kernels, per-utterance fixed-order reductions)."""
    cfg = {**workloads.CONFIGS, **workloads.EXTRA_CONFIGS}[name]
    B, T, U, V, H = cfg.B, cfg.Tmax, cfg.Umax, cfg.V, 512
    T_b, U_b = workloads.lengths(cfg)
    y = workloads.targets(cfg, U_b)
    enc, pred, W, b = workloads.joint_inputs(B, T, U, H, V, seed=91)
    args = (W.cuda(), b.cuda())
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), *args, y, T_b, U_b, cfg.blank, "rnnt")
    torch.cuda.synchronize()
    cells = T_b.astype(np.int64) * (U_b.astype(np.int64) + 1)
    i = int(np.argmin(cells))  # the cheapest utterance for the oracle
    ref = oj.joint_loss(*_np(enc[i:i + 1], pred[i:i + 1], W, b), y[i:i + 1], T_b[i:i + 1], U_b[i:i + 1], cfg.blank,
                        "rnnt")
    l = float(out[0][i])
    assert abs(l - ref[0]) <= 1e-5 * max(abs(ref[0]), 1.0), (l, ref[0])
    db = out[4].double()
    bound = 2.0 ** -8 * 2.0 * float(np.sum(T_b.astype(np.float64) + U_b)) + 1e-3
    assert abs(float(db.sum())) <= bound, (float(db.sum()), bound)
    for j in (i, B - 1):
        o1 = rb.rnnt_joint_loss_grad(enc[j:j + 1].cuda(), pred[j:j + 1].cuda(), *args, y[j:j + 1], T_b[j:j + 1],
                                     U_b[j:j + 1], cfg.blank, "rnnt")
        torch.cuda.synchronize()
        assert torch.equal(o1[0][0], out[0][j])
        assert torch.equal(o1[1][0], out[1][j]) and torch.equal(o1[2][0], out[2][j])


def test_joint_grad_no_valid_rows(rb):
    """Every utterance invalid (T_b > Tmax): no GEMM rows at all -- NaN losses, every gradient exactly zero."""
    H, V = 128, 130
    enc, pred, W, b = workloads.joint_inputs(2, 4, 2, H, V, seed=61)
    out = rb.rnnt_joint_loss_grad(enc.cuda(), pred.cuda(), W.cuda(), b.cuda(), np.array([[1, 2], [3, 4]], np.int32),
                                  np.array([5, 9], np.int32), np.array([2, 2], np.int32), 0, "rnnt")
    torch.cuda.synchronize()
    assert torch.isnan(out[0]).all()
    for g in out[1:]:
        assert not g.any()


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
    ref_l = oj.joint_loss(*_np(enc[:2], pred[:2], W, b), y[:2], T_b[:2], U_b[:2], 0, "allow_ignore")
    lg = l.cpu().numpy().astype(np.float64)
    assert np.isnan(lg[2]) and np.isnan(out[0][2].item())
    assert (np.abs(lg[:2] - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5
    assert not out[1][2].any() and not out[2][2].any()
    # the two valid utterances' gradients; W / bias gradients get nothing from the invalid one
    assert_grads_r23((out[0][:2], out[1][:2], out[2][:2], out[3], out[4]), enc[:2], pred[:2], W, b, y[:2],
                     T_b[:2], U_b[:2], 0, "allow_ignore", tag="edge")
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
    assert not out[1][2].any()  # scale 0: no gradient into utterance 2's encoder frames
    assert_grads_r23(out, enc, pred, W, b, y, T_b, U_b, 0, "rnnt", scales=scale.numpy(), tag="grad_scale")


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
