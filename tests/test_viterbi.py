"""GPU parity for Viterbi forced alignment: rnnt_viterbi through the C ABI vs the
oracle's max-plus DP (itself pinned to path enumeration in tests/test_oracle.py).  Best scores within 1e-5
relative; alignments (emission frame of every unit, covered span) exactly -- unless the two alignments'
scores are within rounding of each other (a near-tie), which the test checks explicitly."""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads

pytestmark = pytest.mark.gpu
VARIANTS = ("rnnt", "force_final", "allow_ignore")


@pytest.fixture(scope="module")
def rb():
    import paper_2303_10384_b200
    return paper_2303_10384_b200


def _log_softmax(z):
    z = z.astype(np.float64)
    m = z.max(axis=-1, keepdims=True)
    return z - (m + np.log(np.exp(z - m).sum(axis=-1, keepdims=True)))


def _path_score(z, y, T, U, blank, frames, span, variant):
    """Log-weight of the alignment described by (frames, span): units emitted at their frames, blanks in
    between, skips outside the span (weight 0); a force-final skip still ends with the terminating blank."""
    X = _log_softmax(z[:T, :U + 1])
    t0, t1 = span
    s, u = 0.0, 0
    for t in range(t0, t1 + 1):
        while u < U and frames[u] == t:
            s += X[t, u, y[u]]
            u += 1
        if t < t1 or t1 == T - 1:      # blank to the next frame, or the terminating blank at T-1
            s += X[t, u, blank]
    if variant == "force_final" and t1 < T - 1:
        s += X[T - 1, U, blank]
    return s


def _check(rb, pb, variant, z_gpu=None):
    z = pb["logits"]
    zg = z.cuda() if z_gpu is None else z_gpu
    best, frames, span = rb.rnnt_viterbi(zg, pb["targets"], pb["logit_lens"], pb["target_lens"], pb["blank"],
                                         variant)
    torch.cuda.synchronize()
    best, frames, span = best.cpu().numpy(), frames.cpu().numpy(), span.cpu().numpy()
    zn = zg.float().cpu().numpy()
    for b in range(zn.shape[0]):
        T, U = int(pb["logit_lens"][b]), int(pb["target_lens"][b])
        y = list(pb["targets"][b][:U])
        s, f, sp = oracle.viterbi(zn[b], T, U, y, pb["blank"], variant)
        assert abs(best[b] - s) <= 1e-5 * max(1.0, abs(s)), (b, best[b], s)
        if list(frames[b][:U]) != list(f) or tuple(span[b]) != tuple(sp):
            # a legitimate near-tie: the GPU's alignment must score as well as the oracle's, to rounding
            sg = _path_score(zn[b], y, T, U, pb["blank"], frames[b][:U], tuple(span[b]), variant)
            assert abs(sg - s) <= 1e-6 * max(1.0, abs(s)), (b, sg, s, frames[b][:U], f, span[b], sp)
        assert (frames[b][U:] == -1).all()


SHAPES = [(3, 9, 4, 8, 0), (4, 33, 31, 129, 128), (2, 70, 40, 260, 77), (3, 41, 63, 512, 300),
          (2, 120, 200, 36, 3), (6, 5, 2, 2, 1)]


@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "B{}_T{}_U{}_V{}_b{}".format(*s))
@pytest.mark.parametrize("variant", VARIANTS)
def test_viterbi_random_shapes(rb, shape, variant):
    B, T, U, V, blank = shape
    cfg = workloads.random_config(B, T, U, V, seed=sum(shape) + 7, blank=blank, variant=variant)
    _check(rb, workloads.problem(cfg, scale=2.0), variant)


def test_viterbi_uniform_ties_and_fig1(rb):
    """All-equal logits: every path ties; blank-first resolves to every unit at frame 0 (reading R21)."""
    pb = workloads.problem(workloads.CONFIGS["c1"])
    pb["logits"].zero_()
    best, frames, span = rb.rnnt_viterbi(pb["logits"].cuda(), pb["targets"], pb["logit_lens"],
                                         pb["target_lens"], 0, "rnnt")
    torch.cuda.synchronize()
    assert frames.cpu().tolist() == [[0, 0]] and span.cpu().tolist() == [[0, 3]]
    assert abs(best.item() - 6 * math.log(1 / 4)) < 1e-5


def test_viterbi_bp_in_global_memory(rb):
    """Tmax x (Umax+1) > 200 KB: back-pointers spill from shared memory to the workspace."""
    cfg = workloads.random_config(2, 2100, 99, 16, seed=41, variable=False)
    pb = workloads.problem(cfg, scale=2.0)
    _check(rb, pb, "force_final")


def test_viterbi_bf16_and_c3_sample(rb):
    cfg = workloads.random_config(3, 60, 20, 256, seed=42)
    pb = workloads.problem(cfg, scale=2.0)
    _check(rb, pb, "allow_ignore", z_gpu=pb["logits"].to(torch.bfloat16).cuda())
    cfg = workloads.CONFIGS["c3"]
    pb = workloads.problem(cfg, b_ids=[0, 1])
    _check(rb, pb, "rnnt")


def test_viterbi_invalid_targets(rb):
    rng = np.random.default_rng(3)
    z = torch.from_numpy(rng.standard_normal((2, 5, 4, 6)).astype(np.float32)).cuda()
    best, frames, span = rb.rnnt_viterbi(z, np.array([[1, 2, 3], [1, 0, 2]], np.int32), [5, 5], [3, 3], 0, "rnnt")
    torch.cuda.synchronize()
    assert math.isfinite(best[0].item()) and math.isnan(best[1].item())
    assert (frames[1] == -1).all() and (span[1] == -1).all()


def test_viterbi_nan_logit(rb):
    """A NaN logit in a valid cell of utterance 1: NaN best score, frames and span -1 (as an invalid utterance,
    DESIGN.md R12); the other utterances' results are unchanged."""
    cfg = workloads.random_config(3, 16, 6, 40, seed=9, variable=False)
    pb = workloads.problem(cfg)
    z = pb["logits"].clone()
    z[1, 4, 2, 7] = float("nan")
    r0 = rb.rnnt_viterbi(pb["logits"].cuda(), pb["targets"], pb["logit_lens"], pb["target_lens"], 0, "rnnt")
    r1 = rb.rnnt_viterbi(z.cuda(), pb["targets"], pb["logit_lens"], pb["target_lens"], 0, "rnnt")
    (b0, f0, s0), (b1, f1, s1) = [[t.cpu() for t in r] for r in (r0, r1)]
    assert math.isnan(b1[1].item()) and (f1[1] == -1).all() and (s1[1] == -1).all()
    assert torch.equal(b1[[0, 2]], b0[[0, 2]]) and torch.equal(f1[[0, 2]], f0[[0, 2]])
    assert torch.equal(s1[[0, 2]], s0[[0, 2]])
