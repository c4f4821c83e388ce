"""GPU parity for 16-bit logits / grads (§4.2: the lattice is
populated from a half-precision tensor and the scores are computed in fp32/fp64).

The oracle receives the 16-bit logits widened to fp32 exactly (fp16 and bf16 are subsets of fp32), so the
loss bar is unchanged (1e-5 relative).  Grads are stored in the 16-bit type, rounded to nearest from the
fp32 result, so the grad bar becomes 1e-4 + (one ulp of the storage type) * |g|: 2^-8 |g| for bf16 (8
significant bits), 2^-10 |g| for fp16 (11 bits) -- DESIGN.md reading R20."""
import numpy as np
import pytest
import torch

import oracle
import workloads

pytestmark = pytest.mark.gpu

VARIANTS = ("rnnt", "force_final", "allow_ignore")
REL_ULP = {torch.bfloat16: 2.0 ** -8, torch.float16: 2.0 ** -10}


@pytest.fixture(scope="module")
def rb():
    import paper_2303_10384_b200
    return paper_2303_10384_b200


def _threads():
    import os
    return max(1, len(os.sched_getaffinity(0)))


def _check(rb, pb, variant, dtype, z16=None, grads=True):
    z16 = pb["logits"].to(dtype).cuda() if z16 is None else z16
    z_exact = z16.float().cpu().numpy()              # exact widening: the values the GPU path sees
    ref_l, ref_g = oracle.batch(z_exact, pb["targets"], pb["logit_lens"], pb["target_lens"], pb["blank"],
                                variant, nthreads=_threads())
    l, g = rb.loss(z16, pb["targets"], pb["logit_lens"], pb["target_lens"], pb["blank"], variant, grads=grads)
    torch.cuda.synchronize()
    l = l.cpu().numpy().astype(np.float64)
    rel = np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)
    assert rel.max() <= 1e-5, rel.max()
    if grads is not False:
        assert g.dtype == dtype
        gg = g.float().cpu().numpy().astype(np.float64)
        bound = 1e-4 + REL_ULP[dtype] * np.abs(ref_g)
        excess = np.abs(gg - ref_g) - bound
        assert excess.max() <= 0, (excess.max(), np.abs(gg - ref_g).max())
    return l, g


SHAPES = [(3, 9, 4, 8, 0), (4, 33, 31, 136, 135), (2, 70, 40, 264, 77), (3, 41, 63, 1024, 999), (6, 5, 2, 16, 1),
          (3, 40, 17, 500, 0), (2, 13, 6, 12, 11)]  # the last two: V % 8 == 4 (64-bit vector path; P:124 V = 500)


@pytest.mark.parametrize("dtype", (torch.bfloat16, torch.float16), ids=("bf16", "fp16"))
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: "B{}_T{}_U{}_V{}_b{}".format(*s))
@pytest.mark.parametrize("variant", VARIANTS)
def test_half_random_shapes(rb, shape, variant, dtype):
    B, T, U, V, blank = shape
    cfg = workloads.random_config(B, T, U, V, seed=sum(shape) + 1, blank=blank, variant=variant)
    _check(rb, workloads.problem(cfg), variant, dtype)


@pytest.mark.parametrize("dtype", (torch.bfloat16, torch.float16), ids=("bf16", "fp16"))
def test_half_scalar_path_and_padding(rb, dtype):
    """V not a multiple of 8 and a misaligned base force the scalar path; NaN padding is never read."""
    cfg = workloads.random_config(3, 30, 9, 130, seed=21)
    pb = workloads.problem(cfg, pad_value=float("nan"))
    _check(rb, pb, "rnnt", dtype)
    cfg = workloads.random_config(3, 30, 9, 136, seed=22, variant="force_final")
    pb = workloads.problem(cfg)
    flat = torch.empty(pb["logits"].numel() + 1, dtype=dtype, device="cuda")
    z = flat[1:].view(pb["logits"].shape)
    z.copy_(pb["logits"].to(dtype).cuda())
    _check(rb, pb, "force_final", dtype, z16=z)


def test_bf16_c3_full_size_sampled_in_place(rb):
    cfg = workloads.CONFIGS["c3"]
    pb = workloads.problem(cfg, device="cuda")
    z = pb["logits"].to(torch.bfloat16)
    del pb["logits"]
    torch.cuda.empty_cache()
    sample = [0, 31]
    zs = z[sample].float().cpu().numpy()
    l, g = rb.loss(z, pb["targets"], pb["logit_lens"], pb["target_lens"], cfg.blank, "rnnt", grads="inplace")
    torch.cuda.synchronize()
    ref_l, ref_g = oracle.batch(zs, pb["targets"][sample], pb["logit_lens"][sample], pb["target_lens"][sample],
                                cfg.blank, "rnnt", nthreads=_threads())
    lc = l.cpu().numpy().astype(np.float64)[sample]
    assert (np.abs(lc - ref_l) / np.abs(ref_l)).max() <= 1e-5
    gg = g[sample].float().cpu().numpy().astype(np.float64)
    assert (np.abs(gg - ref_g) - (1e-4 + 2.0 ** -8 * np.abs(ref_g))).max() <= 0


def test_half_loss_equals_fp32_loss_on_widened_input(rb):
    """The storage type changes nothing but the reads: bf16 logits and their exact fp32 widening give
    bit-identical losses."""
    cfg = workloads.random_config(4, 60, 20, 512, seed=23)
    pb = workloads.problem(cfg)
    z16 = pb["logits"].to(torch.bfloat16).cuda()
    l16, _ = rb.loss(z16, pb["targets"], pb["logit_lens"], pb["target_lens"], 0, "rnnt", grads=False)
    l32, _ = rb.loss(z16.float(), pb["targets"], pb["logit_lens"], pb["target_lens"], 0, "rnnt", grads=False)
    torch.cuda.synchronize()
    assert torch.equal(l16, l32)


@pytest.mark.parametrize("dtype", (torch.bfloat16, torch.float16), ids=("bf16", "fp16"))
@pytest.mark.parametrize("blank", (0, 3, 496, 499))
def test_half_v8_4_piece_and_alignment(rb, dtype, blank):
    """V % 8 == 4 rows (P:124's V = 500, 64-bit vectors): rows alternate between 16-byte aligned starts and
    starts 8 bytes past one; blank and labels at both row ends; logits based 16-byte aligned and 8 bytes past it;
    grads new, in place, and preallocated at the other alignment mod 16."""
    B, T, U, V = 3, 21, 9, 500
    cfg = workloads.random_config(B, T, U, V, seed=blank + 31, blank=blank)
    pb = workloads.problem(cfg)
    # labels on the piece positions too (a label never equals the blank)
    tg = pb["targets"].copy()
    for k, y in enumerate((0, 1, 2, 3, 496, 497, 498, 499)):
        if y != blank:
            tg[:, k % U] = y
    pb["targets"] = tg
    for off in (0, 4):  # elements: 0 -> 16-byte aligned base, 4 -> 8 bytes past
        flat = torch.empty(pb["logits"].numel() + 8, dtype=dtype, device="cuda")
        z = flat[off:off + pb["logits"].numel()].view(pb["logits"].shape)
        z.copy_(pb["logits"].to(dtype).cuda())
        _check(rb, pb, "rnnt", dtype, z16=z)
        zi = z.clone() if off == 0 else flat.clone()[off:off + z.numel()].view(z.shape)
        _check(rb, pb, "rnnt", dtype, z16=zi, grads="inplace")
        gflat = torch.empty(z.numel() + 8, dtype=dtype, device="cuda")
        gout = gflat[4 - off:4 - off + z.numel()].view(z.shape)  # the other alignment mod 16
        _, g = _check(rb, pb, "rnnt", dtype, z16=z, grads=gout)
        assert g.data_ptr() == gout.data_ptr()
