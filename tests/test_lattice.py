"""GPU parity for the generic acyclic-lattice engine (rnnt_lattice_loss, NEXT-3) vs the oracles: the grid
oracle on Grid-/W-Transducer lattices, the generic oracle (oracle/lattice_fb.py, pinned in
tests/test_lattice_oracle.py) on random level-structured DAGs.  Bars as the grid path: loss 1e-5 relative,
grads 1e-4 absolute."""
import numpy as np
import pytest
import torch

import oracle
import workloads
from oracle import lattice_fb as lf

pytestmark = pytest.mark.gpu
VARIANTS = ("rnnt", "force_final", "allow_ignore")


@pytest.fixture(scope="module")
def rb():
    import paper_2303_10384_b200
    return paper_2303_10384_b200


@pytest.fixture(scope="module")
def lat():
    from paper_2303_10384_b200 import lattice
    return lattice


def _close(l, g, ref_l, ref_g):
    rel = np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)
    assert rel.max() <= 1e-5, rel.max()
    assert np.abs(g - ref_g).max() <= 1e-4, np.abs(g - ref_g).max()


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("shape", [(3, 9, 4, 8, 0), (4, 40, 20, 100, 7), (2, 60, 40, 256, 255)],
                         ids=lambda s: "B{}_T{}_U{}_V{}_b{}".format(*s))
def test_grid_lattices_match_grid_oracle(rb, lat, shape, variant):
    B, T, U, V, blank = shape
    cfg = workloads.random_config(B, T, U, V, seed=sum(shape) + 11, blank=blank, variant=variant)
    pb = workloads.problem(cfg)
    L = lat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], blank, variant)
    losses, grads = rb.rnnt_lattice_loss(pb["logits"].cuda(), L, pb["logit_lens"], pb["target_lens"])
    torch.cuda.synchronize()
    ref_l, ref_g = oracle.batch(pb["logits"].numpy(), pb["targets"], pb["logit_lens"], pb["target_lens"], blank,
                                variant)
    _close(losses.cpu().numpy().astype(np.float64), grads.cpu().numpy(), ref_l, ref_g)


def test_random_dags_match_generic_oracle(rb, lat):
    from tests.test_lattice_oracle import random_dag
    rng = np.random.default_rng(61)
    B, Tmax, Umax, V = 5, 4, 3, 6
    lats = [random_dag(rng, Tmax, Umax, V, int(rng.integers(3, 9)), 4) for _ in range(B)]
    z = rng.standard_normal((B, Tmax, Umax + 1, V)).astype(np.float32)
    L = lat.from_arcs(lats)
    T_b = np.full(B, Tmax, np.int32)
    U_b = np.full(B, Umax, np.int32)
    losses, grads = rb.rnnt_lattice_loss(torch.from_numpy(z).cuda(), L, T_b, U_b)
    torch.cuda.synchronize()
    ref_l, ref_g = [], []
    for b, (levels, arcs, final) in enumerate(lats):
        l_, g_, *_ = lf.lattice_loss_and_grad(z[b], sum(levels), arcs, final)
        ref_l.append(l_)
        ref_g.append(g_)
    ref_l = np.asarray(ref_l)
    l = losses.cpu().numpy().astype(np.float64)
    fin = np.isfinite(ref_l)
    assert np.array_equal(np.isfinite(l), fin)
    _close(l[fin], grads.cpu().numpy()[fin], ref_l[fin], np.asarray(ref_g)[fin])


def test_generic_engine_agrees_with_grid_kernels_in_place(rb, lat):
    """Same lattice two ways on the GPU: the generic engine (in place) and the specialised grid path."""
    cfg = workloads.random_config(4, 80, 30, 512, seed=62, variant="allow_ignore")
    pb = workloads.problem(cfg)
    L = lat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], 0, "allow_ignore")
    z = pb["logits"].cuda()
    l_grid, g_grid = rb.wrnnt_loss(z, pb["targets"], pb["logit_lens"], pb["target_lens"], 0, "allow_ignore")
    l_gen, g_gen = rb.rnnt_lattice_loss(z, L, pb["logit_lens"], pb["target_lens"], grads="inplace")
    torch.cuda.synchronize()
    assert torch.allclose(l_gen, l_grid, rtol=1e-5, atol=0)
    assert (g_gen - g_grid).abs().max().item() < 1e-4


@pytest.mark.parametrize("variant", ("force_final", "allow_ignore"))
@pytest.mark.parametrize("shape", [(3, 300, 64, 512), (2, 40, 600, 16), (1, 8200, 2, 8)],
                         ids=["ring_overflow_chunked", "wide_levels", "uncached_levels"])
def test_engine_schedule_paths(rb, lat, shape, variant):
    """L3's less common paths: neighbours older than the shared-memory ring (W skips across > 16384 states)
    with the chunk-overlapped schedule (>= 2^24 elements), levels wider than a CTA (strided), and more levels
    than the cached level table; the W skip states also take the warp-cooperative (> 2 arcs) branch."""
    B, T, U, V = shape
    cfg = workloads.random_config(B, T, U, V, seed=T + U + 5, variant=variant, variable=False)
    pb = workloads.problem(cfg)
    L = lat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], 0, variant)
    losses, grads = rb.rnnt_lattice_loss(pb["logits"].cuda(), L, pb["logit_lens"], pb["target_lens"])
    torch.cuda.synchronize()
    ref_l, ref_g = oracle.batch(pb["logits"].numpy(), pb["targets"], pb["logit_lens"], pb["target_lens"], 0,
                                variant)
    _close(losses.cpu().numpy().astype(np.float64), grads.cpu().numpy(), ref_l, ref_g)


def test_row_index_path_is_deterministic_and_matches_atomic_path(rb, lat):
    """The row-index gradient pass (no atomics) equals the float-atomic passes and repeats bit for bit."""
    cfg = workloads.random_config(3, 50, 17, 200, seed=63, variant="force_final")
    pb = workloads.problem(cfg)
    L = lat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], 0, "force_final")
    z = pb["logits"].cuda()
    B, Tmax, Up1, V = z.shape
    d_rows = rb.lattice_to_device(L, "cuda", Tmax, Up1 - 1)
    d_atom = rb.lattice_to_device(L, "cuda")
    l1, g1 = rb.rnnt_lattice_loss(z, d_rows, pb["logit_lens"], pb["target_lens"])
    l2, g2 = rb.rnnt_lattice_loss(z, d_rows, pb["logit_lens"], pb["target_lens"])
    l3, g3 = rb.rnnt_lattice_loss(z, d_atom, pb["logit_lens"], pb["target_lens"])
    torch.cuda.synchronize()
    assert torch.equal(g1, g2) and torch.equal(l1, l2)
    assert torch.equal(l1, l3)
    assert (g1 - g3).abs().max().item() <= 1e-6


@pytest.mark.parametrize("variant", VARIANTS)
def test_nan_logit_gives_nan_loss(rb, lat, variant):
    """A NaN logit in a valid cell of utterance 1 gives it a NaN loss and zero gradients (R12), as on
    the grid path; the other utterances are bit-identical to the run without it."""
    cfg = workloads.random_config(3, 20, 8, 64, seed=7, variant=variant, variable=False)
    pb = workloads.problem(cfg)
    L = lat.grid_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], 0, variant)
    z = pb["logits"].clone()
    z[1, 5, 3, 9] = float("nan")
    l0, g0 = rb.rnnt_lattice_loss(pb["logits"].cuda(), L, pb["logit_lens"], pb["target_lens"])
    l1, g1 = rb.rnnt_lattice_loss(z.cuda(), L, pb["logit_lens"], pb["target_lens"])
    l0, l1, g0, g1 = l0.cpu(), l1.cpu(), g0.cpu(), g1.cpu()
    assert torch.isnan(l1[1]), l1
    assert not g1[1].any()
    assert torch.equal(l1[[0, 2]], l0[[0, 2]]) and torch.equal(g1[[0, 2]], g0[[0, 2]])
