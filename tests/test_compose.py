"""Compose-Transducer lattices (§2.2 Eq.(3), §3.2 Fig.5; paper_2303_10384_b200/compose.py) scored by the
generic lattice oracle and, on the GPU, by the generic lattice engine: the composition route must give the
Grid-Transducer's losses and gradients (the paper: "numerical equivalence", P:80 / P:116)."""
import math

import numpy as np
import pytest
import torch

import oracle
import workloads
from oracle import lattice_fb as lf
from paper_2303_10384_b200 import compose as cmp

VARIANTS = ("rnnt", "force_final", "allow_ignore")


@pytest.mark.parametrize("variant", VARIANTS)
def test_fig1_toy_uniform_probabilities(variant):
    """Fig.1 toy with uniform logits: P = 5/2048, 229/2048, 697/2048 (path enumeration)."""
    T, y, V = 4, [1, 3], 4
    levels, arcs, final = cmp.compose_lattice(T, y, V, 0, variant)
    z = np.zeros((T, 3, V))
    want = {"rnnt": 5 / 2048, "force_final": 229 / 2048, "allow_ignore": 697 / 2048}[variant]
    assert abs(lf.enumerate_loss(z, sum(levels), arcs, final) + math.log(want)) < 1e-12
    l, *_ = lf.lattice_loss_and_grad(z, sum(levels), arcs, final)
    assert abs(l + math.log(want)) < 1e-12


@pytest.mark.parametrize("variant", VARIANTS)
def test_compose_matches_grid_oracle(variant):
    rng = np.random.default_rng(5)
    for T, U, V in ((1, 0, 3), (2, 1, 3), (5, 3, 6), (7, 0, 4), (6, 4, 9)):
        y = [int(v) for v in rng.integers(1, V, size=U)]
        z = rng.standard_normal((T, U + 1, V))
        levels, arcs, final = cmp.compose_lattice(T, y, V, 0, variant)
        l, g, *_ = lf.lattice_loss_and_grad(z, sum(levels), arcs, final)
        ref_l, ref_g = oracle.batch(z[None].astype(np.float32), np.array(y, np.int32).reshape(1, U), [T], [U], 0, variant)
        assert abs(l - ref_l[0]) <= 1e-5 * max(1.0, abs(ref_l[0])), (T, U, l, ref_l[0])
        assert np.abs(g - ref_g[0]).max() <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("variant", VARIANTS)
def test_compose_lattices_on_gpu_engine(variant):
    import paper_2303_10384_b200 as rb
    cfg = workloads.random_config(3, 24, 7, 16, seed=41, variant=variant)
    pb = workloads.problem(cfg)
    L = cmp.compose_lattices(pb["logit_lens"], pb["target_lens"], pb["targets"], cfg.V, 0, variant)
    losses, grads = rb.rnnt_lattice_loss(pb["logits"].cuda(), L, pb["logit_lens"], pb["target_lens"])
    torch.cuda.synchronize()
    ref_l, ref_g = oracle.batch(pb["logits"].numpy(), pb["targets"], pb["logit_lens"], pb["target_lens"], 0, variant)
    l = losses.cpu().numpy().astype(np.float64)
    assert (np.abs(l - ref_l) / np.maximum(np.abs(ref_l), 1.0)).max() <= 1e-5
    assert np.abs(grads.cpu().numpy() - ref_g).max() <= 1e-4


@pytest.mark.parametrize("variant", VARIANTS)
def test_lazy_time_schema_equals_explicit(variant):
    """compose() with the explicit S_time FSA and with the lazy TimeSchema build the same lattice."""
    T, y, V = 6, [2, 1, 3], 5
    a = cmp.compose(cmp.s_time(T, V, 0, variant), cmp.s_unit(y, 0, variant))
    b = cmp.compose(cmp.TimeSchema(T, V, 0, variant), cmp.s_unit(y, 0, variant))
    assert a[0] == b[0] and sorted(a[1]) == sorted(b[1])
