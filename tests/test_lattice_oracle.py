"""Pins for the generic acyclic-lattice oracle (oracle/lattice_fb.py, NEXT-3) -- CPU only.

* on the Grid-/W-Transducer lattices built by the product's vectorised builder (paper_2303_10384_b200/lattice.py),
  it equals the grid oracle (rnnt_oracle.c), which is itself pinned to path enumeration: this pins both the
  generic forward-backward and the builder;
* on random level-structured DAGs it equals exhaustive path enumeration (loss) and central finite
  differences (grads).
"""
import importlib.util
import math
import os

import numpy as np
import pytest

import oracle
from oracle import lattice_fb as lf

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lattice_module():
    spec = importlib.util.spec_from_file_location("rnnt_lattice", os.path.join(ROOT, "paper_2303_10384_b200",
                                                                               "lattice.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)  # host-side graph construction only: no CUDA library needed
    return mod


lat = _lattice_module()


def random_dag(rng, T, U, V, n_levels, width, p_struct=0.2, p_arc=0.5):
    """A random level-structured lattice: arcs only to higher levels, bindings to random live rows."""
    levels = [1] + [int(rng.integers(1, width + 1)) for _ in range(n_levels - 1)]
    first = np.concatenate([[0], np.cumsum(levels)])
    arcs = []
    for li in range(n_levels - 1):
        for s in range(first[li], first[li + 1]):
            for lj in range(li + 1, min(n_levels, li + 3)):
                for d in range(first[lj], first[lj + 1]):
                    if rng.random() < p_arc:
                        v = -1 if rng.random() < p_struct else int(rng.integers(0, V))
                        arcs.append((s, d, int(rng.integers(0, T)), int(rng.integers(0, U + 1)), v))
    final = {int(s): float(rng.normal()) for s in range(first[-2], first[-1])}
    return levels, arcs, final


@pytest.mark.parametrize("variant", ("rnnt", "force_final", "allow_ignore"))
def test_generic_oracle_on_grid_lattice_equals_grid_oracle(variant):
    rng = np.random.default_rng(51)
    for _ in range(40):
        T, U, V = int(rng.integers(1, 8)), int(rng.integers(0, 6)), int(rng.integers(2, 7))
        blank = int(rng.integers(0, V))
        z = (rng.standard_normal((T + 1, U + 2, V)) * 2).astype(np.float32)
        y = [int(c) for c in rng.choice([v for v in range(V) if v != blank], size=U)] if U else []
        levels, arcs, final = lat.grid_lattice(T, U, y, blank, variant)
        L, g, *_ = lf.lattice_loss_and_grad(z, sum(levels), arcs, final)
        r = oracle.utterance(z, T, U, y, blank, variant)
        assert abs(L - r["loss"]) <= 1e-12 * max(1, abs(L))
        assert np.abs(g - r["grad"]).max() <= 1e-12


def test_generic_oracle_random_dags_enumeration_and_fd():
    rng = np.random.default_rng(52)
    h = 2.0 ** -10
    for it in range(25):
        T, U, V = int(rng.integers(1, 4)), int(rng.integers(0, 3)), int(rng.integers(2, 5))
        levels, arcs, final = random_dag(rng, T, U, V, int(rng.integers(2, 6)), 3)
        z = rng.standard_normal((T, U + 1, V)).astype(np.float32)
        L, g, *_ = lf.lattice_loss_and_grad(z, sum(levels), arcs, final)
        E = lf.enumerate_loss(z, sum(levels), arcs, final)
        if math.isinf(E):
            assert math.isinf(L)
            continue
        assert abs(L - E) <= 1e-12 * max(1, abs(E))
        if it % 5 == 0:
            for idx in np.ndindex(z.shape):
                zp, zm = z.copy(), z.copy()
                zp[idx] += np.float32(h)
                zm[idx] -= np.float32(h)
                fd = (lf.lattice_loss_and_grad(zp, sum(levels), arcs, final)[0] -
                      lf.lattice_loss_and_grad(zm, sum(levels), arcs, final)[0]) / (float(zp[idx]) - float(zm[idx]))
                assert abs(fd - g[idx]) < 2e-6


def test_builder_batch_packing_roundtrip():
    """from_arcs packing: per-lattice arcs / finals come back unchanged (up to dst-sorted order)."""
    rng = np.random.default_rng(53)
    lats = [random_dag(rng, 3, 2, 4, 4, 3) for _ in range(3)] + [lat.grid_lattice(3, 2, [1, 2], 0, "force_final")]
    batch = lat.from_arcs(lats)
    for b, (levels, arcs, final) in enumerate(lats):
        assert sorted(batch.arcs_of(b)) == sorted(arcs)
        assert batch.final_of(b) == pytest.approx(final)
        d = np.asarray([a[1] for a in batch.arcs_of(b)])
        assert (np.diff(d) >= 0).all()
