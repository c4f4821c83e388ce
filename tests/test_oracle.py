"""Pins for the CPU oracle (oracle/rnnt_oracle.c) against things other than itself.

Each test states what it pins and which plausible oracle mistake it would catch:
  * exact enumeration (oracle/brute.py, an explicit arc list -- no DP) and the golden file it wrote;
  * values printed in SPEC.md for the worked micro-cases;
  * closed forms (uniform logits; single-path lattices U=0 / T=1);
  * finite differences of the loss (pins the gradient against the pinned loss);
  * torchaudio.functional.rnnt_loss (a library implementation of plain RNN-T, fp32);
  * invariants: alpha_final == beta_0, cut conservation, sum_v grad = 0, W orderings, row-shift invariance.
"""
import math
import os
from fractions import Fraction

import numpy as np
import pytest

import oracle
from oracle import brute

VARIANTS = ("rnnt", "force_final", "allow_ignore")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "uniform_enumeration.txt")


def _rand_instance(rng, T, U, V, blank=None, scale=1.0, pad=1):
    blank = int(rng.integers(0, V)) if blank is None else blank
    z = (rng.standard_normal((T + pad, U + 1 + pad, V)) * scale).astype(np.float32)
    choices = [v for v in range(V) if v != blank]
    y = [int(c) for c in rng.choice(choices, size=U)] if U else []
    return z, y, blank


def _golden_rows():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            body = line.split("#")[0].split()
            T, U, V = map(int, body[:3])
            y = [] if body[3] == "-" else [int(x) for x in body[3].split(",")]
            rows.append((T, U, V, y, body[4], int(body[5]), Fraction(body[6]), float(body[7])))
    return rows


# ----------------------------------------------------------------------------------------- SPEC values
def test_spec_printed_micro_cases():
    """SPEC S:253 (plain 3ln3-ln2), S:436 (force-final 8/27, 3ln3-3ln2), S:437 (allow-ignore 14/27)."""
    printed = {"rnnt": (Fraction(2, 27), 3 * math.log(3) - math.log(2)),
               "force_final": (Fraction(8, 27), 3 * math.log(3) - 3 * math.log(2)),
               "allow_ignore": (Fraction(14, 27), math.log(27 / 14))}
    for variant, (P, loss) in printed.items():
        assert brute.total_probability(brute.uniform_probs(2, 1, 3), [1], 2, 1, 0, variant) == P
        r = oracle.utterance(np.zeros((2, 2, 3), np.float32), 2, 1, [1], 0, variant)
        assert abs(r["loss"] - loss) < 1e-12


def test_spec_path_counts():
    """RNN-T grid T=4,U=2 has C(5,2)=10 paths, T=2,U=1 has 2; W force-final T=2,U=1 has 4."""
    assert len(brute.enumerate_paths(4, 2, "rnnt")) == 10
    assert len(brute.enumerate_paths(2, 1, "rnnt")) == 2
    assert len(brute.enumerate_paths(2, 1, "force_final")) == 4
    for T in range(1, 7):
        for U in range(0, 5):
            assert len(brute.enumerate_paths(T, U, "rnnt")) == math.comb(T - 1 + U, U)


# --------------------------------------------------------------------------------------- golden file
@pytest.mark.parametrize("row", _golden_rows(), ids=lambda r: f"T{r[0]}U{r[1]}V{r[2]}-{r[4]}")
def test_golden_uniform_enumeration(row):
    """The oracle's DP reproduces the exact enumerated total probability of every golden case."""
    T, U, V, y, variant, npaths, P, loss = row
    assert len(brute.enumerate_paths(T, U, variant)) == npaths
    assert brute.total_probability(brute.uniform_probs(T, U, V), y, T, U, 0, variant) == P
    r = oracle.utterance(np.zeros((T, U + 1, V), np.float32), T, U, y, 0, variant)
    assert abs(r["loss"] - (-math.log(P))) < 1e-12 * max(1.0, abs(loss))


# ------------------------------------------------------------------------------------- closed forms
@pytest.mark.parametrize("T,U,V", [(1, 0, 2), (3, 2, 5), (7, 4, 11), (20, 9, 32), (50, 20, 8)])
def test_uniform_rnnt_closed_form(T, U, V):
    """All-equal logits: every path has T+U scored arcs of probability 1/V and there are C(T-1+U,U) paths,
    so loss = (T+U) ln V - ln C(T-1+U, U)."""
    r = oracle.utterance(np.full((T, U + 1, V), 0.25, np.float32), T, U, list(range(1, U + 1)) if V > U else
                         [1] * U, 0, "rnnt")
    expect = (T + U) * math.log(V) - math.log(math.comb(T - 1 + U, U))
    assert abs(r["loss"] - expect) < 1e-10 * expect


def _log_softmax(row):
    row = np.asarray(row, np.float64)
    m = row.max()
    return row - (m + math.log(np.exp(row - m).sum()))


def test_single_path_closed_forms():
    """U=0 plain RNN-T: the only path is T blanks -> loss = -sum_t X[t,0,blank].
    T=1: the only path emits all units at t=0 then the final blank -> loss = -sum_u X[0,u,y_u] - X[0,U,blank]."""
    rng = np.random.default_rng(11)
    for _ in range(20):
        T, V = int(rng.integers(1, 9)), int(rng.integers(2, 9))
        z, _, blank = _rand_instance(rng, T, 0, V, scale=2.0)
        expect = -sum(_log_softmax(z[t, 0])[blank] for t in range(T))
        r = oracle.utterance(z, T, 0, [], blank, "rnnt")
        assert abs(r["loss"] - expect) < 1e-12 * max(1, abs(expect))
    for _ in range(20):
        U, V = int(rng.integers(0, 6)), int(rng.integers(2, 9))
        z, y, blank = _rand_instance(rng, 1, U, V, scale=2.0)
        expect = -sum(_log_softmax(z[0, u])[y[u]] for u in range(U)) - _log_softmax(z[0, U])[blank]
        for variant in VARIANTS:  # T=1 -> W skip ranges are empty
            r = oracle.utterance(z, 1, U, y, blank, variant)
            assert abs(r["loss"] - expect) < 1e-12 * max(1, abs(expect))


# ------------------------------------------------------------------------------------ brute force
def test_bruteforce_random_logits_all_variants():
    """Random logits (scale 1 and 3), random blank, padded buffers: DP loss, occupancies and logits-grads
    equal the path-by-path enumeration (catches wrong index / dropped term / transposed operand)."""
    rng = np.random.default_rng(0)
    worst = 0.0
    for it in range(150):
        T, U, V = int(rng.integers(1, 6)), int(rng.integers(0, 4)), int(rng.integers(2, 6))
        z, y, blank = _rand_instance(rng, T, U, V, scale=1.0 if it % 2 else 3.0)
        for variant in VARIANTS:
            r = oracle.utterance(z, T, U, y, blank, variant, tables=True)
            L, g, ob, oy, _ = brute.loss_and_grad(z, y, T, U, blank, variant)
            assert abs(r["loss"] - L) <= 1e-12 * max(1.0, abs(L))
            g = np.asarray(g)
            worst = max(worst, np.abs(r["grad"][:T, :U + 1] - g).max())
            assert np.abs(r["occ_b"] - np.asarray(ob)).max() < 1e-12
            assert np.abs(r["occ_y"] - np.asarray(oy)).max() < 1e-12
            # padded cells never receive gradient
            assert not r["grad"][T:].any() and not r["grad"][:, U + 1:].any()
    assert worst < 1e-12


# --------------------------------------------------------------------------------- finite differences
def test_finite_difference_gradient():
    """Central differences of the (pinned) loss match the analytic logits-gradient, all variants.
    h = 2^-10 is added exactly in fp32 for |z| < 8, and the actual step is used."""
    rng = np.random.default_rng(5)
    h = 2.0 ** -10
    for it in range(12):
        T, U, V = int(rng.integers(1, 5)), int(rng.integers(0, 4)), int(rng.integers(2, 6))
        z, y, blank = _rand_instance(rng, T, U, V, pad=0)
        for variant in VARIANTS:
            g = oracle.utterance(z, T, U, y, blank, variant)["grad"]
            for idx in np.ndindex(z.shape):
                zp, zm = z.copy(), z.copy()
                zp[idx] += np.float32(h)
                zm[idx] -= np.float32(h)
                step = float(zp[idx]) - float(zm[idx])
                fd = (oracle.utterance(zp, T, U, y, blank, variant, grad=False)["loss"]
                      - oracle.utterance(zm, T, U, y, blank, variant, grad=False)["loss"]) / step
                assert abs(fd - g[idx]) < 2e-6, (variant, idx, fd, g[idx])


# -------------------------------------------------------------------------------------- torchaudio
def test_torchaudio_rnnt_loss_crosscheck():
    """Plain RNN-T equals torchaudio.functional.rnnt_loss (library, fp32, fused log-softmax) on a batch with
    variable lengths; tolerance set by torchaudio's fp32 arithmetic."""
    import torch
    ta = pytest.importorskip("torchaudio.functional")
    rng = np.random.default_rng(3)
    B, Tmax, Umax, V, blank = 4, 30, 8, 12, 3
    z = rng.standard_normal((B, Tmax, Umax + 1, V)).astype(np.float32)
    T_b = np.array([30, 17, 5, 22], np.int32)
    U_b = np.array([8, 3, 0, 7], np.int32)
    y = np.zeros((B, Umax), np.int32)
    for b in range(B):
        y[b, :U_b[b]] = rng.choice([v for v in range(V) if v != blank], size=U_b[b])
    losses, grads = oracle.batch(z, y, T_b, U_b, blank, "rnnt")
    zt = torch.from_numpy(z).requires_grad_(True)
    lt = ta.rnnt_loss(zt, torch.from_numpy(y), torch.from_numpy(T_b), torch.from_numpy(U_b),
                      blank=blank, reduction="none")
    lt.sum().backward()
    assert np.allclose(lt.detach().numpy(), losses, rtol=2e-6, atol=0)
    assert np.abs(zt.grad.numpy() - grads).max() < 2e-5


# -------------------------------------------------------------------------------------- invariants
def test_invariants_random():
    """alpha_final == beta_0; sum_v grad = 0 per row; RNN-T blank cut sum_u occ_b(t,u) = 1
    (S:278); label cut sum_t occ_y(t,u) = 1 for every variant; W ordering AI <= FF <= RNNT."""
    rng = np.random.default_rng(21)
    for it in range(60):
        T, U, V = int(rng.integers(1, 12)), int(rng.integers(0, 7)), int(rng.integers(2, 9))
        z, y, blank = _rand_instance(rng, T, U, V, scale=2.0)
        losses = {}
        for variant in VARIANTS:
            r = oracle.utterance(z, T, U, y, blank, variant, tables=True)
            losses[variant] = r["loss"]
            assert abs(r["loss"] + r["logp_beta"]) < 1e-10 * max(1, abs(r["loss"]))
            assert np.abs(r["grad"].sum(axis=-1)).max() < 1e-12
            if U > 0:
                assert np.allclose(r["occ_y"][:, :U].sum(axis=0), 1.0, atol=1e-12, rtol=0)
            if variant == "rnnt":
                assert np.allclose(r["occ_b"].sum(axis=1), 1.0, atol=1e-12, rtol=0)
        assert losses["allow_ignore"] <= losses["force_final"] + 1e-12
        assert losses["force_final"] <= losses["rnnt"] + 1e-12


def test_row_shift_invariance():
    """Adding a constant to one logits row leaves log_softmax (hence loss and grads) unchanged.
    Values are on a 2^-10 grid so the shifted values are exact in fp32."""
    rng = np.random.default_rng(8)
    for it in range(10):
        T, U, V = int(rng.integers(1, 7)), int(rng.integers(0, 5)), int(rng.integers(2, 8))
        z, y, blank = _rand_instance(rng, T, U, V)
        z = (np.round(z * 1024) / 1024).astype(np.float32)
        zs = z + rng.integers(-16, 17, size=z.shape[:2] + (1,)).astype(np.float32)
        for variant in VARIANTS:
            a = oracle.utterance(z, T, U, y, blank, variant)
            b = oracle.utterance(zs, T, U, y, blank, variant)
            assert abs(a["loss"] - b["loss"]) < 1e-12 * max(1, abs(a["loss"]))
            assert np.abs(a["grad"] - b["grad"]).max() < 1e-12


def test_blank_permutation_equivariance():
    """Moving the blank to another vocabulary slot (and permuting logits/targets alike) changes nothing."""
    rng = np.random.default_rng(9)
    T, U, V = 6, 3, 7
    z, y, _ = _rand_instance(rng, T, U, V, blank=0)
    perm = rng.permutation(V)                      # new index of old vocab entry v is perm[v]
    zp = np.empty_like(z)
    zp[..., perm] = z
    yp = [int(perm[v]) for v in y]
    for variant in VARIANTS:
        a = oracle.utterance(z, T, U, y, 0, variant)
        b = oracle.utterance(zp, T, U, yp, int(perm[0]), variant)
        assert abs(a["loss"] - b["loss"]) < 1e-12 * abs(a["loss"])
        assert np.abs(a["grad"] - b["grad"][..., perm]).max() < 1e-12


# ---------------------------------------------------------------------------------- degenerate cases
def test_no_path_gives_inf_and_zero_grad():
    """All blank logits -inf with U=0, T>=1: no complete alignment -> loss = +inf, grads 0."""
    z = np.zeros((3, 1, 4), np.float32)
    z[..., 0] = -np.inf
    r = oracle.utterance(z, 3, 0, [], 0, "rnnt")
    assert r["loss"] == math.inf and not r["grad"].any()
    L, *_ = brute.loss_and_grad(z, [], 3, 0, 0, "rnnt")
    assert L == math.inf


def test_minus_inf_entries_match_bruteforce():
    """-inf logits forbid single arcs: blank forbidden at frame 0 forces the first unit at t=0."""
    rng = np.random.default_rng(4)
    z, y, blank = _rand_instance(rng, 3, 2, 4, blank=0, pad=0)
    z[0, 0, 0] = -np.inf
    z[1, 2, y[1]] = -np.inf
    for variant in VARIANTS:
        r = oracle.utterance(z, 3, 2, y, 0, variant)
        L, g, *_ = brute.loss_and_grad(z, y, 3, 2, 0, variant)
        assert math.isfinite(L) and abs(r["loss"] - L) < 1e-12 * max(1, abs(L))
        assert np.abs(r["grad"] - np.asarray(g)).max() < 1e-12


def test_invalid_inputs_give_nan():
    z = np.zeros((3, 3, 4), np.float32)
    assert math.isnan(oracle.utterance(z, 3, 2, [1, 0], 0, "rnnt")["loss"])   # target == blank
    assert math.isnan(oracle.utterance(z, 3, 2, [1, 4], 0, "rnnt")["loss"])   # target >= V
    assert math.isnan(oracle.utterance(z, 4, 2, [1, 2], 0, "rnnt")["loss"])   # T > Tmax
    assert math.isnan(oracle.utterance(z, 0, 2, [1, 2], 0, "rnnt")["loss"])   # T < 1


def test_padding_is_never_read():
    """NaN in every padded cell changes neither losses nor grads of the valid cells."""
    rng = np.random.default_rng(6)
    B, Tmax, Umax, V = 3, 7, 4, 5
    z = rng.standard_normal((B, Tmax, Umax + 1, V)).astype(np.float32)
    T_b, U_b = np.array([7, 3, 1], np.int32), np.array([4, 0, 2], np.int32)
    y = rng.integers(1, V, size=(B, Umax)).astype(np.int32)
    zn = z.copy()
    for b in range(B):
        zn[b, T_b[b]:] = np.nan
        zn[b, :, U_b[b] + 1:] = np.nan
    for variant in VARIANTS:
        l1, g1 = oracle.batch(z, y, T_b, U_b, 0, variant)
        l2, g2 = oracle.batch(zn, y, T_b, U_b, 0, variant, nthreads=2)
        assert np.array_equal(l1, l2) and np.array_equal(g1, g2)


# ------------------------------------------------------------------------------------------- Viterbi
def test_viterbi_matches_enumeration():
    """Max-plus DP + back-trace == the best of all enumerated paths (score, emission frames, span), on random
    instances whose best path is unique (gap > 1e-9), all variants (NEXT-2; "forced alignment")."""
    rng = np.random.default_rng(31)
    n = 0
    for it in range(200):
        T, U, V = int(rng.integers(1, 6)), int(rng.integers(0, 4)), int(rng.integers(2, 6))
        z, y, blank = _rand_instance(rng, T, U, V, scale=2.0)
        for variant in VARIANTS:
            s, f, sp = oracle.viterbi(z, T, U, y, blank, variant)
            s2, f2, sp2, gap = brute.best_path(z, y, T, U, blank, variant)
            if gap < 1e-9:
                continue
            n += 1
            assert abs(s - s2) <= 1e-12 * max(1.0, abs(s2))
            assert list(f) == f2 and tuple(sp) == sp2
    assert n > 300


def test_viterbi_bounds_closed_forms_and_ties():
    """best <= log P (a max is below the log-sum-exp) and best >= log P - log(#paths); single-path lattices
    give the path's score; all-equal logits (every path ties) resolve by the blank-first rule to emitting
    every unit at frame 0 (reading R21)."""
    rng = np.random.default_rng(32)
    for _ in range(40):
        T, U, V = int(rng.integers(1, 7)), int(rng.integers(0, 5)), int(rng.integers(2, 7))
        z, y, blank = _rand_instance(rng, T, U, V, scale=2.0)
        for variant in VARIANTS:
            s, _, _ = oracle.viterbi(z, T, U, y, blank, variant)
            logP = -oracle.utterance(z, T, U, y, blank, variant, grad=False)["loss"]
            npaths = len(brute.enumerate_paths(T, U, variant))
            assert s <= logP + 1e-12 and s >= logP - math.log(npaths) - 1e-12
    z, _, blank = _rand_instance(rng, 5, 0, 4, scale=2.0)
    s, _, sp = oracle.viterbi(z, 5, 0, [], blank, "rnnt")
    assert abs(s - sum(_log_softmax(z[t, 0])[blank] for t in range(5))) < 1e-12 and sp == (0, 4)
    z, y, blank = _rand_instance(rng, 1, 3, 6, scale=2.0)
    s, f, _ = oracle.viterbi(z, 1, 3, y, blank, "force_final")
    assert list(f) == [0, 0, 0]
    assert abs(s - (sum(_log_softmax(z[0, u])[y[u]] for u in range(3)) + _log_softmax(z[0, 3])[blank])) < 1e-12
    for T, U in ((4, 2), (6, 3), (3, 1)):
        s, f, sp = oracle.viterbi(np.zeros((T, U + 1, 5), np.float32), T, U, list(range(1, U + 1)), 0, "rnnt")
        assert list(f) == [0] * U and sp == (0, T - 1)
        assert abs(s - (T + U) * math.log(1 / 5)) < 1e-12
