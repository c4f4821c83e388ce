"""Brute-force enumeration oracle: every alignment path of the RNN-T / W-RNNT lattice, one by one.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Independent of ``rnnt_oracle.c``: no dynamic
programming, no log-space arithmetic -- the lattice is an explicit arc list built from the paper's text
and the loss is -log of the plain sum over complete paths of the product of arc probabilities
(Eq.(1): "negative forward scores"; "marginalizing over all possible alignments").

Arc list (one state per grid node (t,u), 0<=t<T, 0<=u<=U, plus the final state "F"):
  * blank arcs  (t,u)->(t+1,u), t<T-1, probability p[t,u,blank]       §2.3 P:92 "every horizontal arc is <blank>"
  * label arcs  (t,u)->(t,u+1), u<U,   probability p[t,u,y[u]]        §2.3 P:92 "each column of arcs is the same"
  * terminating blank (T-1,U)->F,      probability p[T-1,U,blank]     S:373 (grid_lattice)
  * W initial skips (0,0)->(t,0), 1<=t<=T-1, probability one           §3.2
  * force-final skips (t,U)->(T-1,U), 0<=t<=T-2, probability one       §3.2 P:108, P:116 ("previous-to-final state")
  * allow-ignore skips (t,U)->F, 0<=t<=T-2, probability one            §4.3 P:167 ("point to the final state")
where p[t,u,:] = softmax(z[t,u,:]) (§2.1, "log-probabilities tensor").

Parallel arcs (e.g. a blank arc and a skip arc between the same two states) are distinct paths.
"""
from __future__ import annotations

import math
from fractions import Fraction

FINAL = "F"


def lattice_arcs(T, U, variant="rnnt"):
    """Explicit arc list: tuples (src, dst, label) with label ('blank', t, u) | ('label', t, u) |
    ('skip', 'initial', t_dst) | ('skip', 'final', t_src)."""
    arcs = []
    for t in range(T):
        for u in range(U + 1):
            if t + 1 < T:
                arcs.append(((t, u), (t + 1, u), ("blank", t, u)))
            if u < U:
                arcs.append(((t, u), (t, u + 1), ("label", t, u)))
    arcs.append(((T - 1, U), FINAL, ("blank", T - 1, U)))
    if variant != "rnnt":
        for t in range(1, T):
            arcs.append(((0, 0), (t, 0), ("skip", "initial", t)))
        for t in range(0, T - 1):
            if variant == "force_final":
                arcs.append(((t, U), (T - 1, U), ("skip", "final", t)))
            elif variant == "allow_ignore":
                arcs.append(((t, U), FINAL, ("skip", "final", t)))
            else:
                raise ValueError(variant)
    return arcs


def enumerate_paths(T, U, variant="rnnt"):
    """All start->final paths, each a tuple of arc labels (depth-first, exhaustive)."""
    out_arcs = {}
    for src, dst, lab in lattice_arcs(T, U, variant):
        out_arcs.setdefault(src, []).append((dst, lab))
    paths = []

    def walk(state, acc):
        if state == FINAL:
            paths.append(tuple(acc))
            return
        for dst, lab in out_arcs.get(state, []):
            acc.append(lab)
            walk(dst, acc)
            acc.pop()

    walk((0, 0), [])
    return paths


def _arc_vocab_index(lab, y, blank):
    return blank if lab[0] == "blank" else y[lab[2]]


def total_probability(probs, y, T, U, blank=0, variant="rnnt"):
    """P = sum over paths of prod of arc probabilities.  ``probs[t][u][v]`` may hold Fractions (exact)."""
    total = 0
    for path in enumerate_paths(T, U, variant):
        w = 1
        for lab in path:
            if lab[0] != "skip":
                w = w * probs[lab[1]][lab[2]][_arc_vocab_index(lab, y, blank)]
        total = total + w
    return total


def uniform_probs(T, U, V):
    """Exact softmax of all-equal logits: every entry is 1/V."""
    return [[[Fraction(1, V)] * V for _ in range(U + 1)] for _ in range(T)]


def softmax_rows(z, T, U):
    """Plain softmax of each logits row in double (math.exp), rows t<T, u<=U of z[Tmax][Umax+1][V]."""
    probs = []
    for t in range(T):
        rows = []
        for u in range(U + 1):
            row = [float(x) for x in z[t][u]]
            m = max(row)
            e = [math.exp(x - m) for x in row]
            s = math.fsum(e)
            rows.append([x / s for x in e])
        probs.append(rows)
    return probs


def loss_and_grad(z, y, T, U, blank=0, variant="rnnt"):
    """Loss -log P and d loss / d z by direct enumeration (float64).

    The gradient uses the product rule path by path: d log p[t,u,k] / d z[t,u,j] = [k==j] - p[t,u,j], so
    d(-log P)/d z[t,u,j] = -(1/P) sum_paths P_path * sum_{scored arcs of the path at (t,u)} ([k==j] - p[t,u,j]).
    Returns (loss, grad as nested lists [T][U+1][V], occ_b [T][U+1], occ_y [T][U+1], npaths).
    """
    V = len(z[0][0])
    p = softmax_rows(z, T, U)
    paths = enumerate_paths(T, U, variant)
    weights = []
    for path in paths:
        w = 1.0
        for lab in path:
            if lab[0] != "skip":
                w *= p[lab[1]][lab[2]][_arc_vocab_index(lab, y, blank)]
        weights.append(w)
    P = math.fsum(weights)
    grad = [[[0.0] * V for _ in range(U + 1)] for _ in range(T)]
    occ_b = [[0.0] * (U + 1) for _ in range(T)]
    occ_y = [[0.0] * (U + 1) for _ in range(T)]
    if P == 0.0:
        return math.inf, grad, occ_b, occ_y, len(paths)
    for path, w in zip(paths, weights):
        r = w / P
        for lab in path:
            if lab[0] == "skip":
                continue
            t, u = lab[1], lab[2]
            k = _arc_vocab_index(lab, y, blank)
            if lab[0] == "blank":
                occ_b[t][u] += r
            else:
                occ_y[t][u] += r
            g = grad[t][u]
            pr = p[t][u]
            for j in range(V):
                g[j] -= r * ((1.0 if j == k else 0.0) - pr[j])
    return -math.log(P), grad, occ_b, occ_y, len(paths)


def best_path(z, y, T, U, blank=0, variant="rnnt"):
    """Viterbi by enumeration: the complete path with the largest sum of arc log-probabilities (float64).

    Returns (best score, frames [U] (emission frame of each unit), span (first, last covered frame),
    gap to the second-best path score).  The span starts at t0 if the path enters column 0 through the
    initial skip (0,0)->(t0,0) and ends at t* if it leaves row U through a final skip from (t*,U).
    """
    p = softmax_rows(z, T, U)
    scored = []
    for path in enumerate_paths(T, U, variant):
        s = 0.0
        for lab in path:
            if lab[0] != "skip":
                pr = p[lab[1]][lab[2]][_arc_vocab_index(lab, y, blank)]
                s += math.log(pr) if pr > 0 else -math.inf
        scored.append((s, path))
    scored.sort(key=lambda x: -x[0])
    s0, path = scored[0]
    gap = s0 - scored[1][0] if len(scored) > 1 else math.inf
    frames = [-1] * U
    start, end = 0, T - 1
    for lab in path:
        if lab[0] == "label":
            frames[lab[2]] = lab[1]
        elif lab[0] == "skip" and lab[1] == "initial":
            start = lab[2]
        elif lab[0] == "skip" and lab[1] == "final":
            end = lab[2]
    return s0, frames, (start, end), gap
