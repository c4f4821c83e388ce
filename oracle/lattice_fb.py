"""Oracle for the generic acyclic-lattice loss: forward-backward over an explicit arc list.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  PAPER.md Eq.(1) P:54-56 (loss = negative forward score
of the lattice), §2.2 Eq.(3) P:82-88 (the lattice arcs are populated by indexed selection from the
log-probabilities tensor X = log_softmax(logits)), SPEC S:227-275 (forward / backward scores, arc
posteriors, gradient scatter).  Plain float64 loops in topological order; no blocking, no levels.

A lattice is given as plain Python / numpy data:
  num_states, arcs = list of (src, dst, t, u, v) with src < dst (topological numbering, state 0 = start),
  v < 0 marks a structural arc of weight 0, final = {state: log final weight}.
"""
from __future__ import annotations

import math

import numpy as np


def log_softmax_rows(z):
    """X = log_softmax(z) over the last axis, float64."""
    z = np.asarray(z, np.float64)
    m = z.max(axis=-1, keepdims=True)
    m = np.where(np.isfinite(m), m, 0.0)
    with np.errstate(divide="ignore"):
        return z - (m + np.log(np.exp(z - m).sum(axis=-1, keepdims=True)))


def _lse(values):
    vals = [v for v in values if v != -math.inf]
    if not vals:
        return -math.inf
    m = max(vals)
    return m + math.log(math.fsum(math.exp(v - m) for v in vals))


def lattice_loss_and_grad(z, num_states, arcs, final):
    """z: one utterance's logits [Tmax, Umax+1, V].  Returns (loss, d loss / d z, alpha, beta, occ per arc).

    alpha(0) = 0, alpha(s) = LSE over arcs a into s of alpha(src) + w(a)
    beta(s)  = LSE( final(s), LSE over arcs a out of s of w(a) + beta(dst) )
    log P = beta(0);  occ(a) = exp(alpha(src) + w(a) + beta(dst) - log P)
    d loss / d X[t,u,v] = - sum of occ over arcs bound to (t,u,v)
    d loss / d z[t,u,:] = dX - softmax(z[t,u,:]) * sum(dX)                        (chain rule, reading R8)
    """
    X = log_softmax_rows(z)
    w = [0.0 if v < 0 else float(X[t, u, v]) for (_, _, t, u, v) in arcs]
    incoming = [[] for _ in range(num_states)]
    outgoing = [[] for _ in range(num_states)]
    for i, (s, d, *_rest) in enumerate(arcs):
        assert s < d, "arcs must go forward in the state numbering"
        incoming[d].append(i)
        outgoing[s].append(i)
    alpha = [-math.inf] * num_states
    alpha[0] = 0.0
    for s in range(1, num_states):
        alpha[s] = _lse(alpha[arcs[i][0]] + w[i] for i in incoming[s])
    beta = [-math.inf] * num_states
    for s in range(num_states - 1, -1, -1):
        terms = [w[i] + beta[arcs[i][1]] for i in outgoing[s]]
        if s in final:
            terms.append(final[s])
        beta[s] = _lse(terms)
    logP = beta[0]
    grad = np.zeros(np.shape(z), np.float64)
    occ = [0.0] * len(arcs)
    if logP == -math.inf:
        return math.inf, grad, alpha, beta, occ
    dX = np.zeros(np.shape(z), np.float64)
    for i, (s, d, t, u, v) in enumerate(arcs):
        occ[i] = math.exp(alpha[s] + w[i] + beta[d] - logP) if alpha[s] != -math.inf and beta[d] != -math.inf else 0.0
        if v >= 0:
            dX[t, u, v] -= occ[i]
    rows = {(t, u) for (_, _, t, u, v) in arcs if v >= 0}
    for (t, u) in rows:
        p = np.exp(X[t, u])
        grad[t, u] = dX[t, u] - p * dX[t, u].sum()
    return -logP, grad, alpha, beta, occ


def enumerate_loss(z, num_states, arcs, final):
    """-log of the plain sum over all start -> final paths of the product of arc probabilities (brute force)."""
    X = log_softmax_rows(z)
    out = [[] for _ in range(num_states)]
    for (s, d, t, u, v) in arcs:
        out[s].append((d, 1.0 if v < 0 else math.exp(X[t, u, v])))
    total = 0.0

    def walk(s, p):
        nonlocal total
        if s in final:
            total += p * math.exp(final[s])
        for d, q in out[s]:
            walk(d, p * q)

    walk(0, 1.0)
    return -math.log(total) if total > 0 else math.inf
