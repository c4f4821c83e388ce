"""Compose-Transducer lattices for the generic acyclic-lattice engine (rnnt_lattice_loss).

PAPER.md §2.2 Eq.(3): L(X, Y) = Populate(S_time(X) o S_unit(Y), X) -- the lattice is the composition of
a temporal schema and a unit schema, whose auxiliary labels (time index, unit index) survive the composition
and select, with the input label, the log-probability X[t, u, label] of every arc (Fig. 3).  §3.2
P:112-118 (Fig. 5): the W-Transducer as W-Compose-Transducer -- skip-frame connections added to both schemas
with two distinct input labels, so that initial and final skips stay distinguishable in S_time^w.

Host-side graph construction (as k2's compose on the CPU side of the paper's pipeline); the result is packed
with ``lattice.from_arcs`` and scored by the same GPU kernels as any other lattice.  Schemas (reading of the
figures, whose drawings are missing from PAPER.md; reading R24):

  S_time (states 0..T): blank arcs t -> t+1 (time index t) for t < T; for every non-blank label, a self-loop at
      t < T (time index t); final state T.  W: <skip_init> arcs 0 -> t for t in [1, T-1]; <skip_final> arcs
      t -> T-1 (force-final) or t -> T (allow-ignore) for t in [0, T-2].
  S_unit (states 0..U): a blank self-loop at every u (unit index u); the label arc u -> u+1 on y_{u+1} (unit
      index u); final state U.  W: a <skip_init> self-loop at 0 and a <skip_final> self-loop at U.
  Composition matches input labels (both schemas are epsilon-free: every arc consumes its label on both
  sides), product state (t, u); start (0, 0); final (T, U).  Skip arcs are structural (probability one).
"""
from __future__ import annotations

import dataclasses
from collections import defaultdict

from .lattice import LatticeBatch, from_arcs

SKIP_INIT = -2   # input labels of the skip-frame connections (not vocabulary entries)
SKIP_FINAL = -3


@dataclasses.dataclass
class Fsa:
    """An acyclic FSA: states 0..num_states-1, start 0; arcs (src, dst, ilabel, aux); finals."""
    num_states: int
    arcs: list
    finals: set


def s_time(T: int, V: int, blank: int, variant: str = "rnnt") -> Fsa:
    """Temporal schema (aux = time index)."""
    arcs = [(t, t + 1, blank, t) for t in range(T)]
    for t in range(T):
        arcs += [(t, t, v, t) for v in range(V) if v != blank]
    if variant != "rnnt":
        arcs += [(0, t, SKIP_INIT, 0) for t in range(1, T)]
        end = T - 1 if variant == "force_final" else T
        arcs += [(t, end, SKIP_FINAL, t) for t in range(T - 1)]
    return Fsa(T + 1, arcs, {T})


class TimeSchema:
    """S_time without materialising its T x (V-1) label self-loops: arcs_from(t, label) answers the
    composition's queries directly (same arcs as s_time)."""

    def __init__(self, T: int, V: int, blank: int, variant: str = "rnnt"):
        self.T, self.V, self.blank, self.variant = T, V, blank, variant

    def arcs_from(self, t: int, lab: int):
        T = self.T
        if lab == self.blank:
            return [(t + 1, t)] if t < T else []
        if 0 <= lab < self.V:
            return [(t, t)] if t < T else []
        if self.variant == "rnnt":
            return []
        if lab == SKIP_INIT:
            return [(d, 0) for d in range(1, T)] if t == 0 else []
        if lab == SKIP_FINAL:
            return [(T - 1 if self.variant == "force_final" else T, t)] if t < T - 1 else []
        return []


def s_unit(y, blank: int, variant: str = "rnnt") -> Fsa:
    """Unit schema, A_rnnt with unit indices (aux = unit index)."""
    U = len(y)
    arcs = [(u, u, blank, u) for u in range(U + 1)]
    arcs += [(u, u + 1, int(y[u]), u) for u in range(U)]
    if variant != "rnnt":
        arcs += [(0, 0, SKIP_INIT, 0), (U, U, SKIP_FINAL, U)]
    return Fsa(U + 1, arcs, {U})


def compose(a: Fsa, b: Fsa):
    """Composition on input labels (a: an Fsa or an object answering arcs_from(state, label)), from the start
    pair (0, 0) over reachable pairs; self-loops on both sides
    match too (an arc that stays in one component moves in the other).  Returns (pairs, arcs) with arcs
    (src_pair, dst_pair, ilabel, aux_a, aux_b), pairs in discovery order.  Loops of the product (a self-loop
    on both sides) would make it cyclic; the schemas have none (every product arc advances t or u)."""
    if hasattr(a, "arcs_from"):
        arcs_a = a.arcs_from
    else:
        out_a = defaultdict(lambda: defaultdict(list))
        for (s, d, lab, aux) in a.arcs:
            out_a[s][lab].append((d, aux))
        arcs_a = lambda st, lab: out_a[st].get(lab, ())
    out_b = defaultdict(list)
    for (s, d, lab, aux) in b.arcs:
        out_b[s].append((d, lab, aux))
    pairs = {(0, 0): 0}
    order = [(0, 0)]
    arcs = []
    i = 0
    while i < len(order):
        pa, pb = order[i]
        i += 1
        for (db, lab, auxb) in out_b[pb]:
            for (da, auxa) in arcs_a(pa, lab):
                if (da, db) == (pa, pb):
                    raise ValueError("cyclic composition")
                if (da, db) not in pairs:
                    pairs[(da, db)] = len(order)
                    order.append((da, db))
                arcs.append(((pa, pb), (da, db), lab, auxa, auxb))
    return order, arcs


def compose_lattice(T: int, y, V: int, blank: int, variant: str = "rnnt"):
    """One Compose-Transducer lattice in from_arcs' format (levels, arcs, final): the composition, states
    renumbered level by level (level = longest path from the start; all arcs go to a higher level), every arc
    Populated with its (time, unit, label) binding -- or structural (v = -1) for the skips."""
    pairs, arcs = compose(TimeSchema(T, V, blank, variant), s_unit(y, blank, variant))
    # longest-path levels over the (acyclic) product, in a topological order (Kahn)
    idx = {p: k for k, p in enumerate(pairs)}
    n = len(pairs)
    indeg = [0] * n
    succ = defaultdict(list)
    for (s, d, *_r) in arcs:
        indeg[idx[d]] += 1
        succ[idx[s]].append(idx[d])
    level = [0] * n
    stack = [k for k in range(n) if indeg[k] == 0]
    while stack:
        k = stack.pop()
        for d in succ[k]:
            level[d] = max(level[d], level[k] + 1)
            indeg[d] -= 1
            if indeg[d] == 0:
                stack.append(d)
    nlev = max(level) + 1
    by_level = [[] for _ in range(nlev)]
    for k in range(n):
        by_level[level[k]].append(k)
    new_id = {}
    for lv in by_level:
        for k in lv:
            new_id[k] = len(new_id)
    out = []
    for (s, d, lab, t, u) in arcs:
        v = lab if lab >= 0 else -1
        out.append((new_id[idx[s]], new_id[idx[d]], t, u, v))
    U = len(y)
    final = {new_id[idx[(T, U)]]: 0.0} if (T, U) in idx else {}
    return [len(lv) for lv in by_level], out, final


def compose_lattices(T_b, U_b, targets, V: int, blank: int, variant: str = "rnnt") -> LatticeBatch:
    """A LatticeBatch of Compose-Transducer lattices for a padded batch."""
    return from_arcs([compose_lattice(int(T), [int(v) for v in targets[b][:int(U)]], V, blank, variant)
                      for b, (T, U) in enumerate(zip(T_b, U_b))])
