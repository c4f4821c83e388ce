"""Host-side lattice construction for the generic acyclic-lattice engine (rnnt_lattice_loss; SURVEY §8(f)
NEXT-3): the paper's extensibility thesis -- new losses are new graphs, not new kernels (§1 P:27,
§2.2, §3.2).

A ``LatticeBatch`` is the flat, GPU-ready arc-list form the C ABI takes: states of every lattice numbered in
topological *levels* (all arcs go from a lower level to a higher one; the states of a level are contiguous),
arcs sorted by destination (in-CSR) plus an out-CSR permutation, each arc bound to (t, u, v) of the utterance's
logits or structural (v = -1, weight 0), and a log final weight per state.

``grid_lattices`` builds the Grid-Transducer lattices (§2.3) and their W-Transducer extensions
(§3.2, §4.3) in this form with vectorised numpy -- levels are the anti-diagonals t + u and
the final state F sits one level past (T-1, U).  ``from_arcs`` packs arbitrary per-utterance arc lists.
"""
from __future__ import annotations

import dataclasses

import numpy as np


@dataclasses.dataclass
class LatticeBatch:
    state_off: np.ndarray   # [B+1]   states of lattice b: [state_off[b], state_off[b+1])
    lvl_off: np.ndarray     # [B+1]   levels of lattice b: [lvl_off[b], lvl_off[b+1]) into level_off
    level_off: np.ndarray   # [L+1]   states of level k: [level_off[k], level_off[k+1])
    in_off: np.ndarray      # [S+1]   arcs into state s: [in_off[s], in_off[s+1]) (arcs sorted by dst)
    out_off: np.ndarray     # [S+1]   out_arc[out_off[s]:out_off[s+1]] = arcs leaving s
    out_arc: np.ndarray     # [A]
    arc_src: np.ndarray     # [A]     global state ids
    arc_dst: np.ndarray     # [A]
    arc_t: np.ndarray       # [A]     binding into logits[b, t, u, v]; v = -1: structural arc, weight 0
    arc_u: np.ndarray       # [A]
    arc_v: np.ndarray       # [A]
    final_w: np.ndarray     # [S]     float32 log final weight, -inf = not final

    @property
    def B(self):
        return len(self.state_off) - 1

    @property
    def num_states(self):
        return int(self.state_off[-1])

    @property
    def num_arcs(self):
        return len(self.arc_src)

    def arcs_of(self, b):
        """Per-utterance arc list (local state ids) in the oracle's format: (src, dst, t, u, v)."""
        s0 = int(self.state_off[b])
        a0, a1 = int(self.in_off[s0]), int(self.in_off[self.state_off[b + 1]])
        return [(int(self.arc_src[i]) - s0, int(self.arc_dst[i]) - s0, int(self.arc_t[i]), int(self.arc_u[i]),
                 int(self.arc_v[i])) for i in range(a0, a1)]

    def row_index(self, Tmax: int, Umax: int):
        """(row_off [B*Tmax*(Umax+1) + 1], row_arc): the arcs bound to logits row (b, t, u), row index
        (b*Tmax + t)*(Umax+1) + u, in arc order -- lets the engine form each row's gradient in one pass."""
        Up1 = Umax + 1
        b_of_state = np.repeat(np.arange(self.B), np.diff(self.state_off))
        b = b_of_state[self.arc_src]
        bound = self.arc_v >= 0
        rows = (b.astype(np.int64) * Tmax + self.arc_t) * Up1 + self.arc_u
        arcs = np.nonzero(bound)[0]
        order = np.argsort(rows[arcs], kind="stable")
        row_arc = arcs[order].astype(np.int32)
        counts = np.bincount(rows[arcs], minlength=self.B * Tmax * Up1)
        row_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
        return row_off, row_arc

    def final_of(self, b):
        s0, s1 = int(self.state_off[b]), int(self.state_off[b + 1])
        return {s - s0: float(self.final_w[s]) for s in range(s0, s1) if np.isfinite(self.final_w[s])}


def from_arcs(lattices):
    """Pack per-utterance lattices [(levels, arcs, final)] into a LatticeBatch.

    levels: list of state-count per level (states numbered level by level); arcs: list of (src, dst, t, u, v)
    with level(src) < level(dst); final: {state: log weight}.
    """
    state_off, lvl_off, level_off = [0], [0], [0]
    A = []
    finals = []
    for (levels, arcs, final) in lattices:
        s0 = state_off[-1]
        n = int(sum(levels))
        for c in levels:
            level_off.append(level_off[-1] + int(c))
        lvl_off.append(lvl_off[-1] + len(levels))
        state_off.append(s0 + n)
        fw = np.full(n, -np.inf, np.float32)
        for s, wv in final.items():
            fw[s] = wv
        finals.append(fw)
        for (s, d, t, u, v) in arcs:
            A.append((s0 + s, s0 + d, t, u, v))
    A = np.asarray(A, np.int64).reshape(-1, 5)
    order = np.lexsort((A[:, 0], A[:, 1]))  # by dst, then src
    A = A[order]
    S = state_off[-1]
    in_off = np.zeros(S + 1, np.int64)
    np.add.at(in_off, A[:, 1] + 1, 1)
    in_off = np.cumsum(in_off)
    out_arc = np.argsort(A[:, 0], kind="stable")
    out_off = np.zeros(S + 1, np.int64)
    np.add.at(out_off, A[:, 0] + 1, 1)
    out_off = np.cumsum(out_off)
    i32 = lambda x: np.ascontiguousarray(x, np.int32)
    return LatticeBatch(i32(state_off), i32(lvl_off), i32(level_off), i32(in_off), i32(out_off), i32(out_arc),
                        i32(A[:, 0]), i32(A[:, 1]), i32(A[:, 2]), i32(A[:, 3]), i32(A[:, 4]),
                        np.concatenate(finals) if finals else np.zeros(0, np.float32))


def grid_lattice(T, U, y, blank, variant="rnnt"):
    """One Grid-Transducer lattice (levels, arcs, final) in anti-diagonal level order (§2.3).

    Cell (t,u) lives at level t+u; F at level T+U.  Arcs: blank (t,u)->(t+1,u) bound (t,u,blank); label
    (t,u)->(t,u+1) bound (t,u,y[u]); terminating blank (T-1,U)->F bound (T-1,U,blank).  W (§3.2 P:106-116,
    §4.3): structural initial skips (0,0)->(t,0), t in [1,T-1]; final skips from (t,U), t in [0,T-2],
    to (T-1,U) (force-final) or to F (allow-ignore).
    """
    D = T + U  # levels 0..D-1 hold cells, level D holds F
    d = np.arange(D)
    lo = np.maximum(0, d - (T - 1))
    hi = np.minimum(d, U)
    counts = hi - lo + 1
    first = np.concatenate([[0], np.cumsum(counts)])

    def sid(t, u):  # vectorised state id of cell (t,u)
        dd = t + u
        return first[dd] + (u - lo[dd])

    F = int(first[D])
    levels = list(counts) + [1]
    tt, uu = np.meshgrid(np.arange(T), np.arange(U + 1), indexing="ij")
    tt, uu = tt.ravel(), uu.ravel()
    arcs = []
    m = tt < T - 1  # blank arcs
    arcs.append(np.stack([sid(tt[m], uu[m]), sid(tt[m] + 1, uu[m]), tt[m], uu[m], np.full(m.sum(), blank)], 1))
    m = uu < U      # label arcs
    yy = np.asarray(y, np.int64)[uu[m]] if U > 0 else np.zeros(0, np.int64)
    arcs.append(np.stack([sid(tt[m], uu[m]), sid(tt[m], uu[m] + 1), tt[m], uu[m], yy], 1))
    arcs.append(np.array([[sid(T - 1, U), F, T - 1, U, blank]]))
    if variant != "rnnt" and T > 1:
        ts = np.arange(1, T)
        arcs.append(np.stack([np.full(T - 1, sid(0, 0)), sid(ts, np.zeros_like(ts)), ts * 0, ts * 0,
                              np.full(T - 1, -1)], 1))
        ts = np.arange(0, T - 1)
        dst = np.full(T - 1, sid(T - 1, U)) if variant == "force_final" else np.full(T - 1, F)
        arcs.append(np.stack([sid(ts, np.full_like(ts, U)), dst, ts * 0, ts * 0, np.full(T - 1, -1)], 1))
    arcs = np.concatenate(arcs).astype(np.int64)
    return levels, [tuple(int(x) for x in a) for a in arcs], {F: 0.0}


def grid_lattices(T_b, U_b, targets, blank, variant="rnnt"):
    """A LatticeBatch of grid (or W-grid) lattices for a padded batch."""
    return from_arcs([grid_lattice(int(T), int(U), targets[b][:int(U)], blank, variant)
                      for b, (T, U) in enumerate(zip(T_b, U_b))])
