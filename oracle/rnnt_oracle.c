/*
 * oracle/rnnt_oracle.c -- CPU ORACLE for the RNN-T / W-RNNT loss and its gradient w.r.t. the logits.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` leg may load this library.  The product path (paper_2303_10384_b200/) never
 * links, imports or calls it, and this file shares no code, header, table or helper with csrc/.
 *
 * Plain, slow, obviously-correct double-precision implementation, written from the paper:
 *   /root/reference/PAPER.md  (cited P:<line>)   -- authority on WHAT is computed
 *   /root/reference/SPEC.md   (cited S:<line>)   -- used for the grid/W arc sets it spells out
 *
 *   Loss      Eq.(1) P:54-56  "Loss(X,Y) = -Fwd(E(X) o (T o Y(Y)))": negative forward score of the lattice.
 *   Lattice   §2.3 P:90-92    Grid-Transducer: rectangular grid, horizontal (time) arcs are <blank>,
 *                             vertical (unit) arcs emit y_{u+1}; arcs per S:373 (grid_lattice).
 *   X         §2.1 P:64       "RNN-T output log-probabilities tensor": X = log_softmax(logits) over V.
 *   Populate  §2.2 P:88       arcs get their weight by indexed selection from X.
 *   W arcs    §3.2 P:106      initial skip-frame <eps> arcs "with probability one from the initial state
 *                             to any state before non-<blank> emissions" -> (0,0)->(t,0), t in [1,T-1].
 *             §3.2 P:108,116  force-final: final skip arcs "point to the previous-to-final state"
 *                             -> (t,U)->(T-1,U), t in [0,T-2].
 *             §4.3 P:167      allow-ignore: final skip arcs "point to the final state" -> (t,U)->F,
 *                             t in [0,T-2]; the ordinary terminating blank (T-1,U)->F is kept.
 *   Gradient  chain rule of -log P through the log-softmax (reading R8): with per-arc
 *             occupancies occ(a) = exp(alpha(src)+w(a)+beta(dst)-logP),
 *             d loss / d X[t,u,v] = -sum of occ over scored arcs bound to (t,u,v) and
 *             d X[k]/d z[j] = [k==j] - softmax_j.
 *
 * Precision: double throughout (reading R11).  The fp32 logits are widened once.
 * Conventions (DESIGN.md readings): LSE of an empty set / all -inf is -inf; logP = -inf ("no path")
 * gives loss = +inf and zero grads; invalid lengths/targets give loss = NaN and zero grads;
 * cells outside t<T, u<=U get zero grads.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

enum { ORACLE_RNNT = 0, ORACLE_W_FORCE_FINAL = 1, ORACLE_W_ALLOW_IGNORE = 2 };

/* log(sum_i exp(x_i)) over n terms, max-subtracted; -inf if every term is -inf. */
static double log_sum_exp(const double *x, int n) {
    double m = -INFINITY;
    for (int i = 0; i < n; ++i)
        if (x[i] > m) m = x[i];
    if (m == -INFINITY) return -INFINITY;
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += exp(x[i] - m);
    return m + log(s);
}

/*
 * One utterance.  z: the utterance's logits block [Tmax][Umax+1][V] (fp32, row-major, V innermost).
 * y: its targets, y[u] = the (u+1)-th unit, u < U.  Outputs (each may be NULL):
 *   loss      -logP
 *   grad      [Tmax][Umax+1][V]  d loss / d z, zeros outside t<T, u<=U
 *   alpha_out, beta_out          [T][U+1] forward / backward log scores
 *   occb_out, occy_out           [T][U+1] occupancy of the blank arc leaving (t,u) / label arc leaving (t,u)
 *   logp_beta                    beta(0,0) (the backward total, for the alpha_final == beta_0 check)
 * Returns 0 on success, 1 for invalid arguments (loss = NaN, grads zero).
 */
int rnnt_oracle_utterance(const float *z, int Tmax, int Umax, int V, int T, int U, const int32_t *y,
                          int blank, int variant, double *loss, double *grad, double *alpha_out,
                          double *beta_out, double *occb_out, double *occy_out, double *logp_beta) {
    const int64_t Up1max = (int64_t)Umax + 1;
    if (grad) memset(grad, 0, sizeof(double) * (size_t)Tmax * (size_t)Up1max * (size_t)V);
    int bad = (T < 1 || T > Tmax || U < 0 || U > Umax || V < 2 || blank < 0 || blank >= V ||
               variant < 0 || variant > 2);
    for (int u = 0; !bad && u < U; ++u)
        if (y[u] < 0 || y[u] >= V || y[u] == blank) bad = 1;
    if (bad) {
        if (loss) *loss = NAN;
        if (logp_beta) *logp_beta = NAN;
        return 1;
    }
    const int W = (variant != ORACLE_RNNT);
    const int Up1 = U + 1;
#define CELL(t, u) ((size_t)(t) * (size_t)Up1 + (size_t)(u))
#define ZROW(t, u) (z + ((int64_t)(t) * Up1max + (u)) * (int64_t)V)
    double *lse = malloc(sizeof(double) * (size_t)T * Up1);
    double *lpb = malloc(sizeof(double) * (size_t)T * Up1); /* X[t,u,blank]          */
    double *lpy = malloc(sizeof(double) * (size_t)T * Up1); /* X[t,u,y_{u+1}], u < U */
    double *alpha = malloc(sizeof(double) * (size_t)T * Up1);
    double *beta = malloc(sizeof(double) * (size_t)T * Up1);
    double *occb = malloc(sizeof(double) * (size_t)T * Up1);
    double *occy = malloc(sizeof(double) * (size_t)T * Up1);
    double *terms = malloc(sizeof(double) * (size_t)(T + 4));

    /* Step 1 (§2.1, §2.2): X = log_softmax(z) over V, then Populate = indexed selection. */
    for (int t = 0; t < T; ++t)
        for (int u = 0; u <= U; ++u) {
            const float *row = ZROW(t, u);
            double m = -INFINITY;
            for (int v = 0; v < V; ++v)
                if ((double)row[v] > m) m = (double)row[v];
            double l = -INFINITY;
            if (m != -INFINITY) {
                double s = 0.0;
                for (int v = 0; v < V; ++v) s += exp((double)row[v] - m);
                l = m + log(s);
            }
            lse[CELL(t, u)] = l;
            /* an all -inf row forbids its arcs (reading R12) */
            lpb[CELL(t, u)] = (l == -INFINITY) ? -INFINITY : (double)row[blank] - l;
            lpy[CELL(t, u)] = (u < U && l != -INFINITY) ? (double)row[y[u]] - l : -INFINITY;
        }

    /* Step 2: forward scores alpha over the lattice, t-major order (a topological order of the grid;
     * S:227-235).  Incoming arcs of (t,u):
     *   blank arc  (t-1,u) -> (t,u)   weight X[t-1,u,blank]                    (§2.3)
     *   label arc  (t,u-1) -> (t,u)   weight X[t,u-1,y_u]                      (§2.3)
     *   W initial skip (0,0) -> (t,0), t>=1, weight 0                          (§3.2)
     *   force-final skip (t',U) -> (T-1,U), t' <= T-2, weight 0                (§3.2) */
    for (int t = 0; t < T; ++t)
        for (int u = 0; u <= U; ++u) {
            if (t == 0 && u == 0) {
                alpha[CELL(0, 0)] = 0.0;
                continue;
            }
            int n = 0;
            if (t >= 1) terms[n++] = alpha[CELL(t - 1, u)] + lpb[CELL(t - 1, u)];
            if (u >= 1) terms[n++] = alpha[CELL(t, u - 1)] + lpy[CELL(t, u - 1)];
            if (W && u == 0 && t >= 1) terms[n++] = alpha[CELL(0, 0)] + 0.0;
            if (variant == ORACLE_W_FORCE_FINAL && u == U && t == T - 1)
                for (int tp = 0; tp <= T - 2; ++tp) terms[n++] = alpha[CELL(tp, U)] + 0.0;
            alpha[CELL(t, u)] = log_sum_exp(terms, n);
        }

    /* Step 3: total score logP = alpha(F) (Eq.(1) "Fwd").  Arcs into F:
     *   terminating blank (T-1,U) -> F, weight X[T-1,U,blank]
     *   allow-ignore skips (t',U) -> F, t' <= T-2, weight 0       (§4.3) */
    double logP;
    {
        int n = 0;
        terms[n++] = alpha[CELL(T - 1, U)] + lpb[CELL(T - 1, U)];
        if (variant == ORACLE_W_ALLOW_IGNORE)
            for (int tp = 0; tp <= T - 2; ++tp) terms[n++] = alpha[CELL(tp, U)] + 0.0;
        logP = log_sum_exp(terms, n);
    }

    /* Step 4: backward scores beta(s) = LSE over outgoing arcs of (w + beta(dst)), beta(F) = 0
     * (S:237-245), reverse t-major order.  Outgoing arcs of (t,u): the mirror of step 2/3. */
    for (int t = T - 1; t >= 0; --t)
        for (int u = U; u >= 0; --u) {
            int n = 0;
            if (t == T - 1 && u == U) terms[n++] = lpb[CELL(t, u)] + 0.0; /* -> F */
            if (t <= T - 2) terms[n++] = lpb[CELL(t, u)] + beta[CELL(t + 1, u)];
            if (u <= U - 1) terms[n++] = lpy[CELL(t, u)] + beta[CELL(t, u + 1)];
            if (variant == ORACLE_W_FORCE_FINAL && u == U && t <= T - 2)
                terms[n++] = 0.0 + beta[CELL(T - 1, U)];
            if (variant == ORACLE_W_ALLOW_IGNORE && u == U && t <= T - 2) terms[n++] = 0.0 + 0.0;
            if (W && t == 0 && u == 0)
                for (int tp = 1; tp <= T - 1; ++tp) terms[n++] = 0.0 + beta[CELL(tp, 0)];
            beta[CELL(t, u)] = log_sum_exp(terms, n);
        }

    /* Step 5: occupancies of the scored arcs; skip arcs are structural, carry no binding. */
    const int nopath = (logP == -INFINITY);
    for (int t = 0; t < T; ++t)
        for (int u = 0; u <= U; ++u) {
            double ob = 0.0, oy = 0.0;
            if (!nopath) {
                if (t <= T - 2)
                    ob = exp(alpha[CELL(t, u)] + lpb[CELL(t, u)] + beta[CELL(t + 1, u)] - logP);
                else if (u == U)
                    ob = exp(alpha[CELL(t, u)] + lpb[CELL(t, u)] + 0.0 - logP); /* terminating blank */
                if (u <= U - 1)
                    oy = exp(alpha[CELL(t, u)] + lpy[CELL(t, u)] + beta[CELL(t, u + 1)] - logP);
            }
            occb[CELL(t, u)] = ob;
            occy[CELL(t, u)] = oy;
        }

    /* Step 6: d loss / d z.  dX[v] = -(occ of the arcs bound to (t,u,v)); chain rule through
     * X = z - lse(z): d loss/d z_j = dX_j - softmax_j * sum_k dX_k. */
    if (grad && !nopath) {
        double *dX = malloc(sizeof(double) * (size_t)V);
        for (int t = 0; t < T; ++t)
            for (int u = 0; u <= U; ++u) {
                const double l = lse[CELL(t, u)];
                if (l == -INFINITY) continue; /* forbidden row: no arc carries mass */
                for (int v = 0; v < V; ++v) dX[v] = 0.0;
                dX[blank] -= occb[CELL(t, u)];
                if (u < U) dX[y[u]] -= occy[CELL(t, u)];
                double sum_dX = 0.0;
                for (int v = 0; v < V; ++v) sum_dX += dX[v];
                const float *row = ZROW(t, u);
                double *g = grad + ((int64_t)t * Up1max + u) * (int64_t)V;
                for (int v = 0; v < V; ++v) g[v] = dX[v] - exp((double)row[v] - l) * sum_dX;
            }
        free(dX);
    }

    if (loss) *loss = -logP;
    if (logp_beta) *logp_beta = beta[CELL(0, 0)];
    if (alpha_out) memcpy(alpha_out, alpha, sizeof(double) * (size_t)T * Up1);
    if (beta_out) memcpy(beta_out, beta, sizeof(double) * (size_t)T * Up1);
    if (occb_out) memcpy(occb_out, occb, sizeof(double) * (size_t)T * Up1);
    if (occy_out) memcpy(occy_out, occy, sizeof(double) * (size_t)T * Up1);
    free(lse); free(lpb); free(lpy); free(alpha); free(beta); free(occb); free(occy); free(terms);
#undef CELL
#undef ZROW
    return 0;
}

/*
 * A padded batch: z [B][Tmax][Umax+1][V] fp32, y [B][Umax] int32, T_b/U_b [B] int32.
 * losses [B] double; grads [B][Tmax][Umax+1][V] double or NULL.  Utterances are independent
 * ("Batch items are embarrassingly parallel"); nthreads > 0 runs them on that many OpenMP threads.
 * Returns the number of invalid utterances.
 */
int rnnt_oracle_batch(const float *z, const int32_t *y, const int32_t *T_b, const int32_t *U_b, int B,
                      int Tmax, int Umax, int V, int blank, int variant, double *losses, double *grads,
                      int nthreads) {
    const int64_t ustride = (int64_t)Tmax * ((int64_t)Umax + 1) * (int64_t)V;
    int nbad = 0;
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads) reduction(+ : nbad)
    for (int b = 0; b < B; ++b) {
        nbad += rnnt_oracle_utterance(z + b * ustride, Tmax, Umax, V, T_b[b], U_b[b],
                                      y + (int64_t)b * Umax, blank, variant, &losses[b],
                                      grads ? grads + b * ustride : NULL, NULL, NULL, NULL, NULL, NULL);
    }
    return nbad;
}

int rnnt_oracle_max_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * Viterbi forced alignment over the same lattice (§2.1: the lattice serves "model training
 * and forced alignment tasks").  Max-plus instead of log-sum-exp:
 *   delta(0,0) = 0;  delta(t,u) = max over incoming arcs of (delta(src) + w(arc))      (same arc set as above)
 * Ties are broken in a fixed order (reading R21): blank (time) arc, then label arc, then skip arc;
 * among final skips the earliest source frame.  Outputs (each may be NULL):
 *   best        max over complete paths of the summed log-weights
 *   frames[u]   frame t at which unit u (0-based) is emitted on the best path, u < U
 *   span[0..1]  first and last frame the best path covers with scored arcs: the frame it enters column 0
 *               (after an initial skip, else 0) and the frame it leaves row U (before a final skip, else T-1)
 * Returns 0, or 1 for invalid arguments (best = NaN).  A lattice with no finite path gives best = -inf and
 * frames / span = -1.
 */
enum { BP_BLANK = 0, BP_LABEL = 1, BP_SKIP = 2 };

int rnnt_oracle_viterbi(const float *z, int Tmax, int Umax, int V, int T, int U, const int32_t *y, int blank,
                        int variant, double *best, int32_t *frames, int32_t *span) {
    const int64_t Up1max = (int64_t)Umax + 1;
    int bad = (T < 1 || T > Tmax || U < 0 || U > Umax || V < 2 || blank < 0 || blank >= V ||
               variant < 0 || variant > 2);
    for (int u = 0; !bad && u < U; ++u)
        if (y[u] < 0 || y[u] >= V || y[u] == blank) bad = 1;
    if (frames)
        for (int u = 0; u < U && u < Umax; ++u) frames[u] = -1;
    if (span) span[0] = span[1] = -1;
    if (bad) {
        if (best) *best = NAN;
        return 1;
    }
    const int W = (variant != ORACLE_RNNT);
    const int Up1 = U + 1;
#define CELL(t, u) ((size_t)(t) * (size_t)Up1 + (size_t)(u))
#define ZROW(t, u) (z + ((int64_t)(t) * Up1max + (u)) * (int64_t)V)
    double *lpb = malloc(sizeof(double) * (size_t)T * Up1);
    double *lpy = malloc(sizeof(double) * (size_t)T * Up1);
    double *delta = malloc(sizeof(double) * (size_t)T * Up1);
    unsigned char *bp = malloc((size_t)T * Up1);

    /* log-softmax + Populate, exactly as in rnnt_oracle_utterance */
    for (int t = 0; t < T; ++t)
        for (int u = 0; u <= U; ++u) {
            const float *row = ZROW(t, u);
            double m = -INFINITY;
            for (int v = 0; v < V; ++v)
                if ((double)row[v] > m) m = (double)row[v];
            double l = -INFINITY;
            if (m != -INFINITY) {
                double s = 0.0;
                for (int v = 0; v < V; ++v) s += exp((double)row[v] - m);
                l = m + log(s);
            }
            lpb[CELL(t, u)] = (l == -INFINITY) ? -INFINITY : (double)row[blank] - l;
            lpy[CELL(t, u)] = (u < U && l != -INFINITY) ? (double)row[y[u]] - l : -INFINITY;
        }

    /* max-plus forward pass, t-major; candidate order = tie-break order (strict '>' keeps the first) */
    for (int t = 0; t < T; ++t)
        for (int u = 0; u <= U; ++u) {
            if (t == 0 && u == 0) {
                delta[CELL(0, 0)] = 0.0;
                bp[CELL(0, 0)] = BP_BLANK;
                continue;
            }
            double d = -INFINITY;
            unsigned char from = BP_BLANK;
            if (t >= 1) {
                d = delta[CELL(t - 1, u)] + lpb[CELL(t - 1, u)];
                from = BP_BLANK;
            }
            if (u >= 1) {
                const double c = delta[CELL(t, u - 1)] + lpy[CELL(t, u - 1)];
                if (c > d || (d == -INFINITY && t < 1)) {
                    d = c;
                    from = BP_LABEL;
                }
            }
            if (W && u == 0 && t >= 1) {
                const double c = delta[CELL(0, 0)] + 0.0; /* initial skip (0,0)->(t,0) */
                if (c > d) {
                    d = c;
                    from = BP_SKIP;
                }
            }
            delta[CELL(t, u)] = d;
            bp[CELL(t, u)] = from;
        }

    /* final arcs: terminating blank from (T-1,U); force-final skips into (T-1,U); allow-ignore skips to F */
    int end_t = T - 1, final_skip_from = -1;
    double score;
    {
        double dm = -INFINITY;
        int tm = -1;
        if (W)
            for (int tp = 0; tp <= T - 2; ++tp)
                if (delta[CELL(tp, U)] > dm) {
                    dm = delta[CELL(tp, U)];
                    tm = tp;
                }
        if (variant == ORACLE_W_FORCE_FINAL) {
            double into = delta[CELL(T - 1, U)];
            if (dm > into) { /* force-final skip (t*,U)->(T-1,U) */
                into = dm;
                final_skip_from = tm;
            }
            score = into + lpb[CELL(T - 1, U)];
        } else if (variant == ORACLE_W_ALLOW_IGNORE) {
            score = delta[CELL(T - 1, U)] + lpb[CELL(T - 1, U)];
            if (dm > score) { /* allow-ignore skip (t*,U)->F */
                score = dm;
                final_skip_from = tm;
            }
        } else {
            score = delta[CELL(T - 1, U)] + lpb[CELL(T - 1, U)];
        }
        if (final_skip_from >= 0) end_t = final_skip_from;
    }
    if (best) *best = score;
    if (score == -INFINITY) {
        free(lpb); free(lpy); free(delta); free(bp);
        return 0;
    }
    /* back-trace */
    int t = end_t, u = U, start_t = 0;
    while (!(t == 0 && u == 0)) {
        const unsigned char f = bp[CELL(t, u)];
        if (f == BP_BLANK) {
            t -= 1;
        } else if (f == BP_LABEL) {
            if (frames) frames[u - 1] = t;
            u -= 1;
        } else { /* initial skip into (t,0) */
            start_t = t;
            t = 0;
        }
    }
    if (span) {
        span[0] = start_t;
        span[1] = end_t;
    }
    free(lpb); free(lpy); free(delta); free(bp);
#undef CELL
#undef ZROW
    return 0;
}
