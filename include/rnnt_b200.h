/*
 * rnnt_b200.h -- C ABI of the B200 (sm_100a) RNN-T / W-RNNT loss + logits-gradient library.
 *
 * What is computed (PAPER.md = /root/reference/PAPER.md, cited P:<line>):
 *   loss_b = -Fwd(L_b) = -log sum over complete alignment paths pi of the lattice L_b of
 *            prod_{arcs a in pi} w(a)                              Eq.(1), P:54-56 ("negative forward scores")
 *   L_b    = the Grid-Transducer lattice: a T_b x (U_b+1) grid whose horizontal (time) arcs emit <blank>
 *            and whose vertical (unit) arcs emit y_{u+1}; a terminating <blank> arc leaves (T_b-1, U_b)
 *                                                                   §2.3
 *   w(a)   = softmax(logits[b,t,u,:])[label(a)]: the lattice is populated by indexed selection from the
 *            log-probabilities tensor X = log_softmax(logits)       §2.1, §2.2 P:88 ("Populate")
 *   W-RNNT adds weight-1 <eps> skip-frame arcs:                       §3.2, §4.3
 *            initial skips (0,0) -> (t,0), 1 <= t <= T_b-1           ("from the initial state to any state
 *                                                                      before non-<blank> emissions")
 *            force-final:  (t,U_b) -> (T_b-1,U_b), 0 <= t <= T_b-2   ("point to the previous-to-final state")
 *            allow-ignore: (t,U_b) -> final,       0 <= t <= T_b-2   ("point to the final state"),
 *                          the ordinary terminating blank is kept.
 *   grads  = d loss_b / d logits[b,t,u,v] (chain rule through the log-softmax; reading R8).
 *
 * Conventions shared by every entry point:
 *   - All tensor pointers are DEVICE pointers owned by the caller unless the name ends in _host.  The
 *     library allocates no device memory and keeps no data between calls; every call is asynchronous on
 *     `stream` (a cudaStream_t passed as void*; NULL = the legacy default stream).  Large calls fork
 *     internal work onto up to 4 high-priority streams (a per-host-thread, per-device cache created on
 *     first use) and join it back into `stream` before returning, so stream semantics are unchanged.
 *   - logits  fp32 [B][Tmax][Umax+1][V], contiguous, V innermost.  Cells with t >= T_b or u > U_b are
 *             padding: never read.
 *   - targets int32 [B][Umax] (may be NULL when Umax == 0); targets[b][u], u < U_b, is unit u+1 of
 *             utterance b and must lie in [0,V) and differ from `blank`.  Entries u >= U_b are never read.
 *   - logit_lens / target_lens int32 [B]: 1 <= T_b <= Tmax, 0 <= U_b <= Umax.
 *   - losses  fp32 [B] out: per-utterance -log P_b (no reduction; reading R10).
 *   - grads   fp32 [B][Tmax][Umax+1][V] out, or NULL (loss only: the gradient pass is skipped).  grads
 *             MAY EQUAL logits (in place: each element is read before it is overwritten) but must not
 *             otherwise overlap it.  Padding cells receive exact zeros.
 *   - grad_scale fp32 [B] or NULL (= 1): grads[b] are multiplied by grad_scale[b] (e.g. 1/B for a mean
 *             reduction) inside the gradient pass, at no extra memory traffic.
 *   - Data-dependent errors are NOT reported synchronously (that would need a device sync): an utterance
 *     whose lengths or targets are out of range gets loss = NaN and all-zero grads.  An utterance whose
 *     lattice has no path of non-zero probability (e.g. -inf logits) gets loss = +inf and zero grads.  An
 *     utterance with a NaN (or +inf) logit in a valid cell gets loss = NaN and zero grads (R12).
 *   - Argument errors detectable on the host (sizes, null pointers, workspace size, overlap) are returned
 *     as a status before anything is launched.
 *   - Limits: Umax + 1 <= 4096 (one CTA per utterance and direction in the alpha/beta wavefront, up to 8
 *     columns per thread); rnnt_viterbi / rnnt_joint_viterbi: Umax + 1 <= 1024 (one thread per column);
 *     element offsets are 64-bit (a single call may exceed 2^31 elements).
 */
#ifndef RNNT_B200_H
#define RNNT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    RNNT_OK = 0,
    RNNT_ERR_INVALID_ARG = 1,          /* bad size, null pointer, blank out of range, partial overlap */
    RNNT_ERR_WORKSPACE_TOO_SMALL = 2,  /* workspace_bytes < rnnt_workspace_bytes(B, Tmax, Umax) */
    RNNT_ERR_UNSUPPORTED = 3,          /* Umax + 1 > 4096 (> 1024 for Viterbi); fused joint H % 128 != 0 or > 512 */
    RNNT_ERR_CUDA = 4                  /* a CUDA launch / copy failed (cudaGetLastError) */
} rnnt_status;

typedef enum {
    RNNT_F32 = 0,   /* fp32 logits / grads (the default entry points) */
    RNNT_F16 = 1,   /* IEEE fp16 storage; all arithmetic fp32 / fp64 (§4.2: "populate the
                       lattice with a half (fp16) precision tensor and cast it to fp32 or fp64 only for the
                       forward-backward score calculation") */
    RNNT_BF16 = 2   /* bfloat16 storage, same arithmetic */
} rnnt_dtype;

typedef enum {
    WRNNT_FORCE_FINAL = 0,   /* final skips land on (T_b-1, U_b): the last blank is still emitted */
    WRNNT_ALLOW_IGNORE = 1   /* final skips land on the final state */
} wrnnt_variant;

/* Device workspace (bytes) one call needs for these padded sizes; 0 if the sizes are invalid.
 * Holds, per (b,t,u) cell: log-softmax normalizer (fp32), blank/label log-probs (fp32 x2, anti-diagonal
 * major), alpha and beta (fp64); per utterance: log P (fp64). About 28 B per cell. */
size_t rnnt_workspace_bytes(int B, int Tmax, int Umax);

/* Plain RNN-T loss (Eq.(1) over the §2.3 grid) and, if grads != NULL, its logits-gradient. */
rnnt_status rnnt_loss(const float* logits, const int32_t* targets, const int32_t* logit_lens,
                      const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank,
                      float* losses, float* grads, const float* grad_scale,
                      void* workspace, size_t workspace_bytes, void* stream);

/* W-Transducer loss (§3.2 + §4.3) in the given variant; same arguments and conventions as rnnt_loss. */
rnnt_status wrnnt_loss(const float* logits, const int32_t* targets, const int32_t* logit_lens,
                       const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank,
                       float* losses, float* grads, const float* grad_scale,
                       void* workspace, size_t workspace_bytes, void* stream, wrnnt_variant variant);

/* rnnt_loss / wrnnt_loss with per-kernel timing (the profiling hook bench.py uses).  variant: -1 = plain
 * RNN-T, else a wrnnt_variant.  If events != NULL, events[0..5] are cudaEvent_t handles recorded as:
 * [0] before K1 (log-softmax + gather) and [1] after it, [2] before K3 (gradient) and [3] after it -- all on
 * `stream` -- and [4] before / [5] after K2 (alpha/beta wavefront).  Large calls run K2 of one half of the
 * batch concurrently with K1 / K3 of the other half on an internal high-priority stream, where [4] / [5]
 * are recorded; [2] - [1] is then the time `stream` waited for K2.  Small calls run K1, K2, K3 in order on
 * `stream` ([1] = [4], [5] = [2]). */
rnnt_status rnnt_loss_timed(const float* logits, const int32_t* targets, const int32_t* logit_lens,
                            const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank,
                            float* losses, float* grads, const float* grad_scale,
                            void* workspace, size_t workspace_bytes, void* stream, int variant,
                            void* const* events);

/* The general entry point: logits / grads in any rnnt_dtype (grads have the logits' type and are rounded to
 * nearest from the fp32 result), variant -1 = plain RNN-T or a wrnnt_variant, optional 6 timing events as in
 * rnnt_loss_timed.  Losses are fp32 whatever the storage type.  Same conventions as rnnt_loss otherwise. */
rnnt_status rnnt_loss_ex(const void* logits, rnnt_dtype dtype, const int32_t* targets,
                         const int32_t* logit_lens, const int32_t* target_lens, int B, int Tmax, int Umax,
                         int V, int blank, int variant, float* losses, void* grads, const float* grad_scale,
                         void* workspace, size_t workspace_bytes, void* stream, void* const* events);

/* Viterbi forced alignment (§2.1 P:80 "forced alignment tasks"): the single
 * best path through the same lattice (max-plus instead of log-sum-exp), ties broken blank arc > label arc >
 * skip arc, earliest frame among final skips (reading R21).  Outputs (device):
 *   best_logp [B]        fp32 log-probability of the best alignment (NaN: invalid utterance; -inf: no path)
 *   frames    [B][Umax]  frame at which unit u is emitted on the best path (u < U_b; -1 elsewhere)
 *   span      [B][2]     (first, last) frame covered by scored arcs: > 0 / < T_b-1 when the W skips are taken;
 *                        may be NULL.
 * variant: -1 = plain RNN-T, else a wrnnt_variant.  Same inputs, workspace and stream conventions as
 * rnnt_loss_ex; Umax + 1 <= 1024 (else RNNT_ERR_UNSUPPORTED). */
rnnt_status rnnt_viterbi(const void* logits, rnnt_dtype dtype, const int32_t* targets,
                         const int32_t* logit_lens, const int32_t* target_lens, int B, int Tmax, int Umax,
                         int V, int blank, int variant, float* best_logp, int32_t* frames, int32_t* span,
                         void* workspace, size_t workspace_bytes, void* stream);

/* Generic acyclic-lattice loss (§1, §2.2 Eq.(3): new losses are new
 * graphs populated from the log-probabilities tensor, not new kernels).  A batch of B lattices in arc-list
 * form (all int32 device arrays; builders in paper_2303_10384_b200/lattice.py):
 *   state_off [B+1]  states of lattice b: [state_off[b], state_off[b+1]); its first state is the start
 *   lvl_off   [B+1]  levels of lattice b: [lvl_off[b], lvl_off[b+1]) into level_off
 *   level_off [L+1]  states of level k: [level_off[k], level_off[k+1]); every arc goes to a higher level
 *   in_off    [S+1]  arcs are sorted by destination: the arcs into s are [in_off[s], in_off[s+1])
 *   out_off   [S+1], out_arc [A]: out_arc[out_off[s] .. out_off[s+1]) are the arcs leaving s
 *   arc_src / arc_dst [A] (global state ids), arc_t / arc_u / arc_v [A]: arc weight X[b, t, u, v] =
 *                    logits[b,t,u,v] - logsumexp_v logits[b,t,u,:], or 0 when arc_v < 0 (structural arc)
 *   final_w   [S]    fp32 log final weight (-inf: not final)
 *   row_off [B*Tmax*(Umax+1) + 1], row_arc [#bound arcs] or both NULL: the arcs bound to logits row
 *                    r = (b*Tmax + t)*(Umax+1) + u are row_arc[row_off[r] .. row_off[r+1]) (lattice.py builds it);
 *                    with it the gradient is one deterministic row pass, without it two float-atomic passes
 * Rows (t,u) with t < logit_lens[b], u <= target_lens[b] are live; every arc must bind a live row.
 * losses[b] = -log sum over start->final paths of exp(sum of arc weights + final weight) (Eq.(1)); grads
 * (fp32, may equal logits, or NULL) = d losses[b] / d logits, zero on non-live rows.  fp32 only; without a
 * row index, float atomics make grads order-dependent where > 2 arcs share a row or > 1 arc shares a (t,u,v). */
size_t rnnt_lattice_workspace_bytes(int B, int Tmax, int Umax, int num_states, int num_arcs);
rnnt_status rnnt_lattice_loss(const float* logits, const int32_t* logit_lens, const int32_t* target_lens,
                              int B, int Tmax, int Umax, int V, const int32_t* state_off,
                              const int32_t* lvl_off, const int32_t* level_off, const int32_t* in_off,
                              const int32_t* out_off, const int32_t* out_arc, const int32_t* arc_src,
                              const int32_t* arc_dst, const int32_t* arc_t, const int32_t* arc_u,
                              const int32_t* arc_v, const float* final_w, const int32_t* row_off,
                              const int32_t* row_arc, int num_states, int num_arcs,
                              float* losses, float* grads, void* workspace, size_t workspace_bytes,
                              void* stream);

/* Deterministic fp64 sum of losses[0..B) into *loss_sum (device), fixed summation order for a given B.
 * This is the per-rank operand of the cross-GPU all-reduce of the loss sum (BASELINE.json north_star (5)). */
rnnt_status rnnt_loss_sum(const float* losses, int B, double* loss_sum, void* stream);

/* Host-buffer entry point (the end-to-end path): logits_host / targets_host / lens_host / losses_host /
 * grads_host are HOST pointers (pinned memory recommended; pageable works but serialises the copies).
 * device_buffer must hold rnnt_host_buffer_bytes(...) bytes of device memory: a ring of 3 staging slots of
 * ~B/16 utterances each (logits in, grads out in place) plus their workspaces -- not the whole batch.
 * variant: -1 = plain RNN-T, else a wrnnt_variant.  Copies and compute are pipelined over chunks of
 * utterances (H2D of chunk c+1, compute of c and D2H of c-1 at once) on `stream` and two internal copy
 * streams (cached per host thread and device) joined back into `stream`; the call returns after enqueueing --
 * synchronize `stream` before reading the host outputs.  grads_host may be NULL (loss only).
 * The _ex forms take the logits' storage type (rnnt_dtype: fp32 / fp16 / bf16, as rnnt_loss_ex; grads_host
 * in the same type), so 16-bit storage halves the PCIe bytes. */
size_t rnnt_host_buffer_bytes(int B, int Tmax, int Umax, int V);
size_t rnnt_host_buffer_bytes_ex(int B, int Tmax, int Umax, int V, rnnt_dtype dtype);
rnnt_status rnnt_loss_host(const float* logits_host, const int32_t* targets_host,
                           const int32_t* logit_lens_host, const int32_t* target_lens_host,
                           int B, int Tmax, int Umax, int V, int blank, int variant,
                           float* losses_host, float* grads_host,
                           void* device_buffer, size_t device_buffer_bytes, void* stream);
rnnt_status rnnt_loss_host_ex(const void* logits_host, rnnt_dtype dtype, const int32_t* targets_host,
                              const int32_t* logit_lens_host, const int32_t* target_lens_host,
                              int B, int Tmax, int Umax, int V, int blank, int variant,
                              float* losses_host, void* grads_host,
                              void* device_buffer, size_t device_buffer_bytes, void* stream);

/* Fused joint network + loss (§4.1: the benchmark's joint over Encoder
 * and Predictor embeddings of size 512; X comes from the joint network).  The logits
 *   z[b,t,u,v] = bias[v] + sum_k bf16(tanh(enc[b,t,k] + pred[b,u,k])) * weight[v,k]      (R22)
 * are computed tile by tile on the tensor cores (tcgen05, fp32 accumulation) and reduced on chip to the
 * log-softmax normalizer and the Populate gathers -- the [B,Tmax,Umax+1,V] tensor is never written -- and
 * the losses follow as for rnnt_loss / wrnnt_loss of z (variant: -1 = RNN-T, else a wrnnt_variant).
 *   enc    [B][Tmax][H] bf16, pred [B][Umax+1][H] bf16, weight [V][H] bf16, bias [V] fp32 or NULL (= 0),
 *          all four 16-byte aligned (else RNNT_ERR_INVALID_ARG); targets / lens / losses / workspace as for
 *          rnnt_loss (rnnt_workspace_bytes).
 * Forward only (losses).  Requires H % 128 == 0 and H <= 512 (else RNNT_ERR_UNSUPPORTED); any V >= 2 (shared
 * memory does not grow with V: the bias is read from global memory). */
rnnt_status rnnt_joint_loss(const void* enc, const void* pred, const void* weight, const float* bias,
                            const int32_t* targets, const int32_t* logit_lens, const int32_t* target_lens,
                            int B, int Tmax, int Umax, int H, int V, int blank, int variant, float* losses,
                            void* workspace, size_t workspace_bytes, void* stream);
/* As rnnt_joint_loss; events (NULL or 4 cudaEvent_t): K6 start / end, K2 start / end. */
rnnt_status rnnt_joint_loss_ex(const void* enc, const void* pred, const void* weight, const float* bias,
                               const int32_t* targets, const int32_t* logit_lens, const int32_t* target_lens,
                               int B, int Tmax, int Umax, int H, int V, int blank, int variant, float* losses,
                               void* workspace, size_t workspace_bytes, void* stream, void* const* events);
/* Viterbi forced alignment (as rnnt_viterbi) on the fused joint's logits: K6 then K4, the logits never written.
 * Outputs as rnnt_viterbi: best_logp [B] fp32, frames [B][Umax] int32, span [B][2] int32 or NULL. */
rnnt_status rnnt_joint_viterbi(const void* enc, const void* pred, const void* weight, const float* bias,
                               const int32_t* targets, const int32_t* logit_lens, const int32_t* target_lens,
                               int B, int Tmax, int Umax, int H, int V, int blank, int variant, float* best_logp,
                               int32_t* frames, int32_t* span, void* workspace, size_t workspace_bytes,
                               void* stream);

/* Training step of the fused joint (NEXT-4 backward; R22, R23): losses as rnnt_joint_loss, and the
 * gradients of sum_b losses[b] with respect to the joint's inputs, fp32 row-major:
 *   d_enc [B][Tmax][H], d_pred [B][Umax+1][H] (zero on padded frames / units), d_weight [V][H], d_bias [V]
 *   (or NULL); grad_scale [B] or NULL: gradients of sum_b grad_scale[b] * losses[b] (1/B gives the mean),
 *   as rnnt_loss.  dz = d loss / d z is formed on chip from the recomputed logits (K3's formula) and stored in bf16
 *   for the two backward GEMMs (dh = dz W stored in bf16, dW = dz^T h; cuBLAS, fp32 accumulation); tanh' uses
 *   the stored bf16 h.  workspace: rnnt_joint_grad_workspace_bytes(...) bytes (it holds dz, h and dh of every
 *   padded cell: ~ (2 V + 4 H) bytes per cell).  Same constraints as rnnt_joint_loss.
 *   valid_rows: the number of valid cells, sum over the valid utterances (1 <= T_b <= Tmax, 0 <= U_b <= Umax)
 *   of T_b (U_b + 1), when the caller knows it (the host usually holds the lengths), else -1.  Given, the two
 *   GEMMs run over the valid cells only (no work on padding); it must equal the device's count, else every
 *   loss is set to NaN (and the gradients are undefined).  Out of [-1, B Tmax (Umax+1)]: RNNT_ERR_INVALID_ARG. */
size_t rnnt_joint_grad_workspace_bytes(int B, int Tmax, int Umax, int H, int V);
rnnt_status rnnt_joint_loss_grad(const void* enc, const void* pred, const void* weight, const float* bias,
                                 const int32_t* targets, const int32_t* logit_lens, const int32_t* target_lens,
                                 int B, int Tmax, int Umax, int H, int V, int blank, int variant, float* losses,
                                 float* d_enc, float* d_pred, float* d_weight, float* d_bias,
                                 const float* grad_scale, int64_t valid_rows, void* workspace,
                                 size_t workspace_bytes, void* stream);

const char* rnnt_status_string(rnnt_status status);

/* Library version, e.g. "rnnt_b200 0.1 sm_100a". */
const char* rnnt_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RNNT_B200_H */
