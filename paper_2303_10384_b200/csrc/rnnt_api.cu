// rnnt_api.cu -- the C ABI (include/rnnt_b200.h): host-side argument checks, workspace carve-up, and the
// K1 -> K2 -> K3 launch sequence on the caller's stream; plus the chunk-pipelined host-buffer path.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "elem.cuh"
#include "rnnt_b200.h"

using rnnt::Problem;
using rnnt::Workspace;

namespace {

bool ranges_overlap(const void* a, size_t na, const void* b, size_t nb) {
    const uintptr_t pa = reinterpret_cast<uintptr_t>(a), pb = reinterpret_cast<uintptr_t>(b);
    return pa < pb + nb && pb < pa + na;
}

rnnt_status check_sizes(int B, int Tmax, int Umax, int V, int blank) {
    if (B < 0 || Tmax < 1 || Umax < 0 || V < 2 || blank < 0 || blank >= V) return RNNT_ERR_INVALID_ARG;
    if (Umax + 1 > rnnt::kMaxUp1) return RNNT_ERR_UNSUPPORTED;
    return RNNT_OK;
}

rnnt_status launch_path(const rnnt::Problem& p, const rnnt::Workspace& w, cudaStream_t s,
                        void* const* events);

// A timing event: while the stream is being captured into a CUDA graph it becomes an external event-record
// node, which (unlike a plain captured record) is timed on every replay.
cudaError_t record_timing(cudaEvent_t e, cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(s, &st) != cudaSuccess) return cudaErrorUnknown;
    return st == cudaStreamCaptureStatusActive ? cudaEventRecordWithFlags(e, s, cudaEventRecordExternal)
                                               : cudaEventRecord(e, s);
}

rnnt_status run(const void* logits, int dtype, const int32_t* targets, const int32_t* logit_lens,
                const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank, float* losses,
                void* grads, const float* grad_scale, void* workspace, size_t workspace_bytes, void* stream,
                int variant, void* const* events = nullptr) {
    rnnt_status st = check_sizes(B, Tmax, Umax, V, blank);
    if (st != RNNT_OK) return st;
    if (variant < rnnt::kRnnt || variant > rnnt::kAllowIgnore) return RNNT_ERR_INVALID_ARG;
    if (dtype != rnnt::kF32 && dtype != rnnt::kF16 && dtype != rnnt::kBF16) return RNNT_ERR_INVALID_ARG;
    if (B == 0) return RNNT_OK;  // empty batch: nothing to do
    if (!logits || !logit_lens || !target_lens || !losses || !workspace) return RNNT_ERR_INVALID_ARG;
    if (Umax > 0 && !targets) return RNNT_ERR_INVALID_ARG;
    if (workspace_bytes < rnnt::workspace_bytes(B, Tmax, Umax)) return RNNT_ERR_WORKSPACE_TOO_SMALL;
    const size_t tensor_bytes = rnnt::dtype_size(dtype) * static_cast<size_t>(B) * Tmax * (Umax + 1) * V;
    if (grads && grads != logits && ranges_overlap(grads, tensor_bytes, logits, tensor_bytes))
        return RNNT_ERR_INVALID_ARG;

    Problem p{logits, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, variant, losses, grads,
              grad_scale, dtype};
    const Workspace w = rnnt::carve(workspace, B, Tmax, Umax);
    return launch_path(p, w, static_cast<cudaStream_t>(stream), events);
}

int variant_kind(int variant) {  // C-ABI variant code (-1 RNN-T, wrnnt_variant) -> internal kind
    return (variant < 0) ? rnnt::kRnnt : (variant == WRNNT_FORCE_FINAL ? rnnt::kForceFinal : rnnt::kAllowIgnore);
}

// Utterances [b0, b0+nb) of a call: every array is utterance-major, so a chunk is a pointer offset.
void slice(const Problem& p, const Workspace& w, int b0, int nb, Problem& pc, Workspace& wc) {
    const int64_t Up1 = p.Umax + 1, Dmax = static_cast<int64_t>(p.Tmax) + p.Umax;
    const int64_t cells = static_cast<int64_t>(p.Tmax) * Up1;
    pc = p;
    pc.B = nb;
    const int64_t esize = static_cast<int64_t>(rnnt::dtype_size(p.dtype));
    pc.logits = static_cast<const char*>(p.logits) + b0 * cells * p.V * esize;
    pc.targets = p.targets ? p.targets + static_cast<int64_t>(b0) * p.Umax : nullptr;
    pc.T_b = p.T_b + b0;
    pc.U_b = p.U_b + b0;
    pc.losses = p.losses + b0;
    pc.grads = p.grads ? static_cast<char*>(p.grads) + b0 * cells * p.V * esize : nullptr;
    pc.grad_scale = p.grad_scale ? p.grad_scale + b0 : nullptr;
    wc.lse = w.lse + b0 * cells;
    wc.lp = w.lp + b0 * Dmax * Up1;
    wc.alpha = w.alpha + b0 * Dmax * Up1;
    wc.beta = w.beta + b0 * Dmax * Up1;
    wc.logp = w.logp + b0;
}

// Number of utterance chunks the call is split into so that K2 (latency-bound, 2 CTAs per utterance) of one
// chunk runs concurrently with K1 / K3 (bandwidth-bound, the whole GPU) of the others.  Small calls (where
// the split buys nothing) stay sequential.
int overlap_chunks(const Problem& p) {
    return rnnt::overlap_chunks(p.B, static_cast<int64_t>(p.B) * p.Tmax * (p.Umax + 1) * p.V);
}
using rnnt::AuxPool;
using rnnt::aux_pool;
using rnnt::kMaxChunks;

// K1 -> K2 -> K3 for one call.  With chunks c = 0..n-1 the order is
//   stream s:       K1(0) K1(1) .. K1(n-1)  [wait K2(0)] K3(0)  [wait K2(1)] K3(1) ..
//   stream aux[c]:  [wait K1(c)] K2(c)                              (high priority, one stream per chunk)
// so every K2 hides under the remaining K1 / K3 traffic; small calls put K3(c) on aux[c] after K2(c) instead.  events[0..5] (optional): K1 start / end and K3
// start (after the first K2 wait) / end on s; K2 start / end on aux[0] (the first chunk's wavefront).
rnnt_status launch_path(const Problem& p, const Workspace& w, cudaStream_t s, void* const* events) {
    auto ev = [&](int i) { return static_cast<cudaEvent_t>(events[i]); };
    const int nch = overlap_chunks(p);
    AuxPool* pool = (nch > 1) ? aux_pool() : nullptr;
    if (nch == 1 || pool == nullptr) {
        if (events && record_timing(ev(0), s) != cudaSuccess) return RNNT_ERR_CUDA;
        if (rnnt::launch_k1_lse_gather(p, w, s) != cudaSuccess) return RNNT_ERR_CUDA;
        if (events && (record_timing(ev(1), s) != cudaSuccess || record_timing(ev(4), s) != cudaSuccess))
            return RNNT_ERR_CUDA;
        if (rnnt::launch_k2_alpha_beta(p, w, s) != cudaSuccess) return RNNT_ERR_CUDA;
        if (events && (record_timing(ev(5), s) != cudaSuccess || record_timing(ev(2), s) != cudaSuccess))
            return RNNT_ERR_CUDA;
        if (p.grads && rnnt::launch_k3_grad(p, w, s) != cudaSuccess) return RNNT_ERR_CUDA;
        if (events && record_timing(ev(3), s) != cudaSuccess) return RNNT_ERR_CUDA;
        return RNNT_OK;
    }
    Problem pc[kMaxChunks];
    Workspace wc[kMaxChunks];
    for (int c = 0, b0 = 0; c < nch; ++c) {
        const int nb = p.B / nch + (c < p.B % nch ? 1 : 0);
        slice(p, w, b0, nb, pc[c], wc[c]);
        b0 += nb;
    }
    auto ok = [](cudaError_t e) { return e == cudaSuccess; };
    if (events && !ok(record_timing(ev(0), s))) return RNNT_ERR_CUDA;
    // Small calls (< 2^28 joint elements, e.g. c2): K3(c) follows K2(c) on aux[c] instead of queueing on s behind
    // every K1 chunk, so the first chunks' gradient passes overlap the later chunks' K1 and the K2 latency of the
    // last chunk hides under them (c2 0.101 -> 0.094 ms); on large calls the overlapping K1 / K3 streams compete
    // for HBM and lose (c3 2.91 -> 3.01 ms, p124 0.93 -> 0.95 ms).  RNNT_K3_ON_AUX=0 / 1 forces either (A/B).
    const int64_t elems = static_cast<int64_t>(p.B) * p.Tmax * (p.Umax + 1) * p.V;
    bool k3_aux = elems < (int64_t(1) << 28);
    if (const char* e = getenv("RNNT_K3_ON_AUX")) k3_aux = atoi(e) != 0;
    if (k3_aux) {
        for (int c = 0; c < nch; ++c) {
            cudaStream_t a = pool->aux[c];
            if (!ok(rnnt::launch_k1_lse_gather(pc[c], wc[c], s)) || !ok(cudaEventRecord(pool->k1_done[c], s)) ||
                !ok(cudaStreamWaitEvent(a, pool->k1_done[c], 0)))
                return RNNT_ERR_CUDA;
            if (c == 0 && events && !ok(record_timing(ev(4), a))) return RNNT_ERR_CUDA;
            if (!ok(rnnt::launch_k2_alpha_beta(pc[c], wc[c], a))) return RNNT_ERR_CUDA;
            if (c == 0 && events && (!ok(record_timing(ev(5), a)) || !ok(record_timing(ev(2), a)))) return RNNT_ERR_CUDA;
            if (p.grads && !ok(rnnt::launch_k3_grad(pc[c], wc[c], a))) return RNNT_ERR_CUDA;
            if (!ok(cudaEventRecord(pool->k2_done[c], a))) return RNNT_ERR_CUDA;
        }
        if (events && !ok(record_timing(ev(1), s))) return RNNT_ERR_CUDA;
        for (int c = 0; c < nch; ++c)
            if (!ok(cudaStreamWaitEvent(s, pool->k2_done[c], 0))) return RNNT_ERR_CUDA;
        if (events && !ok(record_timing(ev(3), s))) return RNNT_ERR_CUDA;
        return RNNT_OK;
    }
    for (int c = 0; c < nch; ++c) {
        cudaStream_t a = pool->aux[c];
        if (!ok(rnnt::launch_k1_lse_gather(pc[c], wc[c], s)) || !ok(cudaEventRecord(pool->k1_done[c], s)) ||
            !ok(cudaStreamWaitEvent(a, pool->k1_done[c], 0)))
            return RNNT_ERR_CUDA;
        if (c == 0 && events && !ok(record_timing(ev(4), a))) return RNNT_ERR_CUDA;
        if (!ok(rnnt::launch_k2_alpha_beta(pc[c], wc[c], a))) return RNNT_ERR_CUDA;
        // ev(5) before k2_done: everything on aux is then joined back into s by the wait on k2_done (a graph
        // capture of this call must not leave work on aux unjoined).
        if (c == 0 && events && !ok(record_timing(ev(5), a))) return RNNT_ERR_CUDA;
        if (!ok(cudaEventRecord(pool->k2_done[c], a))) return RNNT_ERR_CUDA;
    }
    if (events && !ok(record_timing(ev(1), s))) return RNNT_ERR_CUDA;
    for (int c = 0; c < nch; ++c) {
        if (!ok(cudaStreamWaitEvent(s, pool->k2_done[c], 0))) return RNNT_ERR_CUDA;
        if (c == 0 && events && !ok(record_timing(ev(2), s))) return RNNT_ERR_CUDA;
        if (p.grads && !ok(rnnt::launch_k3_grad(pc[c], wc[c], s))) return RNNT_ERR_CUDA;
    }
    if (events && !ok(record_timing(ev(3), s))) return RNNT_ERR_CUDA;
    return RNNT_OK;
}

}  // namespace

namespace rnnt {

int overlap_chunks(int64_t B, int64_t elems) {
    if (B < 2 || elems < (int64_t(1) << 24)) return 1;
    return static_cast<int>(std::min<int64_t>(B, kMaxChunks));
}

// Per-host-thread, per-device cache of the internal streams / events of the overlapped path (creating
// them per call would cost tens of microseconds of host time, comparable to a small call's device time).
// Thread-local, so concurrent callers on different threads never share an event.
namespace {
constexpr int kMaxDevices = 64;
thread_local AuxPool t_pools[kMaxDevices];
}  // namespace

AuxPool* aux_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
    AuxPool& pool = t_pools[dev];
    if (pool.ready) return &pool;
    int lo = 0, hi = 0;
    if (cudaDeviceGetStreamPriorityRange(&lo, &hi) != cudaSuccess) return nullptr;
    for (int c = 0; c < kMaxChunks; ++c) {
        if (cudaStreamCreateWithPriority(&pool.aux[c], cudaStreamNonBlocking, hi) != cudaSuccess ||
            cudaEventCreateWithFlags(&pool.k1_done[c], cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&pool.k2_done[c], cudaEventDisableTiming) != cudaSuccess)
            return nullptr;
    }
    pool.ready = true;
    return &pool;
}

}  // namespace rnnt

namespace {

// Chunk size of the host path: ~16 chunks, so the pipeline fill (first H2D) and drain (last D2H) are short
// against the overlapped middle where H2D(c+1), compute(c) and D2H(c-1) run together.
int host_chunk(int B) { return std::max(1, (B + 15) / 16); }
// Device staging slots of the host path: a ring (chunk c uses slot c % kHostSlots), so the device holds
// kHostSlots chunks -- one arriving, one computing, one leaving -- not the whole batch.
constexpr int kHostSlots = 3;
int dtype_size(int dtype) { return dtype == rnnt::kF32 ? 4 : 2; }

// Per-host-thread, per-device cache of the host path's copy streams and events (created once: creating them
// per call cost tens of microseconds of host time).
struct HostPool {
    bool ready = false;
    cudaStream_t h2d = nullptr, d2h = nullptr;
    cudaEvent_t start = nullptr, done = nullptr;
    cudaEvent_t in[kHostSlots] = {}, computed[kHostSlots] = {}, out[kHostSlots] = {};
};
thread_local HostPool t_host_pools[64];

HostPool* host_pool() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
    HostPool& hp = t_host_pools[dev];
    if (hp.ready) return &hp;
    auto ev = [](cudaEvent_t* e) { return cudaEventCreateWithFlags(e, cudaEventDisableTiming) == cudaSuccess; };
    if (cudaStreamCreateWithFlags(&hp.h2d, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&hp.d2h, cudaStreamNonBlocking) != cudaSuccess || !ev(&hp.start) || !ev(&hp.done))
        return nullptr;
    for (int k = 0; k < kHostSlots; ++k)
        if (!ev(&hp.in[k]) || !ev(&hp.computed[k]) || !ev(&hp.out[k])) return nullptr;
    hp.ready = true;
    return &hp;
}

}  // namespace

extern "C" {

size_t rnnt_workspace_bytes(int B, int Tmax, int Umax) {
    if (B < 0 || Tmax < 1 || Umax < 0) return 0;
    return rnnt::workspace_bytes(B, Tmax, Umax);
}

rnnt_status rnnt_loss(const float* logits, const int32_t* targets, const int32_t* logit_lens,
                      const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank, float* losses,
                      float* grads, const float* grad_scale, void* workspace, size_t workspace_bytes,
                      void* stream) {
    return run(logits, rnnt::kF32, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, losses, grads,
               grad_scale, workspace, workspace_bytes, stream, rnnt::kRnnt);
}

rnnt_status wrnnt_loss(const float* logits, const int32_t* targets, const int32_t* logit_lens,
                       const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank, float* losses,
                       float* grads, const float* grad_scale, void* workspace, size_t workspace_bytes,
                       void* stream, wrnnt_variant variant) {
    int v;
    if (variant == WRNNT_FORCE_FINAL)
        v = rnnt::kForceFinal;
    else if (variant == WRNNT_ALLOW_IGNORE)
        v = rnnt::kAllowIgnore;
    else
        return RNNT_ERR_INVALID_ARG;
    return run(logits, rnnt::kF32, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, losses, grads,
               grad_scale, workspace, workspace_bytes, stream, v);
}

rnnt_status rnnt_loss_timed(const float* logits, const int32_t* targets, const int32_t* logit_lens,
                            const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank,
                            float* losses, float* grads, const float* grad_scale, void* workspace,
                            size_t workspace_bytes, void* stream, int variant, void* const* events) {
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    return run(logits, rnnt::kF32, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, losses, grads,
               grad_scale, workspace, workspace_bytes, stream, variant_kind(variant), events);
}

rnnt_status rnnt_loss_ex(const void* logits, rnnt_dtype dtype, const int32_t* targets, const int32_t* logit_lens,
                         const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank, int variant,
                         float* losses, void* grads, const float* grad_scale, void* workspace,
                         size_t workspace_bytes, void* stream, void* const* events) {
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    return run(logits, static_cast<int>(dtype), targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, losses,
               grads, grad_scale, workspace, workspace_bytes, stream, variant_kind(variant), events);
}

rnnt_status rnnt_viterbi(const void* logits, rnnt_dtype dtype, const int32_t* targets, const int32_t* logit_lens,
                         const int32_t* target_lens, int B, int Tmax, int Umax, int V, int blank, int variant,
                         float* best_logp, int32_t* frames, int32_t* span, void* workspace, size_t workspace_bytes,
                         void* stream) {
    rnnt_status st = check_sizes(B, Tmax, Umax, V, blank);
    if (st != RNNT_OK) return st;
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    if (dtype != RNNT_F32 && dtype != RNNT_F16 && dtype != RNNT_BF16) return RNNT_ERR_INVALID_ARG;
    if (Umax + 1 > rnnt::kMaxUp1Viterbi) return RNNT_ERR_UNSUPPORTED;
    if (B == 0) return RNNT_OK;
    if (!logits || !logit_lens || !target_lens || !best_logp || !workspace) return RNNT_ERR_INVALID_ARG;
    if (Umax > 0 && (!targets || !frames)) return RNNT_ERR_INVALID_ARG;
    if (workspace_bytes < rnnt::workspace_bytes(B, Tmax, Umax)) return RNNT_ERR_WORKSPACE_TOO_SMALL;
    Problem p{logits, targets, logit_lens, target_lens, B, Tmax, Umax, V, blank, variant_kind(variant), nullptr,
              nullptr, nullptr, static_cast<int>(dtype)};
    const Workspace w = rnnt::carve(workspace, B, Tmax, Umax);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (rnnt::launch_k1_lse_gather(p, w, s) != cudaSuccess) return RNNT_ERR_CUDA;
    if (rnnt::launch_k4_viterbi(p, w, best_logp, frames, span, s) != cudaSuccess) return RNNT_ERR_CUDA;
    return RNNT_OK;
}

rnnt_status rnnt_loss_sum(const float* losses, int B, double* loss_sum, void* stream) {
    if (B < 0 || !loss_sum || (B > 0 && !losses)) return RNNT_ERR_INVALID_ARG;
    if (rnnt::launch_loss_sum(losses, B, loss_sum, static_cast<cudaStream_t>(stream)) != cudaSuccess)
        return RNNT_ERR_CUDA;
    return RNNT_OK;
}

// Device buffer of the host path: [kHostSlots staging slots of C utterances' logits / grads][targets][T_b][U_b]
// [losses][one chunk workspace per slot].  All 256-byte aligned.
size_t rnnt_host_buffer_bytes_ex(int B, int Tmax, int Umax, int V, rnnt_dtype dtype) {
    if (check_sizes(B, Tmax, Umax, V, 0) != RNNT_OK) return 0;
    if (dtype != RNNT_F32 && dtype != RNNT_F16 && dtype != RNNT_BF16) return 0;
    const int64_t cells = static_cast<int64_t>(Tmax) * (Umax + 1);
    const int C = host_chunk(B);
    const int slots = std::min(kHostSlots, (B + C - 1) / C);
    size_t s = 0;
    s += static_cast<size_t>(std::max(slots, 1)) * rnnt::align256(static_cast<size_t>(dtype_size(dtype)) * C * cells * V);
    s += rnnt::align256(sizeof(int32_t) * B * std::max(Umax, 1));
    s += 2 * rnnt::align256(sizeof(int32_t) * B);
    s += rnnt::align256(sizeof(float) * B);
    s += static_cast<size_t>(std::max(slots, 1)) * rnnt::workspace_bytes(C, Tmax, Umax);
    return s;
}

size_t rnnt_host_buffer_bytes(int B, int Tmax, int Umax, int V) {
    return rnnt_host_buffer_bytes_ex(B, Tmax, Umax, V, RNNT_F32);
}

rnnt_status rnnt_loss_host_ex(const void* logits_host, rnnt_dtype dtype, const int32_t* targets_host,
                              const int32_t* logit_lens_host, const int32_t* target_lens_host, int B, int Tmax,
                              int Umax, int V, int blank, int variant, float* losses_host, void* grads_host,
                              void* device_buffer, size_t device_buffer_bytes, void* stream) {
    rnnt_status st = check_sizes(B, Tmax, Umax, V, blank);
    if (st != RNNT_OK) return st;
    if (variant < -1 || variant > 1) return RNNT_ERR_INVALID_ARG;
    if (dtype != RNNT_F32 && dtype != RNNT_F16 && dtype != RNNT_BF16) return RNNT_ERR_INVALID_ARG;
    if (B == 0) return RNNT_OK;
    if (!logits_host || !logit_lens_host || !target_lens_host || !losses_host || !device_buffer)
        return RNNT_ERR_INVALID_ARG;
    if (Umax > 0 && !targets_host) return RNNT_ERR_INVALID_ARG;
    if (device_buffer_bytes < rnnt_host_buffer_bytes_ex(B, Tmax, Umax, V, dtype)) return RNNT_ERR_WORKSPACE_TOO_SMALL;
    HostPool* hp = host_pool();
    if (!hp) return RNNT_ERR_CUDA;
    const int kind = (variant < 0) ? rnnt::kRnnt : (variant == 0 ? rnnt::kForceFinal : rnnt::kAllowIgnore);
    const int es = dtype_size(dtype);
    const int64_t cells = static_cast<int64_t>(Tmax) * (Umax + 1);
    const int64_t utt_bytes = cells * V * es;
    const int C = host_chunk(B);
    const int nchunks = (B + C - 1) / C;
    const int slots = std::min(kHostSlots, nchunks);
    const size_t slot_bytes = rnnt::align256(static_cast<size_t>(C) * utt_bytes);
    char* p = static_cast<char*>(device_buffer);
    char* d_stage = p;
    p += static_cast<size_t>(slots) * slot_bytes;
    int32_t* d_targets = reinterpret_cast<int32_t*>(p);
    p += rnnt::align256(sizeof(int32_t) * B * std::max(Umax, 1));
    int32_t* d_T = reinterpret_cast<int32_t*>(p);
    p += rnnt::align256(sizeof(int32_t) * B);
    int32_t* d_U = reinterpret_cast<int32_t*>(p);
    p += rnnt::align256(sizeof(int32_t) * B);
    float* d_losses = reinterpret_cast<float*>(p);
    p += rnnt::align256(sizeof(float) * B);
    const size_t ws_chunk = rnnt::workspace_bytes(C, Tmax, Umax);
    const char* lh = static_cast<const char*>(logits_host);
    char* gh = static_cast<char*>(grads_host);

    cudaStream_t s = static_cast<cudaStream_t>(stream);
    auto ok = [](cudaError_t e) { return e == cudaSuccess; };
    // The copy streams start after prior work on the caller's stream; small inputs go first, on s.
    if (!ok(cudaEventRecord(hp->start, s)) || !ok(cudaStreamWaitEvent(hp->h2d, hp->start, 0)) ||
        !ok(cudaStreamWaitEvent(hp->d2h, hp->start, 0)))
        return RNNT_ERR_CUDA;
    if (Umax > 0 && !ok(cudaMemcpyAsync(d_targets, targets_host, sizeof(int32_t) * B * Umax, cudaMemcpyHostToDevice, s)))
        return RNNT_ERR_CUDA;
    if (!ok(cudaMemcpyAsync(d_T, logit_lens_host, sizeof(int32_t) * B, cudaMemcpyHostToDevice, s)) ||
        !ok(cudaMemcpyAsync(d_U, target_lens_host, sizeof(int32_t) * B, cudaMemcpyHostToDevice, s)))
        return RNNT_ERR_CUDA;
    // Chunk c, slot k = c % slots:  H2D(c) on h2d (after D2H(c - slots) has drained slot k)  ->  K1..K3(c) on
    // s (in place)  ->  D2H(c) on d2h.  The three streams pipeline H2D(c+1), compute(c) and D2H(c-1).
    for (int c = 0; c < nchunks; ++c) {
        const int k = c % slots, b0 = c * C, nb = std::min(C, B - b0);
        char* slot = d_stage + static_cast<size_t>(k) * slot_bytes;
        const size_t bytes = static_cast<size_t>(nb) * utt_bytes;
        if (c >= slots && !ok(cudaStreamWaitEvent(hp->h2d, hp->out[k], 0))) return RNNT_ERR_CUDA;
        if (!ok(cudaMemcpyAsync(slot, lh + b0 * utt_bytes, bytes, cudaMemcpyHostToDevice, hp->h2d)) ||
            !ok(cudaEventRecord(hp->in[k], hp->h2d)) || !ok(cudaStreamWaitEvent(s, hp->in[k], 0)))
            return RNNT_ERR_CUDA;
        void* ws = p + static_cast<size_t>(k) * ws_chunk;
        const rnnt_status r = run(slot, static_cast<int>(dtype), d_targets + static_cast<int64_t>(b0) * Umax, d_T + b0,
                                  d_U + b0, nb, Tmax, Umax, V, blank, d_losses + b0, grads_host ? slot : nullptr,
                                  nullptr, ws, ws_chunk, s, kind);
        if (r != RNNT_OK) return r;
        if (!ok(cudaEventRecord(hp->computed[k], s)) || !ok(cudaStreamWaitEvent(hp->d2h, hp->computed[k], 0)))
            return RNNT_ERR_CUDA;
        if (grads_host && !ok(cudaMemcpyAsync(gh + b0 * utt_bytes, slot, bytes, cudaMemcpyDeviceToHost, hp->d2h)))
            return RNNT_ERR_CUDA;
        if (!ok(cudaEventRecord(hp->out[k], hp->d2h))) return RNNT_ERR_CUDA;
    }
    if (!ok(cudaMemcpyAsync(losses_host, d_losses, sizeof(float) * B, cudaMemcpyDeviceToHost, s)) ||
        !ok(cudaEventRecord(hp->done, hp->d2h)) || !ok(cudaStreamWaitEvent(s, hp->done, 0)))
        return RNNT_ERR_CUDA;
    return RNNT_OK;
}

rnnt_status rnnt_loss_host(const float* logits_host, const int32_t* targets_host, const int32_t* logit_lens_host,
                           const int32_t* target_lens_host, int B, int Tmax, int Umax, int V, int blank,
                           int variant, float* losses_host, float* grads_host, void* device_buffer,
                           size_t device_buffer_bytes, void* stream) {
    return rnnt_loss_host_ex(logits_host, RNNT_F32, targets_host, logit_lens_host, target_lens_host, B, Tmax, Umax, V,
                             blank, variant, losses_host, grads_host, device_buffer, device_buffer_bytes, stream);
}

const char* rnnt_status_string(rnnt_status status) {
    switch (status) {
        case RNNT_OK: return "RNNT_OK";
        case RNNT_ERR_INVALID_ARG: return "RNNT_ERR_INVALID_ARG: invalid argument";
        case RNNT_ERR_WORKSPACE_TOO_SMALL: return "RNNT_ERR_WORKSPACE_TOO_SMALL: workspace too small";
        case RNNT_ERR_UNSUPPORTED:
            return "RNNT_ERR_UNSUPPORTED: Umax + 1 > 4096 (1024 for Viterbi), or a fused-joint H that is not a "
                   "multiple of 128 up to 512";
        case RNNT_ERR_CUDA: return "RNNT_ERR_CUDA: CUDA launch or copy failed";
    }
    return "unknown rnnt_status";
}

const char* rnnt_version(void) { return "rnnt_b200 0.1 sm_100a"; }

}  // extern "C"
