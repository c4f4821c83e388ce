"""B200-native RNN-T / W-RNNT loss + logits-gradient (arXiv 2303.10384 Grid-Transducer hot path).

Thin ctypes binding over the C ABI in ``include/rnnt_b200.h`` (``lib/librnnt_b200.so``): argument
marshalling only -- every step of the path runs in the sm_100a kernels.  PyTorch supplies device memory
and the current CUDA stream.  There is no CPU fallback: importing this package without the built library
raises, and the compute entry points require CUDA tensors.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from ._build import LIB_PATH

__all__ = ["rnnt_loss", "wrnnt_loss", "rnnt_loss_sum", "rnnt_loss_host", "rnnt_workspace_bytes",
           "rnnt_host_buffer_bytes", "RnntError", "library", "LIB_PATH", "EXPORTS"]

RNNT_OK = 0
VARIANTS = {"rnnt": -1, "force_final": 0, "allow_ignore": 1}

# Every symbol include/rnnt_b200.h declares.
EXPORTS = ("rnnt_workspace_bytes", "rnnt_loss", "wrnnt_loss", "rnnt_loss_timed", "rnnt_loss_ex", "rnnt_viterbi",
           "rnnt_loss_sum", "rnnt_lattice_workspace_bytes", "rnnt_lattice_loss",
           "rnnt_host_buffer_bytes", "rnnt_loss_host", "rnnt_host_buffer_bytes_ex", "rnnt_loss_host_ex",
           "rnnt_joint_loss", "rnnt_joint_loss_ex", "rnnt_joint_viterbi",
           "rnnt_joint_grad_workspace_bytes", "rnnt_joint_loss_grad",
           "rnnt_status_string", "rnnt_version")
DTYPES = {torch.float32: 0, torch.float16: 1, torch.bfloat16: 2}


class RnntError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (nvcc, sm_100a). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, S, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_int64
    common = [P, P, P, P, I, I, I, I, I, P, P, P, P, S, P]
    sigs = {
        "rnnt_workspace_bytes": ([I, I, I], S),
        "rnnt_loss": (common, I),
        "wrnnt_loss": (common + [I], I),
        "rnnt_loss_timed": (common + [I, P], I),
        "rnnt_loss_ex": ([P, I, P, P, P, I, I, I, I, I, I, P, P, P, P, S, P, P], I),
        "rnnt_viterbi": ([P, I, P, P, P, I, I, I, I, I, I, P, P, P, P, S, P], I),
        "rnnt_lattice_workspace_bytes": ([I, I, I, I, I], S),
        "rnnt_lattice_loss": ([P, P, P, I, I, I, I] + [P] * 14 + [I, I, P, P, P, S, P], I),
        "rnnt_loss_sum": ([P, I, P, P], I),
        "rnnt_host_buffer_bytes": ([I, I, I, I], S),
        "rnnt_loss_host": ([P, P, P, P, I, I, I, I, I, I, P, P, P, S, P], I),
        "rnnt_host_buffer_bytes_ex": ([I, I, I, I, I], S),
        "rnnt_loss_host_ex": ([P, I, P, P, P, I, I, I, I, I, I, P, P, P, S, P], I),
        "rnnt_joint_loss": ([P, P, P, P, P, P, P, I, I, I, I, I, I, I, P, P, S, P], I),
        "rnnt_joint_loss_ex": ([P, P, P, P, P, P, P, I, I, I, I, I, I, I, P, P, S, P, P], I),
        "rnnt_joint_viterbi": ([P, P, P, P, P, P, P, I, I, I, I, I, I, I, P, P, P, P, S, P], I),
        "rnnt_joint_grad_workspace_bytes": ([I, I, I, I, I], S),
        "rnnt_joint_loss_grad": ([P, P, P, P, P, P, P, I, I, I, I, I, I, I, P, P, P, P, P, P, L, P, S, P], I),
        "rnnt_status_string": ([I], ctypes.c_char_p),
        "rnnt_version": ([], ctypes.c_char_p),
    }
    for name, (argtypes, restype) in sigs.items():
        if hasattr(lib, name):  # every symbol is checked present by build() and tests/test_abi.py; an older
            fn = getattr(lib, name)  # library loaded through RNNT_B200_LIB for A/B timing may lack new ones
            fn.argtypes, fn.restype = argtypes, restype
    return lib


library = _load()


def _check(status: int):
    if status != RNNT_OK:
        raise RnntError(library.rnnt_status_string(status).decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _keep(stream, *tensors):
    """The library queues its kernels on ``stream``; temporaries allocated here belong to the current stream's
    pool.  When the caller passes another stream, record it on each temporary so that the caching allocator
    does not hand their memory out again before the queued kernels are done with it."""
    if stream is None or stream == torch.cuda.current_stream():
        return
    for t in tensors:
        if isinstance(t, torch.Tensor) and t.is_cuda:
            t.record_stream(stream)


def _check_joint_inputs(enc, pred, weight):
    """enc [B, Tmax, H], pred [B, Umax+1, H], weight [V, H]: contiguous CUDA bfloat16 on one device."""
    for name, x in (("enc", enc), ("pred", pred), ("weight", weight)):
        if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.bfloat16 and x.is_contiguous()):
            raise TypeError(f"{name} must be a contiguous CUDA bfloat16 tensor (no CPU fallback)")
    if enc.dim() != 3 or pred.dim() != 3 or weight.dim() != 2:
        raise ValueError("shapes: enc [B, Tmax, H], pred [B, Umax+1, H], weight [V, H]")
    B, Tmax, H = enc.shape
    Up1 = pred.shape[1]
    V = weight.shape[0]
    if pred.shape != (B, Up1, H) or weight.shape != (V, H) or Up1 < 1:
        raise ValueError("shapes: enc [B, Tmax, H], pred [B, Umax+1, H], weight [V, H]")
    if pred.device != enc.device or weight.device != enc.device:
        raise ValueError("enc, pred and weight must be on one device")
    return B, Tmax, Up1 - 1, H, V


def _check_f32_out(name, t, shape, device):
    if not (isinstance(t, torch.Tensor) and t.dtype == torch.float32 and t.device == device and t.is_contiguous()
            and tuple(t.shape) == tuple(shape)):
        raise ValueError(f"{name} must be a contiguous float32 tensor of shape {tuple(shape)} on {device}")


def _check_grad_scale(grad_scale, B, dev):
    if grad_scale is None:
        return None
    grad_scale = torch.as_tensor(grad_scale).to(device=dev, dtype=torch.float32).contiguous()
    if grad_scale.numel() != B:
        raise ValueError(f"grad_scale needs {B} elements (one per utterance), got {grad_scale.numel()}")
    return grad_scale


def rnnt_workspace_bytes(B: int, Tmax: int, Umax: int) -> int:
    return int(library.rnnt_workspace_bytes(B, Tmax, Umax))


def rnnt_host_buffer_bytes(B: int, Tmax: int, Umax: int, V: int, dtype=torch.float32) -> int:
    return int(library.rnnt_host_buffer_bytes_ex(B, Tmax, Umax, V, DTYPES[dtype]))


def _as_i32(x, device):
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    return x.to(device=device, dtype=torch.int32).contiguous()


def _call(fn_variant, logits, targets, logit_lens, target_lens, blank, grads, grad_scale, losses, workspace,
          stream, events=None):
    if not (isinstance(logits, torch.Tensor) and logits.is_cuda and logits.dtype in DTYPES):
        raise TypeError("logits must be a CUDA float32 / float16 / bfloat16 tensor [B, Tmax, Umax+1, V] "
                        "(no CPU fallback)")
    if not logits.is_contiguous():
        raise ValueError("logits must be contiguous")
    B, Tmax, Up1, V = logits.shape
    Umax = Up1 - 1
    dev = logits.device
    targets = _as_i32(targets, dev).reshape(B, Umax) if Umax > 0 else None
    logit_lens = _as_i32(logit_lens, dev)
    target_lens = _as_i32(target_lens, dev)
    if losses is None:
        losses = torch.empty(B, dtype=torch.float32, device=dev)
    if isinstance(grads, str) and grads == "inplace":
        grads = logits
    elif grads is True:
        grads = torch.empty_like(logits)
    elif grads is False:
        grads = None
    if grads is not None and (grads.shape != logits.shape or not grads.is_contiguous()
                              or grads.dtype != logits.dtype or grads.device != dev):
        raise ValueError("grads must be contiguous, on the logits' device, with the logits' shape and dtype")
    grad_scale = _check_grad_scale(grad_scale, B, dev)
    need = rnnt_workspace_bytes(B, Tmax, Umax)
    if workspace is None:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    _keep(stream, targets, logit_lens, target_lens, losses, grads, grad_scale, workspace)
    args = [_ptr(logits), _ptr(targets), _ptr(logit_lens), _ptr(target_lens), B, Tmax, Umax, V, int(blank),
            _ptr(losses), _ptr(grads), _ptr(grad_scale), _ptr(workspace), workspace.numel(), _stream(stream)]
    ev = None
    if events is not None:
        handles = [e.cuda_event for e in events]
        if len(handles) != 6 or not all(handles):
            raise ValueError("need 6 recorded torch.cuda.Events")
        ev = ctypes.cast((ctypes.c_void_p * 6)(*handles), ctypes.c_void_p)
    if logits.dtype == torch.float32 and ev is None:
        if fn_variant < 0:
            _check(library.rnnt_loss(*args))
        else:
            _check(library.wrnnt_loss(*args, fn_variant))
    else:
        _check(library.rnnt_loss_ex(args[0], DTYPES[logits.dtype], *args[1:9], fn_variant, *args[9:], ev))
    return losses, grads


def rnnt_loss(logits, targets, logit_lens, target_lens, blank=0, grads=True, grad_scale=None, losses=None,
              workspace=None, stream=None):
    """Per-utterance RNN-T losses and d loss_b / d logits (Eq.(1), §2.3 Grid-Transducer).

    grads: True (new tensor), "inplace" (overwrite logits), False (loss only) or a preallocated tensor.
    Returns (losses fp32 [B], grads or None).  Asynchronous on the current CUDA stream.
    """
    return _call(-1, logits, targets, logit_lens, target_lens, blank, grads, grad_scale, losses, workspace,
                 stream)


def wrnnt_loss(logits, targets, logit_lens, target_lens, blank=0, variant="force_final", grads=True,
               grad_scale=None, losses=None, workspace=None, stream=None):
    """W-Transducer losses (§3.2; variant "force_final" P:116 or "allow_ignore" P:167)."""
    return _call(VARIANTS[variant], logits, targets, logit_lens, target_lens, blank, grads, grad_scale, losses,
                 workspace, stream)


def loss(logits, targets, logit_lens, target_lens, blank=0, variant="rnnt", **kw):
    """Dispatch on variant name: "rnnt" | "force_final" | "allow_ignore"."""
    if variant == "rnnt":
        return rnnt_loss(logits, targets, logit_lens, target_lens, blank, **kw)
    return wrnnt_loss(logits, targets, logit_lens, target_lens, blank, variant, **kw)


def rnnt_loss_timed(logits, targets, logit_lens, target_lens, blank=0, variant="rnnt", events=None, grads=True,
                    grad_scale=None, losses=None, workspace=None, stream=None):
    """rnnt_loss / wrnnt_loss recording 6 torch.cuda.Events: K1 start/end, K3 start/end, K2 start/end
    (see include/rnnt_b200.h; the events must be recorded once beforehand so that their handles exist)."""
    return _call(VARIANTS[variant], logits, targets, logit_lens, target_lens, blank, grads, grad_scale, losses,
                 workspace, stream, events)


def rnnt_viterbi(logits, targets, logit_lens, target_lens, blank=0, variant="rnnt", workspace=None, stream=None):
    """Viterbi forced alignment (best path, ties blank > label > skip).  Returns (best_logp fp32 [B],
    frames int32 [B, Umax] (emission frame of each unit, -1 past U_b), span int32 [B, 2])."""
    if not (isinstance(logits, torch.Tensor) and logits.is_cuda and logits.dtype in DTYPES):
        raise TypeError("logits must be a CUDA float32 / float16 / bfloat16 tensor (no CPU fallback)")
    B, Tmax, Up1, V = logits.shape
    Umax = Up1 - 1
    dev = logits.device
    targets = _as_i32(targets, dev).reshape(B, Umax) if Umax > 0 else None
    logit_lens = _as_i32(logit_lens, dev)
    target_lens = _as_i32(target_lens, dev)
    best = torch.empty(B, dtype=torch.float32, device=dev)
    frames = torch.empty((B, Umax), dtype=torch.int32, device=dev)
    span = torch.empty((B, 2), dtype=torch.int32, device=dev)
    if workspace is None:
        workspace = torch.empty(max(rnnt_workspace_bytes(B, Tmax, Umax), 1), dtype=torch.uint8, device=dev)
    logits = logits.contiguous()  # a named reference keeps any copy alive across the call
    _keep(stream, logits, targets, logit_lens, target_lens, best, frames, span, workspace)
    _check(library.rnnt_viterbi(_ptr(logits), DTYPES[logits.dtype], _ptr(targets), _ptr(logit_lens),
                                _ptr(target_lens), B, Tmax, Umax, V, int(blank), VARIANTS[variant], _ptr(best),
                                _ptr(frames) if Umax > 0 else None, _ptr(span), _ptr(workspace), workspace.numel(),
                                _stream(stream)))
    return best, frames, span


def rnnt_joint_loss(enc, pred, weight, bias, targets, logit_lens, target_lens, blank=0, variant="rnnt",
                    losses=None, workspace=None, stream=None, events=None):
    """Fused joint network + loss (NEXT-4): z = bf16(tanh(enc[:, :, None] + pred[:, None])) @ weight.T + bias
    is reduced on chip (tcgen05 GEMM + log-softmax / Populate epilogue) and never materialised; returns the
    per-utterance losses [B].  enc [B, Tmax, H], pred [B, Umax+1, H], weight [V, H]: CUDA bfloat16; bias [V]
    float32 or None.  events: None or 4 recorded torch.cuda.Events (K6 start / end, K2 start / end)."""
    B, Tmax, Umax, H, V = _check_joint_inputs(enc, pred, weight)
    dev = enc.device
    if bias is not None:
        bias = bias.to(device=dev, dtype=torch.float32).contiguous()
    targets = _as_i32(targets, dev).reshape(B, Umax) if Umax > 0 else None
    logit_lens = _as_i32(logit_lens, dev)
    target_lens = _as_i32(target_lens, dev)
    if losses is None:
        losses = torch.empty(B, dtype=torch.float32, device=dev)
    if workspace is None:
        workspace = torch.empty(max(rnnt_workspace_bytes(B, Tmax, Umax), 1), dtype=torch.uint8, device=dev)
    ev = None
    if events is not None:
        handles = [e.cuda_event for e in events]
        if len(handles) != 4 or not all(handles):
            raise ValueError("need 4 recorded torch.cuda.Events")
        ev = ctypes.cast((ctypes.c_void_p * 4)(*handles), ctypes.c_void_p)
    _keep(stream, bias, targets, logit_lens, target_lens, losses, workspace)
    _check(library.rnnt_joint_loss_ex(_ptr(enc), _ptr(pred), _ptr(weight), _ptr(bias), _ptr(targets),
                                      _ptr(logit_lens), _ptr(target_lens), B, Tmax, Umax, H, V, int(blank),
                                      VARIANTS[variant], _ptr(losses), _ptr(workspace), workspace.numel(),
                                      _stream(stream), ev))
    return losses


def rnnt_joint_loss_grad(enc, pred, weight, bias, targets, logit_lens, target_lens, blank=0, variant="rnnt",
                         workspace=None, stream=None, outputs=None, grad_scale=None, valid_rows=None):
    """Training step of the fused joint (NEXT-4 backward): returns (losses [B], d_enc [B, Tmax, H],
    d_pred [B, Umax+1, H], d_weight [V, H], d_bias [V]), the gradients (fp32) of sum(losses).  Inputs as
    rnnt_joint_loss; bias may be None (then d_bias is still returned, for a zero bias).  outputs: optional
    preallocated (losses, d_enc, d_pred, d_weight, d_bias) fp32 tensors of those shapes.  grad_scale: optional
    [B] per-utterance weights (gradients of sum_b grad_scale[b] * losses[b]; 1/B gives the mean).
    valid_rows: the valid-cell count sum_b T_b (U_b + 1) (the GEMMs then skip the padding; a wrong count gives
    NaN losses); None computes it when both length arrays are on the host, else passes -1 (unknown)."""
    B, Tmax, Umax, H, V = _check_joint_inputs(enc, pred, weight)
    dev = enc.device
    if bias is not None:
        bias = bias.to(device=dev, dtype=torch.float32).contiguous()
    targets = _as_i32(targets, dev).reshape(B, Umax) if Umax > 0 else None
    if valid_rows is None:
        valid_rows = joint_valid_rows(logit_lens, target_lens, Tmax, Umax)
    logit_lens = _as_i32(logit_lens, dev)
    target_lens = _as_i32(target_lens, dev)
    if outputs is None:
        outputs = (torch.empty(B, dtype=torch.float32, device=dev),
                   torch.empty((B, Tmax, H), dtype=torch.float32, device=dev),
                   torch.empty((B, Umax + 1, H), dtype=torch.float32, device=dev),
                   torch.empty((V, H), dtype=torch.float32, device=dev),
                   torch.empty(V, dtype=torch.float32, device=dev))
    if len(outputs) != 5:
        raise ValueError("outputs: (losses, d_enc, d_pred, d_weight, d_bias)")
    losses, d_enc, d_pred, d_weight, d_bias = outputs
    for name, t, shape in (("losses", losses, (B,)), ("d_enc", d_enc, (B, Tmax, H)),
                           ("d_pred", d_pred, (B, Umax + 1, H)), ("d_weight", d_weight, (V, H)),
                           ("d_bias", d_bias, (V,))):
        _check_f32_out(name, t, shape, dev)
    need = int(library.rnnt_joint_grad_workspace_bytes(B, Tmax, Umax, H, V))
    if workspace is None:
        workspace = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    grad_scale = _check_grad_scale(grad_scale, B, dev)
    _keep(stream, bias, targets, logit_lens, target_lens, grad_scale, workspace, *outputs)
    _check(library.rnnt_joint_loss_grad(_ptr(enc), _ptr(pred), _ptr(weight), _ptr(bias), _ptr(targets),
                                        _ptr(logit_lens), _ptr(target_lens), B, Tmax, Umax, H, V, int(blank),
                                        VARIANTS[variant], _ptr(losses), _ptr(d_enc), _ptr(d_pred), _ptr(d_weight),
                                        _ptr(d_bias), _ptr(grad_scale), int(valid_rows), _ptr(workspace),
                                        workspace.numel(), _stream(stream)))
    return losses, d_enc, d_pred, d_weight, d_bias


def joint_valid_rows(logit_lens, target_lens, Tmax, Umax):
    """sum_b T_b (U_b + 1) over the valid utterances, from host lengths (numpy / list / CPU tensor); -1 when
    either array is on the GPU (no device sync here)."""
    if any(isinstance(x, torch.Tensor) and x.is_cuda for x in (logit_lens, target_lens)):
        return -1
    T = np.asarray(logit_lens.numpy() if isinstance(logit_lens, torch.Tensor) else logit_lens, np.int64).ravel()
    U = np.asarray(target_lens.numpy() if isinstance(target_lens, torch.Tensor) else target_lens, np.int64).ravel()
    ok = (T >= 1) & (T <= Tmax) & (U >= 0) & (U <= Umax)
    return int((T * (U + 1))[ok].sum())


def rnnt_joint_viterbi(enc, pred, weight, bias, targets, logit_lens, target_lens, blank=0, variant="rnnt",
                       workspace=None, stream=None):
    """Viterbi forced alignment on the fused joint's logits (K6 + K4; the logits are never written).  Inputs as
    rnnt_joint_loss; returns (best_logp fp32 [B], frames int32 [B, Umax], span int32 [B, 2]) as rnnt_viterbi."""
    B, Tmax, Umax, H, V = _check_joint_inputs(enc, pred, weight)
    dev = enc.device
    if bias is not None:
        bias = bias.to(device=dev, dtype=torch.float32).contiguous()
    targets = _as_i32(targets, dev).reshape(B, Umax) if Umax > 0 else None
    logit_lens = _as_i32(logit_lens, dev)
    target_lens = _as_i32(target_lens, dev)
    best = torch.empty(B, dtype=torch.float32, device=dev)
    frames = torch.empty((B, Umax), dtype=torch.int32, device=dev)
    span = torch.empty((B, 2), dtype=torch.int32, device=dev)
    if workspace is None:
        workspace = torch.empty(max(rnnt_workspace_bytes(B, Tmax, Umax), 1), dtype=torch.uint8, device=dev)
    _keep(stream, bias, targets, logit_lens, target_lens, best, frames, span, workspace)
    _check(library.rnnt_joint_viterbi(_ptr(enc), _ptr(pred), _ptr(weight), _ptr(bias), _ptr(targets),
                                      _ptr(logit_lens), _ptr(target_lens), B, Tmax, Umax, H, V, int(blank),
                                      VARIANTS[variant], _ptr(best), _ptr(frames) if Umax > 0 else None, _ptr(span),
                                      _ptr(workspace), workspace.numel(), _stream(stream)))
    return best, frames, span


def rnnt_lattice_loss(logits, lattices, logit_lens, target_lens, grads=True, losses=None, stream=None):
    """Generic acyclic-lattice loss + logits-gradient (NEXT-3).  ``lattices``: a lattice.LatticeBatch (host
    numpy arrays, copied to the device here) or the dict ``lattice_to_device`` returns.  fp32 logits.
    Returns (losses [B], grads or None)."""
    if not (isinstance(logits, torch.Tensor) and logits.is_cuda and logits.dtype == torch.float32):
        raise TypeError("logits must be a CUDA float32 tensor (no CPU fallback)")
    B, Tmax, Up1, V = logits.shape
    dev = logits.device
    dv = lattices if isinstance(lattices, dict) else lattice_to_device(lattices, dev, Tmax, Up1 - 1)
    if losses is None:
        losses = torch.empty(B, dtype=torch.float32, device=dev)
    if isinstance(grads, str) and grads == "inplace":
        grads = logits
    elif grads is True:
        grads = torch.empty_like(logits)
    elif grads is False:
        grads = None
    need = int(library.rnnt_lattice_workspace_bytes(B, Tmax, Up1 - 1, dv["num_states"], dv["num_arcs"]))
    ws = torch.empty(max(need, 1), dtype=torch.uint8, device=dev)
    logit_lens = _as_i32(logit_lens, dev)    # keep the device copies alive across the call
    target_lens = _as_i32(target_lens, dev)
    _keep(stream, logit_lens, target_lens, losses, grads, ws, *[v for v in dv.values() if isinstance(v, torch.Tensor)])
    _check(library.rnnt_lattice_loss(
        _ptr(logits), _ptr(logit_lens), _ptr(target_lens), B, Tmax, Up1 - 1, V,
        *[_ptr(dv[k]) for k in ("state_off", "lvl_off", "level_off", "in_off", "out_off", "out_arc", "arc_src",
                                "arc_dst", "arc_t", "arc_u", "arc_v", "final_w")],
        _ptr(dv.get("row_off")), _ptr(dv.get("row_arc")),
        dv["num_states"], dv["num_arcs"], _ptr(losses), _ptr(grads), _ptr(ws), ws.numel(), _stream(stream)))
    return losses, grads


def lattice_to_device(L, device="cuda", Tmax=None, Umax=None):
    """Upload a lattice.LatticeBatch once (the dict rnnt_lattice_loss accepts).  With the logits' (Tmax, Umax)
    the row index is uploaded too (one deterministic gradient pass; without it, two float-atomic passes)."""
    dv = {k: torch.from_numpy(getattr(L, k)).to(device) for k in (
        "state_off", "lvl_off", "level_off", "in_off", "out_off", "out_arc", "arc_src", "arc_dst", "arc_t", "arc_u",
        "arc_v", "final_w")}
    dv["num_states"], dv["num_arcs"] = L.num_states, L.num_arcs
    if Tmax is not None:
        row_off, row_arc = L.row_index(Tmax, Umax)
        dv["row_off"] = torch.from_numpy(row_off).to(device)
        dv["row_arc"] = torch.from_numpy(row_arc if row_arc.size else np.zeros(1, np.int32)).to(device)
    return dv


def rnnt_loss_sum(losses, out=None, stream=None):
    """Deterministic fp64 device sum of the per-utterance losses (operand of the cross-rank all-reduce)."""
    if out is None:
        out = torch.empty((), dtype=torch.float64, device=losses.device)
    _check(library.rnnt_loss_sum(_ptr(losses), losses.numel(), _ptr(out), _stream(stream)))
    return out


def rnnt_loss_host(logits_host, targets_host, logit_lens_host, target_lens_host, blank=0, variant="rnnt",
                   losses_host=None, grads_host=None, device_buffer=None, stream=None):
    """Host-buffer entry point: host (ideally pinned) CPU tensors in and out; H2D copies, compute and D2H copies
    of utterance chunks overlap through a 3-slot device ring.  logits_host: float32 / float16 / bfloat16
    [B, Tmax, Umax+1, V] (grads_host, if given, the same type and shape); targets int32 [B, Umax], lengths int32
    [B].  Returns (losses_host, grads_host).  Synchronize the stream before reading them.
    """
    def host(name, t, dtype, shape):
        if not (isinstance(t, torch.Tensor) and not t.is_cuda and t.dtype == dtype and t.is_contiguous()
                and tuple(t.shape) == tuple(shape)):
            raise TypeError(f"{name} must be a contiguous CPU {dtype} tensor of shape {tuple(shape)} "
                            f"(got {getattr(t, 'dtype', type(t))} {tuple(getattr(t, 'shape', ()))})")
        return t

    if not (isinstance(logits_host, torch.Tensor) and logits_host.dim() == 4 and logits_host.dtype in DTYPES):
        raise TypeError("logits_host must be a CPU float32 / float16 / bfloat16 tensor [B, Tmax, Umax+1, V]")
    B, Tmax, Up1, V = logits_host.shape
    Umax = Up1 - 1
    dt = logits_host.dtype
    host("logits_host", logits_host, dt, (B, Tmax, Up1, V))
    host("logit_lens_host", logit_lens_host, torch.int32, (B,))
    host("target_lens_host", target_lens_host, torch.int32, (B,))
    if Umax > 0:
        host("targets_host", targets_host, torch.int32, (B, Umax))
    if losses_host is None:
        losses_host = torch.empty(B, dtype=torch.float32, pin_memory=True)
    host("losses_host", losses_host, torch.float32, (B,))
    if grads_host is not None:
        host("grads_host", grads_host, dt, (B, Tmax, Up1, V))
    need = rnnt_host_buffer_bytes(B, Tmax, Umax, V, dt)
    if device_buffer is None:
        device_buffer = torch.empty(need, dtype=torch.uint8, device="cuda")
    _keep(stream, device_buffer)
    tg = targets_host if Umax > 0 else None
    _check(library.rnnt_loss_host_ex(_ptr(logits_host), DTYPES[dt], _ptr(tg), _ptr(logit_lens_host),
                                     _ptr(target_lens_host), B, Tmax, Umax, V, int(blank), VARIANTS[variant],
                                     _ptr(losses_host), _ptr(grads_host), _ptr(device_buffer),
                                     device_buffer.numel(), _stream(stream)))
    return losses_host, grads_host
