"""CPU oracle for the RNN-T / W-RNNT loss and logits-gradient (arXiv 2303.10384).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  The product package
(``paper_2303_10384_b200``) never imports it and shares no code with it.

Two independent oracles live here:

* ``rnnt_oracle.c`` -- the plain double-precision lattice forward-backward (Eq.(1) P:54-56,
  §2.3, §3.2, §4.3), loaded through ctypes by the wrappers below.
* ``brute.py`` -- exhaustive enumeration of every alignment path over an explicit arc list, with exact
  rational arithmetic for uniform / rational inputs.  It pins the C oracle on tiny inputs.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "rnnt_oracle.c")
_LIB_PATH = os.path.join(_HERE, "_build", "librnnt_oracle.so")

VARIANTS = {"rnnt": 0, "force_final": 1, "allow_ignore": 2}

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (double precision, OpenMP over utterances)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11", "-Wall",
                        "-o", tmp, _SRC, "-lm"], check=True)
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.c_void_p
            i = ctypes.c_int
            lib.rnnt_oracle_utterance.argtypes = [P, i, i, i, i, i, P, i, i, P, P, P, P, P, P, P]
            lib.rnnt_oracle_utterance.restype = i
            lib.rnnt_oracle_batch.argtypes = [P, P, P, P, i, i, i, i, i, i, P, P, i]
            lib.rnnt_oracle_batch.restype = i
            lib.rnnt_oracle_viterbi.argtypes = [P, i, i, i, i, i, P, i, i, P, P, P]
            lib.rnnt_oracle_viterbi.restype = i
            lib.rnnt_oracle_max_threads.argtypes = []
            lib.rnnt_oracle_max_threads.restype = i
            _lib = lib
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def utterance(z, T, U, y, blank=0, variant="rnnt", grad=True, tables=False):
    """One utterance.  ``z``: float32 [Tmax, Umax+1, V] logits block; ``y``: int32 targets (len >= U).

    Returns a dict with ``loss`` (= -logP), ``logp_beta`` (= beta(0,0)), ``grad`` (float64, same shape
    as z, or None) and, if ``tables``, ``alpha``, ``beta``, ``occ_b``, ``occ_y`` ([T, U+1] float64).
    """
    lib = _load()
    z = np.ascontiguousarray(z, dtype=np.float32)
    Tmax, Up1max, V = z.shape
    y = np.ascontiguousarray(np.asarray(y, dtype=np.int32).reshape(-1))
    if y.size == 0:
        y = np.zeros(1, np.int32)
    loss = np.zeros(1, np.float64)
    lpb = np.zeros(1, np.float64)
    g = np.zeros(z.shape, np.float64) if grad else None
    tabs = [np.zeros((max(T, 0), max(U + 1, 0)), np.float64) if tables else None for _ in range(4)]
    lib.rnnt_oracle_utterance(_ptr(z), Tmax, Up1max - 1, V, int(T), int(U), _ptr(y), int(blank),
                              VARIANTS[variant], _ptr(loss), _ptr(g), *[_ptr(t) for t in tabs], _ptr(lpb))
    out = {"loss": float(loss[0]), "logp_beta": float(lpb[0]), "grad": g}
    if tables:
        out.update(alpha=tabs[0], beta=tabs[1], occ_b=tabs[2], occ_y=tabs[3])
    return out


def batch(z, y, T_b, U_b, blank=0, variant="rnnt", grad=True, nthreads=1):
    """A padded batch: z float32 [B, Tmax, Umax+1, V]; y int32 [B, Umax]; lengths int32 [B].

    Returns (losses float64 [B], grads float64 like z or None).
    """
    lib = _load()
    z = np.ascontiguousarray(z, dtype=np.float32)
    B, Tmax, Up1max, V = z.shape
    Umax = Up1max - 1
    y = np.ascontiguousarray(np.asarray(y, dtype=np.int32).reshape(B, Umax))
    if Umax == 0:
        y = np.zeros((B, 1), np.int32)
    T_b = np.ascontiguousarray(T_b, dtype=np.int32)
    U_b = np.ascontiguousarray(U_b, dtype=np.int32)
    losses = np.zeros(B, np.float64)
    g = np.zeros(z.shape, np.float64) if grad else None
    lib.rnnt_oracle_batch(_ptr(z), _ptr(y), _ptr(T_b), _ptr(U_b), B, Tmax, Umax, V, int(blank),
                          VARIANTS[variant], _ptr(losses), _ptr(g), int(nthreads))
    return losses, g


def viterbi(z, T, U, y, blank=0, variant="rnnt"):
    """Best alignment of one utterance (max-plus over the same lattice; reading R21 tie-break).

    Returns (best log-score, frames int32 [U] = emission frame of each unit, span (first, last frame)).
    """
    lib = _load()
    z = np.ascontiguousarray(z, dtype=np.float32)
    Tmax, Up1max, V = z.shape
    y = np.ascontiguousarray(np.asarray(y, dtype=np.int32).reshape(-1))
    if y.size == 0:
        y = np.zeros(1, np.int32)
    best = np.zeros(1, np.float64)
    frames = np.full(max(Up1max - 1, 1), -1, np.int32)
    span = np.full(2, -1, np.int32)
    lib.rnnt_oracle_viterbi(_ptr(z), Tmax, Up1max - 1, V, int(T), int(U), _ptr(y), int(blank),
                            VARIANTS[variant], _ptr(best), _ptr(frames), _ptr(span))
    return float(best[0]), frames[:U].copy(), (int(span[0]), int(span[1]))


def max_threads() -> int:
    return int(_load().rnnt_oracle_max_threads())
