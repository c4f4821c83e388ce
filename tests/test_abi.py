"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every symbol include/rnnt_b200.h
declares, and rejects bad host-checkable arguments with the documented status codes (no device work is
launched on those paths)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rnnt_b200.h")


@pytest.fixture(scope="module")
def rb():
    from paper_2303_10384_b200 import _build
    _build.build()
    import paper_2303_10384_b200
    return paper_2303_10384_b200


def _declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w\s\*]*?\b(\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_entry_points():
    names = _declared_functions()
    for n in ("rnnt_loss", "wrnnt_loss", "rnnt_workspace_bytes", "rnnt_status_string", "rnnt_loss_sum",
              "rnnt_loss_host", "rnnt_host_buffer_bytes", "rnnt_loss_host_ex", "rnnt_host_buffer_bytes_ex",
              "rnnt_version"):
        assert n in names


def test_library_exports_every_declared_symbol(rb):
    lib = ctypes.CDLL(rb.LIB_PATH)
    for name in _declared_functions():
        assert hasattr(lib, name), name
    assert set(rb.EXPORTS) == set(_declared_functions())


def test_version_and_status_strings(rb):
    assert b"sm_100a" in rb.library.rnnt_version()
    for code in range(5):
        assert rb.library.rnnt_status_string(code).startswith(b"RNNT_")


def test_workspace_bytes(rb):
    B, T, U = 3, 50, 7
    ws = rb.rnnt_workspace_bytes(B, T, U)
    cells = B * T * (U + 1)
    expect_min = cells * 4 + (B * (T + U) + 32) * (U + 1) * 16 + B * (T + U) * (U + 1) * (8 + 8) + B * 8
    assert expect_min <= ws <= expect_min + 5 * 256
    assert rb.rnnt_workspace_bytes(0, 1, 0) >= 0
    assert rb.rnnt_workspace_bytes(-1, 1, 0) == 0
    assert rb.rnnt_workspace_bytes(1, 0, 0) == 0
    assert rb.rnnt_host_buffer_bytes(4, 10, 3, 16) >= 4 * 10 * 4 * 16 * 4


def _call_raw(rb, B=2, T=3, U=1, V=4, blank=0, ws_bytes=None, fake=1 << 20, grads=None, logits=None):
    # Fake (never dereferenced) device pointers: every path below returns before any launch.
    P = ctypes.c_void_p
    ws = rb.rnnt_workspace_bytes(max(B, 1), max(T, 1), max(U, 0)) if ws_bytes is None else ws_bytes
    logits = P(fake) if logits is None else logits
    return rb.library.rnnt_loss(logits, P(fake), P(fake), P(fake), B, T, U, V, blank, P(fake), grads, None,
                                P(fake), ws, None)


def test_host_argument_errors(rb):
    INVALID, WS, UNSUP = 1, 2, 3
    assert _call_raw(rb, B=-1) == INVALID
    assert _call_raw(rb, T=0) == INVALID
    assert _call_raw(rb, U=-1) == INVALID
    assert _call_raw(rb, V=1) == INVALID
    assert _call_raw(rb, blank=4) == INVALID
    assert _call_raw(rb, blank=-1) == INVALID
    assert _call_raw(rb, U=4096) == UNSUP  # Umax + 1 > kMaxUp1 = 4096 (rnnt_b200.h)
    assert _call_raw(rb, ws_bytes=16) == WS
    # grads partially overlapping logits (but not equal) is rejected
    assert _call_raw(rb, grads=ctypes.c_void_p((1 << 20) + 4)) == INVALID
    # B == 0 is a no-op success
    assert _call_raw(rb, B=0) == 0
    # null logits
    assert _call_raw(rb, logits=ctypes.c_void_p(0)) == INVALID
    P = ctypes.c_void_p
    assert rb.library.wrnnt_loss(P(1 << 20), P(1 << 20), P(1 << 20), P(1 << 20), 2, 3, 1, 4, 0, P(1 << 20),
                                 None, None, P(1 << 20), 1 << 20, None, 7) == INVALID
    assert rb.library.rnnt_loss_sum(None, 3, P(1 << 20), None) == INVALID


def test_compute_entry_points_refuse_cpu_tensors(rb):
    import torch
    with pytest.raises(TypeError):
        rb.rnnt_loss(torch.zeros(1, 2, 2, 3), torch.ones(1, 1), [2], [1])
