"""C-ABI boundary checks that need no GPU: the library loads, exports every function the
header declares, and its host-only paths (error codes, sizes, strings) behave as documented.
No compute call is made here (those are the -m gpu tests)."""

import ctypes
import os
import re

import pytest

from paper_1910_11872_b200 import bosrm

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bos_rootmusic.h")


def header_functions():
    with open(HEADER) as fh:
        src = fh.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bos_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    if not os.path.exists(bosrm.LIB_PATH):
        from paper_1910_11872_b200 import build
        build.build()
    return bosrm.lib()


def test_header_declares_expected_api():
    names = header_functions()
    assert names == sorted(bosrm.SIGNATURES), names


def test_library_exports_every_declared_symbol(L):
    for name in header_functions():
        assert hasattr(L, name), name
        assert getattr(L, name) is not None


def test_strerror_and_version(L):
    for code in (0, -1, -2, -3, 42):
        s = bosrm.bos_strerror(code)
        assert isinstance(s, str) and s
    assert bosrm.bos_strerror(0) == "ok"
    assert bosrm.bos_abi_version() >> 16 == 1


def test_workspace_bytes(L):
    H, W, c = 100, 64, 3
    plane = H * W

    def al(v):
        return (v + 255) // 256 * 256

    expect = al(plane * 4) + 2 * (al(c * plane * 8) + al(c * plane * 4) + al(c * plane))
    assert bosrm.bos_rootmusic_host_workspace_bytes(H, W, c, True) == expect
    expect_nf = al(plane * 4) + 2 * (al(c * plane * 8) + al(c * plane * 4))
    assert bosrm.bos_rootmusic_host_workspace_bytes(H, W, c, False) == expect_nf
    assert bosrm.bos_rootmusic_host_workspace_bytes(0, W, c, True) == 0


def test_error_codes_without_device(L):
    """Argument validation happens before any CUDA call."""
    f = L.bos_rootmusic_demod
    # model_order != 3 → UNSUPPORTED (D3 / [R3])
    assert f(None, 1, 64, 64, 8, 2, None, None, None, None) == bosrm.BOS_ERR_UNSUPPORTED
    # window_len out of range
    assert f(None, 1, 64, 64, 2, 3, None, None, None, None) == bosrm.BOS_ERR_INVALID_ARG
    assert f(None, 1, 64, 64, 33, 3, None, None, None, None) == bosrm.BOS_ERR_UNSUPPORTED
    # frame smaller than the window, no frames, NULL pointers
    assert f(None, 1, 7, 64, 8, 3, None, None, None, None) == bosrm.BOS_ERR_INVALID_ARG
    assert f(None, 0, 64, 64, 8, 3, None, None, None, None) == bosrm.BOS_ERR_INVALID_ARG
    assert f(None, 1, 64, 64, 8, 3, None, None, None, None) == bosrm.BOS_ERR_INVALID_ARG
    # aliasing: out overlaps frames (checked before pointer attributes)
    buf = ctypes.create_string_buffer(64 * 64 * 8)
    p = ctypes.addressof(buf)
    assert f(p, 1, 64, 64, 8, 3, None, p + 16, None, None) == bosrm.BOS_ERR_INVALID_ARG
    s = L.bos_rootmusic_demod_stack
    assert s(None, 2, 64, 64, 8, 3, 5, None, None, None, None) == bosrm.BOS_ERR_INVALID_ARG
    h = L.bos_rootmusic_demod_stack_host
    assert h(None, 2, 64, 64, 8, 3, 0, None, None, None, 0, 1, None) == bosrm.BOS_ERR_INVALID_ARG
    assert h(None, 2, 64, 64, 8, 4, 0, None, None, None, 0, 1, None) == bosrm.BOS_ERR_UNSUPPORTED


def test_binding_rejects_cpu_tensors(L):
    import torch
    with pytest.raises(ValueError):
        bosrm.bos_rootmusic_demod(torch.zeros(1, 16, 16, dtype=torch.complex64))


def test_product_path_does_not_import_oracle():
    """The product package never imports oracle/ (test infrastructure only)."""
    pkg = os.path.join(ROOT, "paper_1910_11872_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(dirpath, fn), encoding="utf-8") as fh:
                    src = fh.read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), fn


def test_index_gradient_argument_errors(L):
    g = L.bos_index_gradient
    assert g(None, 10, 1.333, 1.0, 1e4, 0.01, None, None) == bosrm.BOS_ERR_INVALID_ARG
    buf = ctypes.create_string_buffer(64)
    p = ctypes.addressof(buf)
    assert g(p, 0, 1.333, 1.0, 1e4, 0.01, p, None) == bosrm.BOS_ERR_INVALID_ARG
    assert g(p, 4, 1.333, 0.0, 1e4, 0.01, p, None) == bosrm.BOS_ERR_INVALID_ARG
    assert g(p, 4, 1.333, 1.0, -1.0, 0.01, p, None) == bosrm.BOS_ERR_INVALID_ARG


def test_vertical_profile_argument_errors(L):
    f = L.bos_vertical_profile
    buf = ctypes.create_string_buffer(4096)
    p = ctypes.addressof(buf)
    assert f(None, 1, 4, 4, p, None) == bosrm.BOS_ERR_INVALID_ARG
    assert f(p, 0, 4, 4, p + 2048, None) == bosrm.BOS_ERR_INVALID_ARG
    assert f(p, 1, 4, 4, p + 8, None) == bosrm.BOS_ERR_INVALID_ARG          # overlap
    assert f(p, 1, 4, 4, p + 2048, None) == bosrm.BOS_ERR_INVALID_ARG       # host pointers


def test_analytic_signal_argument_errors(L):
    f = L.bos_analytic_signal
    buf = ctypes.create_string_buffer(4096)
    p = ctypes.addressof(buf)
    assert f(None, 1, 16, 16, 0.125, 0.0, 0.05, 0, p, p, 16, None) == bosrm.BOS_ERR_INVALID_ARG
    # the disc around the carrier must exclude DC
    assert f(p, 1, 16, 16, 0.03, 0.0, 0.05, 0, p + 1024, p, 16, None) == bosrm.BOS_ERR_INVALID_ARG
    # carrier beyond Nyquist, non-positive radius
    assert f(p, 1, 16, 16, 0.7, 0.0, 0.05, 0, p + 1024, p, 16, None) == bosrm.BOS_ERR_INVALID_ARG
    assert f(p, 1, 16, 16, 0.2, 0.0, 0.0, 0, p + 1024, p, 16, None) == bosrm.BOS_ERR_INVALID_ARG


def test_analytic_plan_argument_errors(L):
    h = ctypes.c_void_p()
    assert L.bos_analytic_plan_create(1, 16, 4, ctypes.byref(h), None) == bosrm.BOS_ERR_INVALID_ARG
    assert L.bos_analytic_plan_create(16, 16, 0, ctypes.byref(h), None) == bosrm.BOS_ERR_INVALID_ARG
    assert L.bos_analytic_plan_create(16, 16, 4, None, None) == bosrm.BOS_ERR_INVALID_ARG
    buf = ctypes.create_string_buffer(64)
    p = ctypes.addressof(buf)
    assert L.bos_analytic_signal_planned(None, p, 1, 0.125, 0.0, 0.05, 0, p, p, 16, None) == bosrm.BOS_ERR_INVALID_ARG
    assert L.bos_analytic_plan_destroy(None) == bosrm.BOS_OK


def test_unwrap_workspace_and_errors(L):
    n = 100 * 64
    al = lambda v: (v + 255) // 256 * 256  # noqa: E731

    def edges(n):       # two crossing-edge lists (2n ids), filter flag bytes, per-block counts/offsets,
        nb = (2 * n + 2047) // 2048     # and the per-edge (root, root, key) records of the edge passes
        return 2 * al(4 * 2 * n) + al(nb * 256) + 2 * al(4 * nb) + al(16 * 2 * n)
    expect = al(8 * n) + 5 * al(4 * n) + al(8 * n) + al(4 * n) + al(16) + al(8) + al(4) + edges(n)
    assert L.bos_unwrap_workspace_bytes(100, 64, 1) == expect
    n3 = 3 * n
    expect3 = al(8 * n3) + 5 * al(4 * n3) + al(8 * n3) + al(4 * n3) + al(16) + al(24) + al(12) + edges(n3)
    assert L.bos_unwrap_workspace_bytes(100, 64, 3) == expect3
    assert L.bos_unwrap_workspace_bytes(0, 5, 1) == 0
    assert L.bos_unwrap(None, 1, 8, 8, None, None, 0, None) == bosrm.BOS_ERR_INVALID_ARG
