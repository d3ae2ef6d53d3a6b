"""The strip kernels (csrc/demod_strip.cuh: a warp walks down a strip of rows).  Kind 1
(M ≤ 10, 12, 13) slides R_y by one row per pixel in registers and must equal the row kernel
(csrc/demod_kernel.cuh, R_y formed in full per pixel) BITWISE; kind 2 (M = 11, 14…32, no R_y:
implicit power iteration) is checked against the FP64 oracle.  Kind 1 against the row kernel (csrc/demod_kernel.cuh: R_y formed in full per
pixel): R_y(py+1)(i, j) = R_y(py)(i+1, j+1) exactly (Eq.(4), rows ↔ y), every entry is summed
in the same order, so phase, flags and ω maps must be BITWISE identical — on ragged frames,
at every strip height the launcher picks (small launches: S = 4; large: S = 32), with clamped
border rows, non-finite samples and low SNR.  BOS_THREAD_KERNEL=row / =strip forces either
kernel (read per launch; unset, launches too small for 8-row strips run the row kernel).  Both kernels are also checked against the FP64 oracle elsewhere."""

import numpy as np
import pytest
import torch

from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth

from .parity_util import assert_excluded_valid, assert_parity

DEV = "cuda"


def _run(frames, M, monkeypatch, row):
    monkeypatch.setenv("BOS_THREAD_KERNEL", "row" if row else "strip")
    ph, fl, wx, wy = bosrm.bos_rootmusic_demod_ex(frames, M, flags=True, omega=True)
    torch.cuda.synchronize()
    return ph, fl, wx, wy


def _bits(t):
    return t.contiguous().view(torch.int32)


def _assert_same(a, b, what):
    for x, y, name in zip(a, b, ("phase", "flags", "omega_x", "omega_y")):
        if x.dtype == torch.float32:
            x, y = _bits(x), _bits(y)
        diff = (x != y)
        assert not bool(diff.any()), f"{what} {name}: {int(diff.sum())} of {diff.numel()} differ"


@pytest.mark.gpu
@pytest.mark.parametrize("M", [3, 4, 5, 6, 7, 8, 9, 10, 12, 13])
def test_strip_kernel_bitwise_equals_row_kernel_small(M, monkeypatch):
    """Ragged 3-frame stack (H, W not multiples of the strip / 32-column block), 10 dB, 0 dB
    and a NaN sample: the small launch makes the launcher pick the shortest strips (S = 2)."""
    w = synth.workload("C3", H=M + 61, W=M + 90, seed=7)
    fr = torch.stack([synth.make_frame(w, 2, snr_db=10.0), synth.make_frame(w, 3, snr_db=0.0),
                      synth.make_frame(w, 4, snr_db=-5.0)]).to(DEV)
    fr[1, 30, 17] = complex(float("nan"), 0.0)
    a = _run(fr, M, monkeypatch, row=False)
    b = _run(fr, M, monkeypatch, row=True)
    _assert_same(a, b, f"M={M}")
    assert bool(torch.isnan(a[0][1, 30, 17]))


@pytest.mark.gpu
@pytest.mark.parametrize("M", [8, 9, 12, 13])
def test_strip_kernel_bitwise_equals_row_kernel_large(M, monkeypatch):
    """A launch large enough for the full strip height (16 rows) on 1024² frames."""
    w = synth.workload("C3", seed=11, window_len=M)
    fr = synth.make_stack(w, frames=range(1, 21), device=DEV)
    a = _run(fr, M, monkeypatch, row=False)
    b = _run(fr, M, monkeypatch, row=True)
    _assert_same(a, b, f"M={M} 20x1024^2")


@pytest.mark.gpu
def test_strip_kernel_is_the_default_on_large_launches(monkeypatch):
    """Unset BOS_THREAD_KERNEL: a large M = 8 launch runs the strip kernel — the row kernel's
    output is identical, so check through the launch-size rule instead: a 1-frame 64² launch
    (too small for 8-row strips) and a 20-frame 1024² launch both match the forced kernels."""
    monkeypatch.delenv("BOS_THREAD_KERNEL", raising=False)
    w = synth.workload("C3", seed=3)
    fr = synth.make_stack(w, frames=range(1, 21), device=DEV)
    auto = bosrm.bos_rootmusic_demod(fr, 8)[0]
    monkeypatch.setenv("BOS_THREAD_KERNEL", "strip")
    strip = bosrm.bos_rootmusic_demod(fr, 8)[0]
    assert torch.equal(_bits(auto), _bits(strip))


@pytest.mark.gpu
@pytest.mark.parametrize("M", [11] + list(range(14, 33)))
def test_strip_im_kernel_parity(M, monkeypatch):
    """The implicit-power-iteration strip kernel (M = 11, 14…32; its arithmetic differs from the
    row kernel's, so no bitwise comparison): element-by-element parity with the FP64 oracle on a
    ragged 10 dB and a 0 dB frame (forced onto the strip kernel: the small launch gives 2-row
    strips, so strip starts and the row-by-row walk are both exercised), and validity of every
    oracle-excluded pixel ([R15])."""
    monkeypatch.setenv("BOS_THREAD_KERNEL", "strip")
    w = synth.workload("C3", H=M + 37, W=M + 60, seed=13)
    for t, snr in ((2, 10.0), (3, 0.0)):
        f = synth.make_frame(w, t, snr_db=snr)
        g, gfl, wx, wy = bosrm.bos_rootmusic_demod_ex(f.unsqueeze(0).to(DEV), M, flags=True, omega=True)
        g, gfl, wx, wy = (x[0].cpu().numpy() for x in (g, gfl, wx, wy))
        o, ofl = R.demod_frame(f.numpy(), M)
        assert_parity(g, o, ofl, f"strip_rs M={M} {snr} dB", gpu_flags=gfl)
        assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"strip_rs M={M} {snr} dB")
