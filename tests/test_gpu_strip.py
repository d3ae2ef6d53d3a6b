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


@pytest.mark.gpu
@pytest.mark.parametrize("M", [3, 8, 11, 13, 16, 24, 32])
def test_strip_kernels_minimum_and_thin_frames(M, monkeypatch):
    """Edge shapes on the forced strip kernels: the smallest legal frame (H = W = M), a frame
    one column wide of a 32-column block past a block boundary (W = 33), a single strip row
    (H = M) against many rows, several frames in one launch — parity with the oracle on every
    pixel (all windows clamped), and the kind-1 kernel still bitwise the row kernel."""
    for H, W, T in ((M, M, 2), (M + 5, 33, 3), (M, 70, 2)):
        w = synth.workload("C3", H=H, W=W, seed=17)
        fr = torch.stack([synth.make_frame(w, t + 1, snr_db=15.0) for t in range(T)])
        monkeypatch.setenv("BOS_THREAD_KERNEL", "strip")
        g, gfl, wx, wy = (x.cpu().numpy() for x in bosrm.bos_rootmusic_demod_ex(fr.to(DEV), M, flags=True))
        for t in range(T):
            o, ofl = R.demod_frame(fr[t].numpy(), M)
            assert_parity(g[t], o, ofl, f"strip M={M} {H}x{W} t={t}", gpu_flags=gfl[t], max_interior_excluded_frac=1.0)
            assert_excluded_valid(fr[t].numpy(), M, g[t], wx[t], wy[t], ofl, f"strip M={M} {H}x{W} t={t}")
        if M <= 10 or M in (12, 13):
            b = _run(fr.to(DEV), M, monkeypatch, row=True)
            a = _run(fr.to(DEV), M, monkeypatch, row=False)
            _assert_same(a, b, f"M={M} {H}x{W}")


@pytest.mark.gpu
@pytest.mark.parametrize("M", [17, 20, 24, 28])
def test_strip_fb_kernel_parity(M, monkeypatch):
    """Row f4's forward–backward variant on the implicit strip kernel (M = 17…28): FB(R_y) and
    FB(S) applied from the tile, two starts per axis — parity with the oracle's FB variant
    ([R13]) on a ragged 10 dB and a 0 dB frame, and validity of the excluded pixels."""
    monkeypatch.setenv("BOS_THREAD_KERNEL", "strip")
    w = synth.workload("C3", H=M + 29, W=M + 45, seed=19)
    for t, snr in ((2, 10.0), (3, 0.0)):
        f = synth.make_frame(w, t, snr_db=snr)
        g, gfl, wx, wy = bosrm.bos_rootmusic_demod_variant(f.unsqueeze(0).to(DEV), M, variant=bosrm.VARIANT_FB,
                                                            flags=True, omega=True)
        g, gfl, wx, wy = (x[0].cpu().numpy() for x in (g, gfl, wx, wy))
        o, ofl = R.demod_frame(f.numpy(), M, variant="fb")
        assert_parity(g, o, ofl, f"strip FB M={M} {snr} dB", gpu_flags=gfl)
        assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"strip FB M={M} {snr} dB", variant="fb")
