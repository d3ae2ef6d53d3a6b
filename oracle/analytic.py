"""FP64 oracle for SURVEY §8 row f1: the analytic fringe signal from intensity frames.

TEST INFRASTRUCTURE, NOT PRODUCT CODE (see ``oracle/__init__.py``).

P:L80-81 (Section 2): "by using bandpass filtering and carrier removal, the analytic or
complex fringe signal [Eq.(1)] is obtained".  The paper names no filter; the reading
([R11]) is SPEC's hard circular mask around the +1 lobe: per frame
  I/255 → 2-D DFT → keep bins with |f − (f_x, f_y)| ≤ r → inverse DFT → optionally
  × e^{−j2π(f_x x + f_y y)}  (carrier removal).
Bin frequencies follow ``numpy.fft.fftfreq`` (k/N, then (k−N)/N).  The DFT is
``numpy.fft.fft2`` (a library primitive used as one step).
"""

from __future__ import annotations

import numpy as np


def lobe_mask(H: int, W: int, fx: float, fy: float, radius: float) -> np.ndarray:
    """Boolean [H,W]: DFT bins inside the disc of radius r around (f_x, f_y) cycles/px."""
    fxs = np.fft.fftfreq(W)
    fys = np.fft.fftfreq(H)
    d2 = (fxs[None, :] - fx) ** 2 + (fys[:, None] - fy) ** 2
    return d2 <= radius * radius


def analytic_signal(frames, fx: float, fy: float, radius: float, remove_carrier: bool = False) -> np.ndarray:
    """frames: uint8 (scaled by 1/255) or float intensities, [H,W] or [T,H,W] → complex128."""
    a = np.asarray(frames)
    I = a.astype(np.float64) / 255.0 if a.dtype == np.uint8 else a.astype(np.float64)
    H, W = I.shape[-2:]
    F = np.fft.fft2(I, axes=(-2, -1))
    G = np.fft.ifft2(F * lobe_mask(H, W, fx, fy, radius), axes=(-2, -1))
    if remove_carrier:
        y, x = np.mgrid[0:H, 0:W]
        G = G * np.exp(-2j * np.pi * (fx * x + fy * y))
    return G
