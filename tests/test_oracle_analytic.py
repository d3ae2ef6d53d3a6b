"""Pins of the row-f1 oracle (analytic signal from intensity), CPU only."""

import math

import numpy as np

from oracle import analytic as A
from paper_1910_11872_b200 import synth


def test_integer_bin_cosine_gives_exact_analytic_signal():
    """I = ½ + ½cos(2π(f_x x + f_y y) + φ0) with on-bin carrier: the +1 lobe is one DFT bin,
    so Γ = ¼·e^{j(2π(f_x x+f_y y)+φ0)} exactly; with carrier removal Γ = ¼·e^{jφ0}."""
    H, W, fx, fy, p0 = 64, 128, 16 / 128, 8 / 64, 0.7
    y, x = np.mgrid[0:H, 0:W]
    I = 0.5 + 0.5 * np.cos(2 * np.pi * (fx * x + fy * y) + p0)
    g = A.analytic_signal(I, fx, fy, 0.05)
    assert np.max(np.abs(g - 0.25 * np.exp(1j * (2 * np.pi * (fx * x + fy * y) + p0)))) < 1e-12
    g0 = A.analytic_signal(I, fx, fy, 0.05, remove_carrier=True)
    assert np.max(np.abs(g0 - 0.25 * np.exp(1j * p0))) < 1e-12


def test_smooth_phase_recovered_in_interior():
    """SPEC S:L134 example: carrier 0.125 cycles/px, radius 0.05, a smooth 3-rad Gaussian phase
    → arg Γ ≈ φ in the interior (< 0.05 rad), 8-bit input."""
    H = W = 128
    y, x = np.mgrid[0:H, 0:W]
    g = 3.0 * np.exp(-((x - 64) ** 2 + (y - 64) ** 2) / (2 * 18.0 ** 2))
    I = np.clip(np.round(255 * (0.5 + 0.5 * np.cos(2 * np.pi * 0.125 * x + g))), 0, 255).astype(np.uint8)
    G = A.analytic_signal(I, 0.125, 0.0, 0.05, remove_carrier=True)
    e = np.angle(G * np.exp(-1j * g))
    assert np.max(np.abs(e[24:104, 24:104])) < 0.05


def test_output_spectrum_lives_inside_the_disc():
    rng = np.random.default_rng(1)
    I = rng.integers(0, 256, (40, 56)).astype(np.uint8)
    G = A.analytic_signal(I, 0.2, -0.1, 0.08)
    F = np.fft.fft2(G)
    m = A.lobe_mask(40, 56, 0.2, -0.1, 0.08)
    assert m.sum() > 0
    assert np.max(np.abs(F[~m])) < 1e-10 * np.max(np.abs(F[m]))
    # inside the disc the spectrum is the input's, unchanged
    assert np.allclose(F[m], np.fft.fft2(I / 255.0)[m], atol=1e-9)


def test_intensity_generator_is_uint8_and_keyed_by_frame():
    w = synth.workload("C2", H=48, W=64)
    a = synth.make_intensity_frame(w, 1)
    b = synth.make_intensity_frame(w, 1)
    assert a.dtype.is_floating_point is False and a.shape == (48, 64)
    assert (a == b).all()
    assert not (a == synth.make_intensity_frame(w, 0)).all()
    # carrier + phase recovered from the 8-bit frame (noise-free): arg Γ vs the analytic phase
    w0 = synth.workload("C2", H=128, W=128, snr_db=None)
    i0 = synth.make_intensity_frame(w0, 0).numpy()
    G = A.analytic_signal(i0, synth.CARRIER_FX, synth.CARRIER_FY, 0.05)
    truth = synth.true_phase(w0, 0).numpy()
    e = np.angle(G * np.exp(-1j * truth))
    assert np.max(np.abs(e[16:-16, 16:-16])) < 0.02 and math.isfinite(float(np.abs(G).mean()))
