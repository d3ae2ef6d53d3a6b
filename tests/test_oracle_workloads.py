"""Oracle on the BASELINE workloads vs analytic truth, and the synthetic generator's own
contract (SNR, whiteness, determinism, aliasing).  CPU only."""

import math

import numpy as np
import pytest
import torch

from oracle import rootmusic as R
from paper_1910_11872_b200 import synth


def _interior(H, W, M):
    b = int(math.ceil(M / 2))
    m = np.zeros((H, W), bool)
    m[b:H - b, b:W - b] = True
    return m


@pytest.mark.parametrize("M", [8, 9])
def test_c1_closed_form_phase(M):
    """Config 1 (256², noise-free, window 8): wrapped error of the oracle vs the analytic
    phase (carrier + Gaussian) ≤ 1e-3 rad away from the clamped border (BASELINE north_star
    'closed-form phase on noise-free synthetic fringes').  The curvature bias bound
    max|∇²φ|·(M²-4)/24 ≈ 5e-4 keeps this inside 1e-3."""
    w = synth.workload("C1")
    f = synth.make_frame(w, 0).numpy()
    truth = synth.true_phase(w, 0).numpy()
    ph, fl = R.demod_frame(f, M)
    m = _interior(w.H, w.W, M)
    e = np.abs(R.wrap(ph - truth))[m]
    assert e.max() <= 1e-3, e.max()
    assert not np.any(fl[m] & R.PARITY_EXCLUDE_MASK)


def test_c1_plane_variant_exact():
    w = synth.workload("C1plane", H=64, W=64)
    f = synth.make_frame(w, 0).numpy()
    truth = synth.true_phase(w, 0).numpy()
    ph, fl = R.demod_frame(f, 8)
    m = _interior(w.H, w.W, 8)
    assert np.abs(R.wrap(ph - truth))[m].max() < 2e-5


def test_generator_snr_and_whiteness():
    """η: E|η|² = 10^{-SNR/10} within ±0.1 dB over 512² samples; lag-1
    autocorrelation < 0.02 on both axes (AWGN)."""
    w = synth.workload("C2")
    for snr in (0.0, 10.0):
        noisy = synth.make_frame(w, 1, snr_db=snr).to(torch.complex128).numpy()
        clean = synth.make_frame(w, 1, snr_db=None).to(torch.complex128).numpy()
        eta = noisy - clean
        emp = 10 * math.log10(1.0 / np.mean(np.abs(eta) ** 2))
        assert abs(emp - snr) < 0.1
        for ax in (0, 1):
            a = eta - eta.mean()
            b = np.roll(a, 1, axis=ax)
            rho = abs(np.mean(a * np.conj(b))) / np.mean(np.abs(a) ** 2)
            assert rho < 0.02


def test_generator_deterministic_and_keyed_by_frame():
    w = synth.workload("C3", H=64, W=64)
    a = synth.make_stack(w, frames=[0, 5, 9])
    b = synth.make_stack(w, frames=[5])
    assert torch.equal(a[1], b[0])
    assert not torch.equal(a[0], a[1])


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_diffusion_phantom_no_aliasing(name):
    """|ω_c + ∂φ/∂y| < π: the local frequency stays inside the Nyquist band."""
    w = synth.workload(name)
    t1 = w.times[1]
    s = np.arange(w.H) - w.H / 2.0
    prof = synth.DIFF_PHI0 * math.sqrt(synth.DIFF_T1 / t1) * np.exp(
        -(s * synth.PIXEL_PITCH_M) ** 2 / (4 * synth.DIFFUSION_D * t1))
    g = np.max(np.abs(np.diff(prof)))
    assert 2 * math.pi * synth.CARRIER_FY + g < math.pi
    assert g > 0.05   # the phantom is not trivially flat


def test_rmse_decreases_with_snr():
    """Fig. 4 trend: the estimate's error vs truth falls as SNR rises
    (regime check on a 48×48 block of the 512² C2 flow frame, window 11 = paper L=5)."""
    w = synth.workload("C2")
    truth = synth.true_phase(w, 1).numpy()
    yy, xx = np.meshgrid(np.arange(200, 248), np.arange(150, 198), indexing="ij")
    pix = (yy.ravel(), xx.ravel())
    rmse = []
    for snr in (0.0, 10.0, 20.0):
        f = synth.make_frame(w, 1, snr_db=snr).numpy()
        ph, fl = R.demod_frame(f, 11, pixels=pix)
        e = R.wrap(ph - truth[pix])
        rmse.append(math.sqrt(np.mean(e * e)))
    assert rmse[0] > rmse[1] > rmse[2]
    assert rmse[0] < 0.3 and rmse[2] < 0.05
