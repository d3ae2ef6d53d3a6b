"""Row f2 on the GPU: Borůvka/union-find reliability unwrapping vs the sequential FP64 Herráez
oracle — the 2π multiples must agree exactly."""

import math

import numpy as np
import pytest
import torch

from oracle import rootmusic as R
from oracle import unwrap as U
from paper_1910_11872_b200 import bosrm, synth

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    bosrm.lib()


def gpu_k(w):
    t = torch.as_tensor(np.ascontiguousarray(w), dtype=torch.float32)
    u = bosrm.bos_unwrap(t.to(DEV))
    torch.cuda.synchronize()
    u = u.cpu().numpy().astype(np.float64)
    return np.rint((u - t.numpy().astype(np.float64)) / (2 * math.pi)).astype(np.int64), u


@pytest.mark.parametrize("shape", [(1, 1), (1, 37), (29, 1), (2, 2), (33, 47), (64, 64), (128, 96)])
@pytest.mark.parametrize("noise", [0.3, 1.2])
def test_k_maps_equal_oracle(shape, noise):
    rng = np.random.default_rng(shape[0] * 1000 + shape[1])
    H, W = shape
    y, x = np.mgrid[0:H, 0:W]
    truth = 0.8 * x - 0.45 * y + 2.5 * np.sin(x / 7.0) * np.cos(y / 5.0)
    w = U.gamma(truth + rng.normal(0, noise, (H, W))).astype(np.float32)
    kg, _ = gpu_k(w)
    ko = U.unwrap_k(w.astype(np.float64))
    assert np.array_equal(kg, ko), (np.argwhere(kg != ko)[:5], (kg != ko).sum())


@pytest.mark.parametrize("shape", [(48, 512), (512, 40)])
def test_long_component_chains(shape):
    """Reliability falling monotonically across the frame (φ ∝ s³ along the long axis: the second
    differences grow with s), so after the tile phase every component's best edge points the
    same way and the first global round hooks whole rows of tiles into one chain — the case the
    one-launch chain compression (chase_list) walks longest."""
    H, W = shape
    y, x = np.mgrid[0:H, 0:W]
    s = x if W > H else y
    truth = 2e-6 * s.astype(np.float64) ** 3 + 0.05 * (y if W > H else x)
    rng = np.random.default_rng(H + W)
    w = U.gamma(truth + rng.normal(0, 0.05, (H, W))).astype(np.float32)
    kg, _ = gpu_k(w)
    ko = U.unwrap_k(w.astype(np.float64))
    assert np.array_equal(kg, ko), (np.argwhere(kg != ko)[:5], (kg != ko).sum())


def test_smooth_surface_and_in_place_and_stack():
    H, W = 120, 150
    y, x = np.mgrid[0:H, 0:W]
    truths = [12.0 * np.exp(-((x - 70) ** 2 + (y - 60) ** 2) / (2 * 25.0 ** 2)) + 0.2 * x,
              -9.0 * np.exp(-((x - 30) ** 2 + (y - 90) ** 2) / (2 * 20.0 ** 2)) - 0.3 * y]
    w = np.stack([U.gamma(t) for t in truths]).astype(np.float32)
    t = torch.from_numpy(w).to(DEV)
    bosrm.bos_unwrap(t, out=t)                      # in place, two frames
    torch.cuda.synchronize()
    u = t.cpu().numpy().astype(np.float64)
    for j in range(2):
        d = u[j] - truths[j]
        assert np.max(np.abs(d - d.flat[0])) < 1e-4
        assert abs(d.flat[0] / (2 * math.pi) - round(d.flat[0] / (2 * math.pi))) < 1e-5
        assert np.array_equal(np.rint((u[j] - w[j]) / (2 * math.pi)), U.unwrap_k(w[j].astype(np.float64)))


def test_nonfinite_pixels_untouched():
    w = U.gamma(np.linspace(0, 30, 40 * 50).reshape(40, 50)).astype(np.float32)
    w[10, 20] = np.nan
    kg, u = gpu_k(w)
    assert np.isnan(u[10, 20])
    ko = U.unwrap_k(w.astype(np.float64))
    fin = np.isfinite(w)
    assert np.array_equal(kg[fin], ko[fin])


def test_demod_then_unwrap_pipeline():
    """C2 flow frame at 10 dB (M = 11, paper L = 5) → GPU demod → GPU unwrap: the 2π multiples
    equal the oracle unwrap of the same wrapped map, and the recovered flow phase follows the
    ≈22 rad phantom (interior RMSE after removing one global 2πk; Fig. 4 regime)."""
    w = synth.workload("C2", snr_db=10.0)
    stack = synth.make_stack(w)
    out, _, _ = bosrm.bos_rootmusic_demod_stack(stack.to(DEV), 11, ref_index=0)
    unw = bosrm.bos_unwrap(out[1].contiguous())
    torch.cuda.synchronize()
    wrapped = out[1].cpu().numpy()
    k = np.rint((unw.cpu().numpy().astype(np.float64) - wrapped) / (2 * math.pi))
    assert np.array_equal(k, U.unwrap_k(wrapped.astype(np.float64)))
    truth = (synth.true_phase(w, 1) - synth.true_phase(w, 0)).numpy()
    d = (unw.cpu().numpy() - truth)[20:-20, 20:-20]
    d -= 2 * math.pi * np.round(np.median(d) / (2 * math.pi))
    assert math.sqrt(float(np.mean(d * d))) < 0.1
