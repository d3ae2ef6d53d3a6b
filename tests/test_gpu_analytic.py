"""Row f1 on the GPU: the analytic-signal front end (cuFFT + mask/demod kernels) vs the FP64
oracle, and the camera-to-phase pipeline (f1 → root-MUSIC) vs the oracle pipeline."""

import math

import numpy as np
import pytest
import torch

from oracle import analytic as A
from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth

from .parity_util import assert_parity

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    bosrm.lib()


@pytest.mark.parametrize("remove", [False, True])
@pytest.mark.parametrize("shape", [(11, 96, 160), (1, 128, 128), (3, 77, 50)])
def test_analytic_signal_matches_oracle(shape, remove):
    """Element-wise: |Γ_gpu − Γ_oracle| ≤ 2e-5 · max|Γ_oracle| (FP32 FFT vs FP64); 11 frames cover
    a full 8-frame cuFFT batch plus a 3-frame tail; odd sizes cover non-power-of-two FFTs."""
    T, H, W = shape
    w = synth.workload("C2", H=H, W=W, snr_db=10.0)
    fr = torch.stack([synth.make_intensity_frame(w, t) for t in range(T)])
    g = bosrm.bos_analytic_signal(fr.to(DEV), synth.CARRIER_FX, synth.CARRIER_FY, 0.05, remove)
    torch.cuda.synchronize()
    o = A.analytic_signal(fr.numpy(), synth.CARRIER_FX, synth.CARRIER_FY, 0.05, remove)
    err = np.abs(g.cpu().numpy().astype(np.complex128) - o)
    assert err.max() <= 2e-5 * np.abs(o).max(), (err.max(), np.abs(o).max())


@pytest.mark.parametrize("remove", [False, True])
@pytest.mark.parametrize("shape,carrier,radius", [
    ((9, 256, 512), (synth.CARRIER_FX, synth.CARRIER_FY), 0.05),   # 8-frame chunk + 1
    ((2, 1024, 1024), (synth.CARRIER_FX, synth.CARRIER_FY), 0.05), # the bench frame size
    ((3, 64, 2048), (0.47, -0.2), 0.06),                             # carrier near +Nyquist
    ((2, 4096, 16), (-0.25, 0.4), 0.2),                              # tall, few columns, wide disc
    ((1, 2, 4), (0.25, -0.5), 0.3),                                  # minimum sizes
    ((1, 32, 32), (0.2, 0.1), 0.01),                                 # disc between bins: Γ ≡ 0
])
def test_fused_path_matches_oracle(shape, carrier, radius, remove):
    """Power-of-two frames take the fused pruned path (three passes, in-shared-memory FFTs over
    the kept columns only): element-wise within the same FP32-vs-FP64 bound as the cuFFT path."""
    T, H, W = shape
    rng = np.random.default_rng(H * 7 + W)
    fr = torch.from_numpy(rng.integers(0, 256, (T, H, W), dtype=np.uint8))
    if H >= 64 and W >= 64:
        w = synth.workload("C2", H=H, W=W, snr_db=10.0)
        fr = torch.stack([synth.make_intensity_frame(w, t) for t in range(T)])
    fx, fy = carrier
    g = bosrm.bos_analytic_signal(fr.to(DEV), fx, fy, radius, remove)
    torch.cuda.synchronize()
    o = A.analytic_signal(fr.numpy(), fx, fy, radius, remove)
    err = np.abs(g.cpu().numpy().astype(np.complex128) - o)
    assert err.max() <= 2e-5 * max(np.abs(o).max(), 1e-30) or np.abs(o).max() == 0 and err.max() == 0, \
        (err.max(), np.abs(o).max())


@pytest.mark.parametrize("W", [80, 64])
def test_planned_analytic_signal_matches_oracle_and_unplanned(W):
    """The caller-owned plan (bos_analytic_plan_*) on a ragged frame count (2 full 8-frame
    batches + 3 single-frame tail FFTs) equals the per-call-plan path bit for bit and the
    oracle within the FP32 FFT bound; one plan serves calls of different frame counts.
    W = 80: the cuFFT path; W = 64: the fused power-of-two path."""
    T, H = 19, 64
    w = synth.workload("C2", H=H, W=W, snr_db=10.0)
    fr = torch.stack([synth.make_intensity_frame(w, t) for t in range(T)]).to(DEV)
    plan = bosrm.AnalyticPlan(H, W, T)
    for n in (T, 5, 1):
        g = bosrm.bos_analytic_signal_planned(plan, fr[:n], synth.CARRIER_FX, synth.CARRIER_FY, 0.05, True)
        u = bosrm.bos_analytic_signal(fr[:n], synth.CARRIER_FX, synth.CARRIER_FY, 0.05, True)
        torch.cuda.synchronize()
        assert torch.equal(g, u)
    o = A.analytic_signal(fr.cpu().numpy(), synth.CARRIER_FX, synth.CARRIER_FY, 0.05, True)
    g = bosrm.bos_analytic_signal_planned(plan, fr, synth.CARRIER_FX, synth.CARRIER_FY, 0.05, True)
    torch.cuda.synchronize()
    err = np.abs(g.cpu().numpy().astype(np.complex128) - o)
    assert err.max() <= 2e-5 * np.abs(o).max()
    with pytest.raises(ValueError):
        bosrm.bos_analytic_signal_planned(plan, fr[:, :32], synth.CARRIER_FX, synth.CARRIER_FY, 0.05)
    plan.close()


def test_camera_to_phase_pipeline_parity():
    """8-bit C2 pair (reference + flow, 10 dB) → f1 → root-MUSIC stack demod (M = 11) on the
    GPU vs oracle f1 → oracle demod: sampled pixels within the north_star tolerance."""
    w = synth.workload("C2", snr_db=10.0)
    fr = torch.stack([synth.make_intensity_frame(w, t) for t in (0, 1)])
    g = bosrm.bos_analytic_signal(fr.to(DEV), synth.CARRIER_FX, synth.CARRIER_FY, 0.05)
    out, _, _ = bosrm.bos_rootmusic_demod_stack(g, 11, ref_index=0)
    torch.cuda.synchronize()
    o_gamma = A.analytic_signal(fr.numpy(), synth.CARRIER_FX, synth.CARRIER_FY, 0.05).astype(np.complex64)
    rng = np.random.default_rng(3)
    pix = (rng.integers(0, w.H, 4096), rng.integers(0, w.W, 4096))
    o, ofl = R.demod_stack(o_gamma, 11, pixels=pix, frame_indices=[1])
    assert_parity(out[1].cpu().numpy()[pix], o[0], ofl[0], "f1 + demod pipeline")
    # and the recovered flow phase follows the phantom (interior, loose: f1's filter + noise)
    truth = (synth.true_phase(w, 1) - synth.true_phase(w, 0)).numpy()
    e = R.wrap(out[1].cpu().numpy() - truth)[40:-40, 40:-40]
    assert math.sqrt(float(np.mean(e * e))) < 0.15


def test_analytic_signal_rejects_dc_disc():
    fr = torch.zeros(1, 32, 32, dtype=torch.uint8, device=DEV)
    with pytest.raises(bosrm.BosError):
        bosrm.bos_analytic_signal(fr, 0.02, 0.0, 0.05)
