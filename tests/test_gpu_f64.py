"""GPU parity of row f4's FP64 path (BOS_VARIANT_FP64, alone and with FB): every step of the
pixel in double on the GPU vs the FP64 oracle — a much tighter bar than the FP32 hot path's
north_star tolerance: RMS ≤ 1e-6 rad, max ≤ 2e-5 rad (the float32 output rounding is 2.4e-7
rad at |φ| ≈ π), and the flag bits (including SMALL_GAP, which only this path emits) equal
to the oracle's on ≥ 99.5 % of the pixels."""

import numpy as np
import pytest
import torch

from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth

from .parity_util import assert_excluded_valid, assert_parity

pytestmark = pytest.mark.gpu

DEV = "cuda:0"
RMS64, MAX64 = 1e-6, 2e-5


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    bosrm.lib()


def run64(frames_cpu, M, fb=False, ref=None, omega=False):
    v = bosrm.VARIANT_FP64 | (bosrm.VARIANT_FB if fb else 0)
    r = None if ref is None else torch.as_tensor(ref, dtype=torch.float32).to(DEV)
    out, fl, wx, wy = bosrm.bos_rootmusic_demod_variant(frames_cpu.to(DEV), M, variant=v, ref_phase=r, flags=True,
                                                        omega=omega)
    torch.cuda.synchronize()
    shape = tuple(frames_cpu.shape)
    res = [out.cpu().numpy().reshape(shape), fl.cpu().numpy().reshape(shape)]
    if omega:
        res += [wx.cpu().numpy().reshape(shape), wy.cpu().numpy().reshape(shape)]
    return res


def flag_agreement(g, o):
    return float(np.mean(g == o))


@pytest.mark.parametrize("fb", [False, True])
@pytest.mark.parametrize("M", [3, 4, 8, 11, 17, 24, 32])
def test_f64_ragged_frames(M, fb):
    H, W = (37, 45) if M < 19 else (M + 6, 75)
    f = synth.make_frame(synth.workload("C3", H=H, W=W, seed=M), 5, snr_db=10.0)
    g, gfl, wx, wy = run64(f, M, fb, omega=True)
    o, ofl = R.demod_frame(f.numpy(), M, variant="fb" if fb else "paper")
    assert_parity(g, o, ofl, f"FP64 ragged M={M} fb={fb}", rms_tol=RMS64, max_tol=MAX64)
    assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"FP64 ragged M={M} fb={fb}", variant="fb" if fb else "paper")
    assert flag_agreement(gfl, ofl) >= 0.995, (gfl[gfl != ofl], ofl[gfl != ofl])


@pytest.mark.parametrize("M", [8, 9])
def test_f64_c1_noise_free_full_frame(M):
    """Noise-free frame: near-double roots everywhere; both sides at the √ε root split."""
    w = synth.workload("C1")
    f = synth.make_frame(w, 0)
    g, gfl = run64(f, M)
    o, ofl = R.demod_frame(f.numpy(), M)
    s = assert_parity(g, o, ofl, f"FP64 C1 M={M}", rms_tol=RMS64, max_tol=MAX64)
    assert s["excluded"] == 0, s
    assert flag_agreement(gfl, ofl) >= 0.995


@pytest.mark.parametrize("snr", [0.0, 10.0])
def test_f64_c2_sampled_with_reference_and_omega(snr):
    w = synth.workload("C2")
    st = synth.make_stack(w, snr_db=snr)
    ref, _, _, _ = bosrm.bos_rootmusic_demod_variant(st[0:1].to(DEV), 11, variant=bosrm.VARIANT_FP64)
    g, gfl, wx, wy = run64(st[1], 11, ref=ref[0].cpu(), omega=True)
    rng = np.random.default_rng(int(snr) + 5)
    pix = (rng.integers(0, w.H, 4096), rng.integers(0, w.W, 4096))
    o, ofl = R.demod_stack(st.numpy(), 11, pixels=pix, frame_indices=[1])
    # the GPU subtracts the float32-stored reference: ≤ 2.4e-7 rad more rounding
    assert_parity(g[pix], o[0], ofl[0], f"FP64 C2 snr={snr}", rms_tol=RMS64, max_tol=MAX64)
    win, _ = R.extract_windows(st[1].numpy(), pix[0], pix[1], 11)
    res = R.estimate_windows(win)
    assert_parity(wx[pix], res["omega_x"], res["flags"], "FP64 ω_x", rms_tol=RMS64, max_tol=MAX64)
    assert_parity(wy[pix], res["omega_y"], res["flags"], "FP64 ω_y", rms_tol=RMS64, max_tol=MAX64)


def test_f64_nonfinite_zero_and_errors():
    H = W = 24
    f = synth.make_frame(synth.workload("C1plane", H=H, W=W), 0).clone()
    f[12, 12] = complex(float("nan"), 0.0)
    g, gfl = run64(f, 5)
    o = R.window_offsets(5)
    cover = (np.arange(H) >= 12 - o[-1]) & (np.arange(H) <= 12 - o[0])
    expect = cover[:, None] & cover[None, :]
    assert np.array_equal(np.isnan(g), expect)
    assert np.array_equal((gfl & bosrm.FLAG_NONFINITE) != 0, expect)
    z = torch.zeros(H, W, dtype=torch.complex64)
    g, gfl = run64(z, 5)
    assert np.all(gfl & bosrm.FLAG_LOW_AMPLITUDE)
    d = f.to(DEV)
    out = torch.empty(1, H, W, dtype=torch.float32, device=DEV)
    L = bosrm.lib()
    s = torch.cuda.current_stream().cuda_stream
    assert L.bos_rootmusic_demod_variant(d.data_ptr(), 1, H, W, 8, 0, 3, 4, None, out.data_ptr(), None, None, None,
                                         s) == bosrm.BOS_ERR_UNSUPPORTED


def test_f64_deterministic_and_close_to_fp32_path():
    f = synth.make_frame(synth.workload("C3", H=64, W=96, seed=2), 4, snr_db=10.0).to(DEV)
    a = bosrm.bos_rootmusic_demod_variant(f, 8, variant=bosrm.VARIANT_FP64)[0]
    b = bosrm.bos_rootmusic_demod_variant(f, 8, variant=bosrm.VARIANT_FP64)[0]
    p = bosrm.bos_rootmusic_demod(f, 8)[0]
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    d = np.abs(R.wrap(a.cpu().numpy().astype(np.float64) - p.cpu().numpy()))
    assert np.sqrt(np.mean(d * d)) < 1e-5


@pytest.mark.parametrize("fb", [False, True])
@pytest.mark.parametrize("M,m", [(8, 3), (11, 6), (24, 12), (32, 20)])
def test_f64_spatial_smoothing(M, m, fb):
    """FP64 path with subarray order m (any m ≤ M; the FP32 kernel stops at 16)."""
    H, W = (37, 45) if M < 19 else (M + 6, 75)
    f = synth.make_frame(synth.workload("C3", H=H, W=W, seed=3 * M + m), 5, snr_db=10.0)
    v = bosrm.VARIANT_FP64 | (bosrm.VARIANT_FB if fb else 0)
    out, fl, wx, wy = bosrm.bos_rootmusic_demod_variant(f.to(DEV), M, variant=v, flags=True, subarray_len=m,
                                                        omega=True)
    torch.cuda.synchronize()
    g, gfl = out.cpu().numpy()[0], fl.cpu().numpy()[0]
    o, ofl = R.demod_frame(f.numpy(), M, variant="fb" if fb else "paper", subarray_len=m)
    assert_parity(g, o, ofl, f"FP64 SS M={M} m={m} fb={fb}", rms_tol=RMS64, max_tol=MAX64)
    assert_excluded_valid(f.numpy(), M, g, wx.cpu().numpy()[0], wy.cpu().numpy()[0], ofl, f"FP64 SS M={M} m={m} fb={fb}",
                          variant="fb" if fb else "paper", subarray_len=m)
    assert flag_agreement(gfl, ofl) >= 0.995
