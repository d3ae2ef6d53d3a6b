"""GPU parity of row f4 (forward–backward averaged covariances, NOT in the paper; DESIGN.md
[R13]): bos_rootmusic_demod_variant(variant=BOS_VARIANT_FB) vs the oracle's
``estimate_windows(..., variant="fb")`` on the same seeded complex64 bytes, both kernels
(thread-per-pixel M ≤ 18, warp-per-pixel M ≥ 19 for FB), same tolerance as the paper path."""

import numpy as np
import pytest
import torch

from oracle import rootmusic as R
from paper_1910_11872_b200 import bosrm, synth

from .parity_util import assert_excluded_valid, assert_parity

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    torch.cuda.init()
    bosrm.lib()


def run_fb(frames_cpu, M, ref=None, omega=False):
    f = frames_cpu.to(DEV)
    r = None if ref is None else torch.as_tensor(ref, dtype=torch.float32).to(DEV)
    out, fl, wx, wy = bosrm.bos_rootmusic_demod_variant(f, M, variant=bosrm.VARIANT_FB, ref_phase=r,
                                                        flags=True, omega=omega)
    torch.cuda.synchronize()
    shape = tuple(frames_cpu.shape)
    res = [out.cpu().numpy().reshape(shape), fl.cpu().numpy().reshape(shape)]
    if omega:
        res += [wx.cpu().numpy().reshape(shape), wy.cpu().numpy().reshape(shape)]
    return res


@pytest.mark.parametrize("M", [3, 4, 5, 7, 8, 9, 11, 12, 15, 16, 17, 18, 19, 20, 23, 24, 28, 31, 32])
def test_fb_ragged_frame_parity(M):
    """10 dB fringe frame, ragged sizes; M ≥ 19 frames are wider than one 32-pixel segment."""
    H, W = (37, 45) if M < 19 else (M + 6, 75)
    f = synth.make_frame(synth.workload("C3", H=H, W=W, seed=M), 5, snr_db=10.0)
    g, gfl, wx, wy = run_fb(f, M, omega=True)
    o, ofl = R.demod_frame(f.numpy(), M, variant="fb")
    # FB on these small frames: mostly clamped windows, whose FB R_x is often near-degenerate
    # ([R13] SMALL_GAP on either axis): bounded on interior windows, border outputs checked
    # for validity ([R15])
    assert_parity(g, o, ofl, f"FB ragged M={M}")
    assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"FB ragged M={M}", variant="fb")
    assert np.all((gfl & bosrm.FLAG_BORDER) == (ofl & R.FLAG_BORDER))


@pytest.mark.parametrize("M,snr", [(8, 0.0), (11, 10.0), (8, 20.0), (24, 10.0)])
def test_fb_c2_sampled(M, snr):
    """C2 (512² flow pair) sampled pixels, reference difference through ref_phase."""
    w = synth.workload("C2")
    stack = synth.make_stack(w, snr_db=snr)
    d = stack.to(DEV)
    ref, _, _, _ = bosrm.bos_rootmusic_demod_variant(d[0:1], M, variant=bosrm.VARIANT_FB)
    out, _, _, _ = bosrm.bos_rootmusic_demod_variant(d[1:2], M, variant=bosrm.VARIANT_FB, ref_phase=ref[0])
    torch.cuda.synchronize()
    rng = np.random.default_rng(int(snr) + 31 * M)
    pix = (rng.integers(0, w.H, 8192), rng.integers(0, w.W, 8192))
    o, ofl = R.demod_stack(stack.numpy(), M, pixels=pix, frame_indices=[1], variant="fb")
    assert_parity(out[0].cpu().numpy()[pix], o[0], ofl[0], f"FB C2 M={M} snr={snr}")


@pytest.mark.parametrize("M", [5, 8, 21])
def test_fb_plane_wave_and_omega(M):
    """Noise-free plane wave: ω maps and phase exact (Eq.(3) model) under FB too."""
    H, W = 40, 70
    wx, wy, a = 0.45, -0.8, 0.3
    y, x = np.mgrid[0:H, 0:W]
    f = torch.from_numpy(np.exp(1j * (wx * x + wy * y + a)).astype(np.complex64))
    g, gfl, ox, oy = run_fb(f, M, omega=True)
    ok = (gfl & (R.PARITY_EXCLUDE_MASK | R.FLAG_BORDER)) == 0
    assert ok.mean() > 0.3
    assert np.max(np.abs(ox - wx)[ok]) < 2e-3 and np.max(np.abs(oy - wy)[ok]) < 2e-3
    assert np.max(np.abs(R.wrap(g - (wx * x + wy * y + a)))[ok]) < 2e-3


def test_fb_matches_paper_variant_statistically():
    """On 20 dB C3 fringes the FB and paper maps agree to well within the noise."""
    f = synth.make_frame(synth.workload("C3", H=128, W=160, seed=4), 7, snr_db=20.0).to(DEV)
    a, fa = bosrm.bos_rootmusic_demod(f, 8, flags=True)
    b, fb, _, _ = bosrm.bos_rootmusic_demod_variant(f, 8, variant=bosrm.VARIANT_FB, flags=True)
    p0, _, _, _ = bosrm.bos_rootmusic_demod_variant(f, 8, variant=bosrm.VARIANT_PAPER)
    torch.cuda.synchronize()
    assert torch.equal(a, p0)        # variant 0 is the paper path, bit for bit
    d = np.abs(R.wrap(a.cpu().numpy() - b.cpu().numpy()))
    assert np.median(d) < 0.01 and d.max() > 0


def test_fb_nonfinite_and_errors():
    H = W = 40
    f = synth.make_frame(synth.workload("C1plane", H=H, W=W), 0).clone()
    f[20, 20] = complex(float("nan"), 0.0)
    for M in (7, 20):
        g, gfl = run_fb(f, M)
        # NaN exactly where the window covers (20, 20): p + o ∋ 20 for o ∈ −⌊(M−1)/2⌋..⌊M/2⌋;
        # in particular nothing leaks along the warp-per-pixel segment (M = 20)
        o = R.window_offsets(M)
        cover = (np.arange(H) >= 20 - o[-1]) & (np.arange(H) <= 20 - o[0])
        expect = cover[:, None] & cover[None, :]
        assert np.array_equal(np.isnan(g), expect)
        assert np.all((gfl & bosrm.FLAG_NONFINITE).astype(bool) == expect)
    d = f.to(DEV)
    out = torch.empty(1, H, W, dtype=torch.float32, device=DEV)
    L = bosrm.lib()
    rc = L.bos_rootmusic_demod_variant(d.data_ptr(), 1, H, W, 8, 0, 3, 7, None, out.data_ptr(), None, None, None,
                                       torch.cuda.current_stream().cuda_stream)
    assert rc == bosrm.BOS_ERR_UNSUPPORTED
    rc = L.bos_rootmusic_demod_variant(d.data_ptr(), 1, H, W, 8, 0, 3, 1, None, None, None, None, None,
                                       torch.cuda.current_stream().cuda_stream)
    assert rc == bosrm.BOS_ERR_INVALID_ARG


def test_fb_deterministic():
    f = synth.make_frame(synth.workload("C3", H=96, W=100, seed=1), 3, snr_db=5.0).to(DEV)
    for M in (8, 24):
        a = bosrm.bos_rootmusic_demod_variant(f, M, variant=bosrm.VARIANT_FB)[0]
        b = bosrm.bos_rootmusic_demod_variant(f, M, variant=bosrm.VARIANT_FB)[0]
        torch.cuda.synchronize()
        assert torch.equal(a, b)
        del a, b


# --------------------------------------------------------------------------------------
# Spatial smoothing (subarray_len m < M), FP32 kernel demod_ss.cuh; m = 3 closed-form quartic
# --------------------------------------------------------------------------------------
def run_ss(frames_cpu, M, m, fb=False, ref=None, omega=False):
    v = bosrm.VARIANT_FB if fb else bosrm.VARIANT_PAPER
    r = None if ref is None else torch.as_tensor(ref, dtype=torch.float32).to(DEV)
    out, fl, wx, wy = bosrm.bos_rootmusic_demod_variant(frames_cpu.to(DEV), M, variant=v, ref_phase=r, flags=True,
                                                        omega=omega, subarray_len=m)
    torch.cuda.synchronize()
    shape = tuple(frames_cpu.shape)
    res = [out.cpu().numpy().reshape(shape), fl.cpu().numpy().reshape(shape)]
    if omega:
        res += [wx.cpu().numpy().reshape(shape), wy.cpu().numpy().reshape(shape)]
    return res


@pytest.mark.parametrize("fb", [False, True])
@pytest.mark.parametrize("M,m", [(4, 3), (5, 3), (8, 3), (8, 5), (11, 7), (16, 8), (17, 16), (24, 3), (24, 12),
                                 (32, 16), (32, 3)])
def test_ss_ragged_frame_parity(M, m, fb):
    H, W = (37, 45) if M < 19 else (M + 6, 75)
    f = synth.make_frame(synth.workload("C3", H=H, W=W, seed=M + m), 5, snr_db=10.0)
    g, gfl, wx, wy = run_ss(f, M, m, fb, omega=True)
    o, ofl = R.demod_frame(f.numpy(), M, variant="fb" if fb else "paper", subarray_len=m)
    assert_parity(g, o, ofl, f"SS ragged M={M} m={m} fb={fb}")
    assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"SS ragged M={M} m={m} fb={fb}",
                          variant="fb" if fb else "paper", subarray_len=m)
    assert np.all((gfl & bosrm.FLAG_BORDER) == (ofl & R.FLAG_BORDER))


@pytest.mark.parametrize("M,m,snr", [(11, 6, 10.0), (8, 3, 0.0), (16, 3, 10.0), (16, 9, 20.0)])
def test_ss_c2_sampled(M, m, snr):
    w = synth.workload("C2")
    stack = synth.make_stack(w, snr_db=snr)
    d = stack.to(DEV)
    ref = bosrm.bos_rootmusic_demod_variant(d[0:1], M, variant=0, subarray_len=m)[0]
    out = bosrm.bos_rootmusic_demod_variant(d[1:2], M, variant=0, ref_phase=ref[0], subarray_len=m)[0]
    torch.cuda.synchronize()
    rng = np.random.default_rng(int(snr) + 7 * M + m)
    pix = (rng.integers(0, w.H, 8192), rng.integers(0, w.W, 8192))
    o, ofl = R.demod_stack(stack.numpy(), M, pixels=pix, frame_indices=[1], subarray_len=m)
    assert_parity(out[0].cpu().numpy()[pix], o[0], ofl[0], f"SS C2 M={M} m={m} snr={snr}")


@pytest.mark.parametrize("M,m", [(8, 3), (9, 3), (8, 6)])
def test_ss_noise_free_c1(M, m):
    """Noise-free frames: the quartic / polynomial has a double root on the circle."""
    w = synth.workload("C1")
    f = synth.make_frame(w, 0)
    g, gfl = run_ss(f, M, m)
    o, ofl = R.demod_frame(f.numpy(), M, subarray_len=m)
    s = assert_parity(g, o, ofl, f"SS C1 M={M} m={m}")
    assert s["excluded"] == 0, s


@pytest.mark.parametrize("M,m", [(8, 3), (12, 3), (20, 7)])
def test_ss_plane_wave_and_omega(M, m):
    H, W = 40, 70
    wx, wy, a = -0.9, 0.55, 1.3
    y, x = np.mgrid[0:H, 0:W]
    f = torch.from_numpy(np.exp(1j * (wx * x + wy * y + a)).astype(np.complex64))
    g, gfl, ox, oy = run_ss(f, M, m, omega=True)
    ok = (gfl & (R.PARITY_EXCLUDE_MASK | R.FLAG_BORDER)) == 0
    assert ok.mean() > 0.3
    assert np.max(np.abs(ox - wx)[ok]) < 2e-3 and np.max(np.abs(oy - wy)[ok]) < 2e-3
    assert np.max(np.abs(R.wrap(g - (wx * x + wy * y + a)))[ok]) < 2e-3


def test_ss_argument_errors_and_nan():
    H = W = 40
    f = synth.make_frame(synth.workload("C1plane", H=H, W=W), 0).clone()
    f[20, 20] = complex(float("nan"), 0.0)
    g, gfl = run_ss(f, 9, 3)
    o = R.window_offsets(9)
    cover = (np.arange(H) >= 20 - o[-1]) & (np.arange(H) <= 20 - o[0])
    assert np.array_equal(np.isnan(g), cover[:, None] & cover[None, :])
    d = f.to(DEV)
    out = torch.empty(1, H, W, dtype=torch.float32, device=DEV)
    L = bosrm.lib()
    s = torch.cuda.current_stream().cuda_stream
    for m, rc in ((2, bosrm.BOS_ERR_INVALID_ARG), (9, bosrm.BOS_ERR_INVALID_ARG), (17, bosrm.BOS_ERR_UNSUPPORTED)):
        M = 8 if m != 17 else 20
        assert L.bos_rootmusic_demod_variant(d.data_ptr(), 1, H, W, M, m, 3, 0, None, out.data_ptr(), None, None, None,
                                             s) == rc, (M, m)
