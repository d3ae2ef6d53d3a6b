"""GPU parity: the CUDA path (through the C ABI) vs the FP64 oracle on the same seeded
complex64 bytes.  Tolerance (BASELINE north_star): RMS ≤ 1e-3 rad, max ≤ 1e-2 rad of the
wrapped error over pixels the oracle does not flag (bits 0-4)."""

import math

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


def _interior(H, W, M):
    b = int(math.ceil(M / 2))
    m = np.zeros((H, W), bool)
    m[b:H - b, b:W - b] = True
    return m


def run_gpu(frames_cpu, M, ref=None, flags=True):
    """[H,W] (or [T,H,W]) CPU frames → GPU phase/flags with the same shape."""
    f = frames_cpu.to(DEV)
    r = None if ref is None else torch.as_tensor(ref, dtype=torch.float32).to(DEV)
    out, fl = bosrm.bos_rootmusic_demod(f, M, ref_phase=r, flags=flags)
    torch.cuda.synchronize()
    shape = tuple(frames_cpu.shape)
    return out.cpu().numpy().reshape(shape), (fl.cpu().numpy().reshape(shape) if fl is not None else None)


def run_gpu_ex(frame_cpu, M):
    """[H,W] CPU frame → GPU (α, flags, ω_x, ω_y) maps (raw α) through bos_rootmusic_demod_ex."""
    out, fl, wx, wy = bosrm.bos_rootmusic_demod_ex(frame_cpu.to(DEV), M, flags=True)
    torch.cuda.synchronize()
    shape = tuple(frame_cpu.shape)
    return tuple(t.cpu().numpy().reshape(shape) for t in (out, fl, wx, wy))


# ------------------------------------------------------------------------------- C1
@pytest.mark.parametrize("M", [8, 9])
def test_c1_full_frame_parity_and_closed_form(M):
    w = synth.workload("C1")
    f = synth.make_frame(w, 0)
    g, gfl = run_gpu(f, M)
    o, ofl = R.demod_frame(f.numpy(), M)
    s = assert_parity(g, o, ofl, f"C1 M={M}", gpu_flags=gfl)
    assert s["n"] == 256 * 256 and s["excluded"] == 0
    assert s["gpu_only_flagged_frac"] == 0.0
    truth = synth.true_phase(w, 0).numpy()
    m = _interior(256, 256, M)
    assert np.abs(R.wrap(g - truth))[m].max() <= 1e-3
    assert np.all((gfl & bosrm.FLAG_BORDER) == (ofl & R.FLAG_BORDER))


def test_c1_plane_variant():
    w = synth.workload("C1plane")
    f = synth.make_frame(w, 0)
    g, _ = run_gpu(f, 8, flags=False)
    o, ofl = R.demod_frame(f.numpy(), 8)
    s = assert_parity(g, o, ofl, "C1plane")
    assert s["excluded"] == 0


# ------------------------------------------------------------------------------- C2
@pytest.mark.parametrize("M,snr,full", [(11, 0.0, True), (8, 0.0, False), (11, 10.0, False),
                                        (8, 20.0, False), (11, 5.0, False), (8, 15.0, False)])
def test_c2_pair_parity(M, snr, full):
    """512² reference + flow pair (carrier-only reference) through the stack entry point."""
    w = synth.workload("C2")
    stack = synth.make_stack(w, snr_db=snr)
    out, fl, ref = bosrm.bos_rootmusic_demod_stack(stack.to(DEV), M, ref_index=0, flags=True)
    torch.cuda.synchronize()
    g = out.cpu().numpy()
    assert np.all(g[0][np.isfinite(g[0])] == 0.0)
    if full:
        pix = None
    else:
        rng = np.random.default_rng(int(snr * 10) + M)
        pix = (rng.integers(0, w.H, 16384), rng.integers(0, w.W, 16384))
    o, ofl = R.demod_stack(stack.numpy(), M, pixels=pix, frame_indices=[1])
    gg = g[1] if pix is None else g[1][pix]
    assert_parity(gg, o[0], ofl[0], f"C2 M={M} snr={snr}")


# ------------------------------------------------------------------- ragged / all M
@pytest.mark.parametrize("M", list(range(3, 33)))
def test_all_window_lengths_ragged_frame(M):
    """Every instantiated M on a ragged frame (not a multiple of the 32×4 tile; for the
    warp-per-pixel kernel (M ≥ 17) wider than one 32-pixel segment, so the sliding R_y
    update runs)."""
    w = synth.workload("C2", H=37, W=45, seed=M)
    H, W = (37, 45) if M < 19 else (M + 6, 75)
    # smooth carrier fringe with mild phase, 10 dB
    f = synth.make_frame(synth.workload("C3", H=H, W=W, seed=M), 5, snr_db=10.0)
    g, gfl, wx, wy = run_gpu_ex(f, M)
    o, ofl = R.demod_frame(f.numpy(), M)
    # for M ≥ 17 almost every window of this small frame is clamped (repeated rows/columns),
    # which the oracle more often flags (AMBIGUOUS): bounded on interior windows, and every
    # excluded pixel's output is checked for validity instead ([R15])
    s = assert_parity(g, o, ofl, f"ragged M={M}", gpu_flags=gfl)
    assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"ragged M={M}")
    assert s["gpu_only_flagged_frac"] <= 0.01, s
    assert np.all((gfl & bosrm.FLAG_BORDER) == (ofl & R.FLAG_BORDER))
    del w


def test_minimum_frame_equals_window():
    for M in (3, 8, 16, 17, 32):
        f = synth.make_frame(synth.workload("C3", H=M, W=M, seed=2), 3, snr_db=20.0)
        g, _, wx, wy = run_gpu_ex(f, M)
        o, ofl = R.demod_frame(f.numpy(), M)
        assert_parity(g, o, ofl, f"min M={M}")
        assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"min M={M}")


def test_nonfinite_zero_and_constant_inputs():
    H = W = 40
    f = synth.make_frame(synth.workload("C1plane", H=H, W=W), 0).clone()
    f[20, 20] = complex(float("nan"), 0.0)
    g, gfl = run_gpu(f, 7)
    assert np.isnan(g[20, 20]) and gfl[20, 20] & bosrm.FLAG_NONFINITE
    assert np.isnan(g[17, 23]) and gfl[17, 23] & bosrm.FLAG_NONFINITE
    assert np.isfinite(g[5, 5]) and not (gfl[5, 5] & bosrm.FLAG_NONFINITE)
    z = torch.zeros(H, W, dtype=torch.complex64)
    g, gfl = run_gpu(z, 7)
    assert np.all(gfl & (bosrm.FLAG_LOW_AMPLITUDE | bosrm.FLAG_NONCONVERGED))
    c = torch.full((H, W), complex(math.cos(1.0), math.sin(1.0)), dtype=torch.complex64)
    g, gfl = run_gpu(c, 8)
    assert np.max(np.abs(R.wrap(g - 1.0))) < 1e-4


# ----------------------------------------------------------- stack / determinism / API
def test_stack_determinism_and_shard_invariance():
    w = synth.workload("C3", H=96, W=80)
    stack = synth.make_stack(w, frames=range(6)).to(DEV)
    a, fa, ra = bosrm.bos_rootmusic_demod_stack(stack, 8, ref_index=0, flags=True)
    b, fb, rb = bosrm.bos_rootmusic_demod_stack(stack, 8, ref_index=0, flags=True)
    torch.cuda.synchronize()
    assert torch.equal(a, b) and torch.equal(fa, fb)
    # frame sharding: [0:2] and [2:6] against the same reference give the same bytes
    s1, _ = bosrm.bos_rootmusic_demod(stack[0:2].contiguous(), 8, ref_phase=ra)
    s2, _ = bosrm.bos_rootmusic_demod(stack[2:6].contiguous(), 8, ref_phase=ra)
    torch.cuda.synchronize()
    assert torch.equal(torch.cat([s1, s2]), a)
    fin = torch.isfinite(a[0])
    assert torch.all(a[0][fin] == 0)
    # nonzero ref index
    c, _, rc = bosrm.bos_rootmusic_demod_stack(stack, 8, ref_index=3)
    torch.cuda.synchronize()
    assert torch.all(c[3][torch.isfinite(c[3])] == 0)


def test_host_api_matches_device_api():
    w = synth.workload("C3", H=64, W=96)
    stack = synth.make_stack(w, frames=range(7))
    dev_out, dev_fl, _ = bosrm.bos_rootmusic_demod_stack(stack.to(DEV), 8, ref_index=0, flags=True)
    h = stack.pin_memory()
    h_out, h_fl = bosrm.bos_rootmusic_demod_stack_host(h, 8, ref_index=0, h_flags=True, chunk_frames=2)
    torch.cuda.synchronize()
    assert torch.equal(h_out, dev_out.cpu()) and torch.equal(h_fl, dev_fl.cpu())
    # pageable host memory works too
    h_out2, _ = bosrm.bos_rootmusic_demod_stack_host(stack.clone(), 8, ref_index=0, chunk_frames=3)
    torch.cuda.synchronize()
    assert torch.equal(h_out2, dev_out.cpu())


@pytest.mark.parametrize("T", [1, 2])
def test_host_and_device_stack_tiny(T):
    """One- and two-frame stacks: the host pipeline (the reference chunk alone, then at most one
    flow chunk) and the device stack (one-frame path / small-stack raw launch + difference)
    give the same bytes; the reference's own output is exactly 0."""
    w = synth.workload("C3", H=48, W=40)
    stack = synth.make_stack(w, frames=range(T), snr_db=10.0)
    d_out, d_fl, d_ref = bosrm.bos_rootmusic_demod_stack(stack.to(DEV), 8, ref_index=T - 1, flags=True)
    h_out, h_fl = bosrm.bos_rootmusic_demod_stack_host(stack.pin_memory(), 8, ref_index=T - 1, h_flags=True,
                                                      chunk_frames=1)
    torch.cuda.synchronize()
    assert torch.equal(h_out, d_out.cpu()) and torch.equal(h_fl, d_fl.cpu())
    r = d_out[T - 1]
    assert torch.all(r[torch.isfinite(r)] == 0)


@pytest.mark.parametrize("ref_index,chunk,M", [(3, 4, 8), (9, 5, 8), (6, 3, 15), (0, 16, 5)])
def test_host_api_ramped_chunks(ref_index, chunk, M):
    """The host pipeline's chunk schedule (the reference frame alone first; the other frames in
    chunks ramping 1, 2, 4, … up to chunk_frames and halving over the tail, never across the
    reference) gives the device stack's outputs and flags bit for bit, for any ref_index."""
    w = synth.workload("C3", H=64, W=96)
    stack = synth.make_stack(w, frames=range(10), snr_db=5.0)
    dev_out, dev_fl, dev_ref = bosrm.bos_rootmusic_demod_stack(stack.to(DEV), M, ref_index=ref_index, flags=True)
    h_out, h_fl = bosrm.bos_rootmusic_demod_stack_host(stack.pin_memory(), M, ref_index=ref_index, h_flags=True,
                                                      chunk_frames=chunk)
    torch.cuda.synchronize()
    assert torch.equal(torch.nan_to_num(h_out, 9.0), torch.nan_to_num(dev_out.cpu(), 9.0))
    assert torch.equal(h_fl, dev_fl.cpu())


def test_error_codes_on_device():
    f = torch.zeros(1, 32, 32, dtype=torch.complex64, device=DEV)
    out = torch.empty(1, 32, 32, dtype=torch.float32, device=DEV)
    L = bosrm.lib()
    s = torch.cuda.current_stream().cuda_stream
    assert L.bos_rootmusic_demod(f.data_ptr(), 1, 32, 32, 8, 2, None, out.data_ptr(), None, s) == \
        bosrm.BOS_ERR_UNSUPPORTED
    hostbuf = torch.zeros(1, 32, 32, dtype=torch.float32)
    assert L.bos_rootmusic_demod(f.data_ptr(), 1, 32, 32, 8, 3, None, hostbuf.data_ptr(), None, s) == \
        bosrm.BOS_ERR_INVALID_ARG
    assert L.bos_rootmusic_demod(f.data_ptr(), 1, 32, 32, 8, 3, None, f.data_ptr(), None, s) == \
        bosrm.BOS_ERR_INVALID_ARG
    assert L.bos_rootmusic_demod(f.data_ptr(), 1, 40, 40, 33, 3, None, out.data_ptr(), None, s) == \
        bosrm.BOS_ERR_UNSUPPORTED
    with pytest.raises(bosrm.BosError):
        bosrm.bos_rootmusic_demod(f, 2)


def test_iteration_counts_variant_matches():
    w = synth.workload("C3", H=64, W=64)
    f = synth.make_stack(w, frames=[4]).to(DEV)
    a, _ = bosrm.bos_rootmusic_demod(f, 8)
    c = bosrm.bos_rootmusic_iteration_counts(f, 8)
    torch.cuda.synchronize()
    assert c["pixels"] == 64 * 64
    assert torch.equal(a, c["out"])
    assert 1 <= c["power_its"] / c["pixels"] <= 64
    assert 1 <= c["aberth_y"] / c["pixels"] <= 40


# ------------------------------------------------------------------- C3 at full size
def test_c3_full_size_sampled_parity():
    """1024²×100 diffusion stack, the bench configuration (one stack call, M=8); sampled
    pixels of frames {1, 50, 99} against the oracle on the same bytes."""
    w = synth.workload("C3")
    stack = synth.make_stack(w, device=DEV)
    out, fl, ref = bosrm.bos_rootmusic_demod_stack(stack, 8, ref_index=0, flags=True)
    torch.cuda.synchronize()
    rng = np.random.default_rng(11)
    pix = (rng.integers(0, w.H, 4096), rng.integers(0, w.W, 4096))
    frames = [0, 1, 50, 99]
    host = stack[frames].cpu().numpy()
    o, ofl = R.demod_stack(host, 8, ref_index=0, pixels=pix, frame_indices=[1, 2, 3])
    g = out[[1, 50, 99]].cpu().numpy()
    for j in range(3):
        assert_parity(g[j][pix], o[j], ofl[j], f"C3 frame {frames[j + 1]}")


@pytest.mark.parametrize("M", [4, 5, 8, 11, 16, 17, 24, 32])
@pytest.mark.parametrize("snr", [None, 40.0, 25.0])
def test_high_snr_and_noise_free_parity(M, snr):
    """Near-double roots on the unit circle (noise-free / high SNR) on a 64×72 crop-sized
    frame of the C1 phantom: the regime where the signal root pair merges."""
    w = synth.workload("C1", H=64, W=72)
    f = synth.make_frame(w, 0, snr_db=snr)
    g, _ = run_gpu(f, M)
    o, ofl = R.demod_frame(f.numpy(), M)
    s = assert_parity(g, o, ofl, f"high-SNR M={M} snr={snr}")
    assert s["flagged_frac"] <= 0.02, s


@pytest.mark.parametrize("M", [5, 8, 11, 17, 24])
def test_low_snr_excluded_pixels_valid(M):
    """−5 dB frame (below the paper's 0–20 dB sweep): the oracle flags AMBIGUOUS and
    SMALL_GAP pixels; parity on the rest, and [R15] validity of the GPU output on every
    excluded pixel (Eq.(15) at its own ω; one of the candidates where AMBIGUOUS)."""
    f = synth.make_frame(synth.workload("C3", H=48, W=64, seed=3), 4, snr_db=-5.0)
    g, gfl, wx, wy = run_gpu_ex(f, M)
    o, ofl = R.demod_frame(f.numpy(), M)
    s = assert_parity(g, o, ofl, f"-5dB M={M}", gpu_flags=gfl)
    assert s["excluded"] > 0, s         # the check below must have something to check
    st = assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"-5dB M={M}")
    assert st["eq15"] > 0, st


@pytest.mark.parametrize("M", [5, 8, 11, 16, 24, 32])
def test_exact_two_tone_tie_frame(M):
    """Every interior window is an exact two-frequency tie (tests/test_oracle_ambiguous.py:
    column vector e^{jw0 y}·(real) ⇒ conjugate-symmetric roots about w0): P:L208's "closest
    root" is not unique wherever the closest root is one of the conjugate pairs.  (The
    polynomial in w = z·e^{-j w0} has real coefficients, so a root may also sit on the real
    axis, angle w0 or w0+π, and be unique: at M = 5 that happens on 4 of the 13 interior rows,
    where the column's 2cos(δ(py+o)) profile changes sign inside the window.)  The oracle
    flags AMBIGUOUS; the GPU must flag it too and return one of the valid answers ([R15]);
    the rows with a unique closest root are ordinary parity pixels."""
    w0, delta = 0.5, 0.6 if M < 11 else 0.45
    H, W = M + 12, 70
    y, x = np.mgrid[0:H, 0:W]
    fr = np.exp(1j * 0.3 * x) * (np.exp(1j * (w0 + delta) * y) + np.exp(1j * (w0 - delta) * y))
    f = torch.from_numpy(fr.astype(np.complex64))
    g, gfl, wx, wy = run_gpu_ex(f, M)
    o, ofl = R.demod_frame(f.numpy(), M)
    interior = (ofl & R.FLAG_BORDER) == 0
    amb = interior & ((ofl & R.FLAG_AMBIGUOUS) != 0)
    assert amb.sum() >= 0.6 * interior.sum()
    assert np.mean((gfl[amb] & bosrm.FLAG_AMBIGUOUS) != 0) >= 0.99
    # the tie frame is flagged by construction: no interior-fraction bound, parity elsewhere
    assert_parity(g, o, ofl, f"tie M={M}", max_interior_excluded_frac=1.0)
    st = assert_excluded_valid(f.numpy(), M, g, wx, wy, ofl, f"tie M={M}")
    assert st["ambiguous"] >= int(amb.sum())


@pytest.mark.parametrize("M", [17, 20, 21, 25])
def test_wide_kernel_nonfinite_does_not_leak_along_the_segment(M):
    """A NaN sample poisons only the windows that contain it: the sliding R_y update of the
    warp-per-pixel kernel rebuilds R after a non-finite window."""
    H, W = M + 8, 70
    f = synth.make_frame(synth.workload("C3", H=H, W=W, seed=5), 4, snr_db=15.0).clone()
    f[H // 2, 10] = complex(float("nan"), 0.0)
    g, gfl = run_gpu(f, M)
    o, ofl = R.demod_frame(f.numpy(), M)
    bad = (ofl & R.FLAG_NONFINITE) != 0
    assert np.all(np.isnan(g[bad])) and np.all(gfl[bad] & bosrm.FLAG_NONFINITE)
    assert_parity(g, o, ofl, f"wide NaN M={M}")


def test_64bit_offsets_stack_beyond_2p32_pixels():
    """n_frames·H·W > 2^32 (C5-scale offsets on one GPU): 1025 frames of 2048² (4.3e9 px,
    32 GiB of input).  The last frames' sampled pixels match the oracle."""
    free, _ = torch.cuda.mem_get_info()
    T, H, W = 1025, 2048, 2048
    need = T * H * W * (8 + 4) + (4 << 30)
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB free")
    w = synth.workload("C4")
    frames = torch.empty(T, H, W, dtype=torch.complex64, device=DEV)
    ref_frame = synth.make_frame(w, 0, device=DEV)
    frames[:] = ref_frame                      # every frame = the reference ...
    frames[T - 1] = synth.make_frame(w, 3, device=DEV)   # ... except the last one
    out, _, ref = bosrm.bos_rootmusic_demod_stack(frames, 8, ref_index=0)
    torch.cuda.synchronize()
    rng = np.random.default_rng(64)
    pix = (rng.integers(0, H, 2048), rng.integers(0, W, 2048))
    host = torch.stack([frames[0], frames[T - 1]]).cpu().numpy()
    o, ofl = R.demod_stack(host, 8, ref_index=0, pixels=pix, frame_indices=[1])
    g = out[T - 1].cpu().numpy()[pix]
    assert_parity(g, o[0], ofl[0], "frame 1024 of 1025 (offset > 2^32)")
    mid = out[T // 2].cpu().numpy()
    assert np.all(mid[np.isfinite(mid)] == 0.0)
    del frames, out
    torch.cuda.empty_cache()


def test_c5_full_stack_on_one_gpu():
    """BASELINE config 5 at full size on ONE GPU (what 1 of the 1/2/4/8 shards would hold at
    N = 1): 2048² × 2000 frames of the C5 generator (8.4e9 pixels, 62.5 GiB in, 31 GiB out), one
    stack call at M = 8; sampled pixels of frames {1, 1000, 1999} against the oracle."""
    free, _ = torch.cuda.mem_get_info()
    w = synth.workload("C5")
    T, H, W = w.T, w.H, w.W
    need = T * H * W * (8 + 4) + (4 << 30)
    if free < need:
        pytest.skip(f"needs {need / 2**30:.0f} GiB free")
    frames = torch.empty(T, H, W, dtype=torch.complex64, device=DEV)
    for t in range(T):
        frames[t] = synth.make_frame(w, t, device=DEV)
    out, _, ref = bosrm.bos_rootmusic_demod_stack(frames, 8, ref_index=0)
    torch.cuda.synchronize()
    rng = np.random.default_rng(55)
    pix = (rng.integers(0, H, 4096), rng.integers(0, W, 4096))
    picks = [1, 1000, T - 1]
    host = frames[[0] + picks].cpu().numpy()
    o, ofl = R.demod_stack(host, 8, ref_index=0, pixels=pix, frame_indices=[1, 2, 3])
    for j, t in enumerate(picks):
        assert_parity(out[t].cpu().numpy()[pix], o[j], ofl[j], f"C5 frame {t} of {T}")
    del frames, out
    torch.cuda.empty_cache()


@pytest.mark.parametrize("M", [12, 15, 17, 20, 21, 24, 25, 32])
def test_c4_large_windows_sampled_parity(M):
    """C4 frames (2048², diffusion flow, 10 dB) at every kernel regime: registers (12, 15),
    R_y in shared memory (17, 20), warp kernel (21, 24, 25, 32): 2048 random pixels of frame 7,
    plus the near-tie pixel (2, 255) where the runner-up root must be refined (M = 32)."""
    w = synth.workload("C4")
    frames = synth.make_stack(w, frames=[0, 7], device=DEV)
    raw, _ = bosrm.bos_rootmusic_demod(frames, M)
    torch.cuda.synchronize()
    rng = np.random.default_rng(M)
    py = np.concatenate([[2], rng.integers(0, w.H, 2047)])
    px = np.concatenate([[255], rng.integers(0, w.W, 2047)])
    host = frames.cpu().numpy()
    o, ofl = R.demod_frame(host[1], M, pixels=(py, px))
    assert_parity(raw[1].cpu().numpy()[py, px], o, ofl, f"C4 M={M}")


@pytest.mark.parametrize("M", [8, 11, 20])
def test_omega_maps_match_oracle(M):
    """Row f3: the Eq.(15) local frequencies ω_x = −arg z_x, ω_y = arg z_y (rad/pixel)."""
    w = synth.workload("C2")
    f = synth.make_frame(w, 1, snr_db=10.0)
    out, fl, wx, wy = bosrm.bos_rootmusic_demod_ex(f.to(DEV), M, flags=True)
    base, _ = bosrm.bos_rootmusic_demod(f.to(DEV), M)
    torch.cuda.synchronize()
    assert torch.equal(out, base)                      # the extra outputs do not change the phase
    rng = np.random.default_rng(M)
    pix = (rng.integers(0, w.H, 4096), rng.integers(0, w.W, 4096))
    win, _ = R.extract_windows(f.numpy(), pix[0], pix[1], M)
    res = R.estimate_windows(win)
    assert_parity(wx[0].cpu().numpy()[pix], res["omega_x"], res["flags"], f"omega_x M={M}")
    assert_parity(wy[0].cpu().numpy()[pix], res["omega_y"], res["flags"], f"omega_y M={M}")


def test_index_gradient_kernel():
    """Eq.(17) kernel vs the oracle formula, aligned and unaligned lengths, in place."""
    for n in (1, 7, 4096, 1000003):
        ph = torch.randn(n + 1, dtype=torch.float32, device=DEV)
        for view in (ph[:n], ph[1:]):
            v = view.contiguous() if view.storage_offset() == 0 else view
            out = bosrm.bos_index_gradient(v, 1.333, 1.0, 1e4, 0.01)
            torch.cuda.synchronize()
            expect = R.index_gradient(v.cpu().numpy(), 1.333, 1.0, 1e4, 0.01)
            assert np.allclose(out.cpu().numpy(), expect, rtol=1e-6, atol=0)
    x = torch.randn(1000, dtype=torch.float32, device=DEV)
    ref = x.clone()
    bosrm.bos_index_gradient(x, 1.333, 1.0, 1e4, 0.01, out=x)   # in place
    torch.cuda.synchronize()
    assert np.allclose(x.cpu().numpy(), R.index_gradient(ref.cpu().numpy(), 1.333, 1.0, 1e4, 0.01), rtol=1e-6)


def test_vertical_profile_kernel():
    """Row f3 profile: GPU vs the oracle's FP64 column mean on a demodulated C3 stack with NaN
    pixels and one all-NaN row; ragged widths (not multiples of 32)."""
    w = synth.workload("C3", H=96, W=77)
    st = synth.make_stack(w, frames=range(4)).to(DEV)
    ph, _, _ = bosrm.bos_rootmusic_demod_stack(st, 8, ref_index=0)
    ph[1, 10, 3] = float("nan")
    ph[2, 20, :] = float("inf")
    prof = bosrm.bos_vertical_profile(ph)
    torch.cuda.synchronize()
    expect = R.vertical_profile(ph.cpu().numpy())
    got = prof.cpu().numpy()
    assert got.shape == (4, 96)
    assert np.isnan(got[2, 20]) and np.isnan(expect[2, 20])
    fin = np.isfinite(expect)
    assert np.all(np.isfinite(got[fin]))
    assert np.max(np.abs(got[fin] - expect[fin])) <= 1e-6 * max(1.0, np.max(np.abs(expect[fin])))
    for W in (1, 31, 33, 1000):
        x = torch.randn(3, 5, W, dtype=torch.float32, device=DEV)
        g = bosrm.bos_vertical_profile(x)
        torch.cuda.synchronize()
        assert np.allclose(g.cpu().numpy(), R.vertical_profile(x.cpu().numpy()), rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("M", [5, 8, 17, 24])
def test_outputs_do_not_write_outside_their_buffers(M):
    """Canary guard bands around out / flags / ω buffers (compute-sanitizer is not available on
    this pool): every kernel writes exactly its [T,H,W] slice."""
    T, H, W = 2, M + 5, 45
    st = synth.make_stack(synth.workload("C3", H=H, W=W), frames=[0, 4], device=DEV)
    n = T * H * W
    pad = 4096
    big = torch.full((n + 2 * pad,), 12345.0, dtype=torch.float32, device=DEV)
    fbig = torch.full((n + 2 * pad,), 77, dtype=torch.uint8, device=DEV)
    wx = torch.full((n + 2 * pad,), -7.0, dtype=torch.float32, device=DEV)
    wy = torch.full((n + 2 * pad,), -8.0, dtype=torch.float32, device=DEV)
    L = bosrm.lib()
    s = torch.cuda.current_stream().cuda_stream
    rc = L.bos_rootmusic_demod_ex(st.data_ptr(), T, H, W, M, 3, None, big[pad:].data_ptr(), fbig[pad:].data_ptr(),
                                  wx[pad:].data_ptr(), wy[pad:].data_ptr(), s)
    assert rc == 0
    torch.cuda.synchronize()
    for buf, val in ((big, 12345.0), (wx, -7.0), (wy, -8.0)):
        assert torch.all(buf[:pad] == val) and torch.all(buf[pad + n:] == val)
        assert torch.all(torch.isfinite(buf[pad:pad + n]))
    assert torch.all(fbig[:pad] == 77) and torch.all(fbig[pad + n:] == 77)
