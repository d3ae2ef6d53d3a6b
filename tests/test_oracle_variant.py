"""Pins of the oracle's row-f4 variant (forward–backward averaged covariances, NOT in the
paper; DESIGN.md [R13]).  CPU only.

What pins it to something other than itself:
* the textbook definition of FB averaging as the covariance of forward + backward snapshots
  (the backward snapshot of x is J·conj(x)) — computed here by an SVD of the augmented data
  matrix [Γ_w, J·conj(Γ_w)], a different route from fb_subspaces' eigh of ½(R + J R* J);
* the Eq.(3) plane-wave model is still recovered exactly (odd and even M);
* the backward window J·conj(Γ_w)·J has the same FB covariances, hence the same ω and the
  conjugate phase;
* the metamorphic invariants of the paper variant (transpose, global phase) still hold.
"""

import math

import numpy as np
import pytest

from oracle import rootmusic as R


def noisy_windows(M, n, seed, sigma=0.7):
    rng = np.random.default_rng(seed)
    o = R.window_offsets(M)
    wx = rng.uniform(-2, 2, n)
    wy = rng.uniform(-2, 2, n)
    a = rng.uniform(-math.pi, math.pi, n)
    win = np.exp(1j * (wx[:, None, None] * o[None, None, :] + wy[:, None, None] * o[None, :, None]
                       + a[:, None, None]))
    return win + sigma * (rng.standard_normal(win.shape) + 1j * rng.standard_normal(win.shape))


def test_exchange_matrix():
    J = R.exchange(4)
    assert np.array_equal(J @ np.arange(4), np.arange(4)[::-1])


@pytest.mark.parametrize("M", [3, 6, 8, 11, 19, 32])
def test_fb_equals_augmented_snapshot_svd(M):
    """Dominant eigenvectors of the FB averages = dominant left singular vectors of the
    augmented snapshot matrices [Γ, J Γ*] (y axis: columns are snapshots) and [Γ^T, J Γ^H]
    conjugated (x axis: the rows of Γ read as snapshots of e^{-jω_x k} after conjugation,
    v_1 ∝ Γ^H u_1 convention)."""
    win = noisy_windows(M, 16, 300 + M)
    J = R.exchange(M)
    U, S, Vh, Sx = R.fb_subspaces(win)
    for t in range(win.shape[0]):
        G = win[t]
        aug_y = np.concatenate([G, J @ np.conj(G)], axis=1)
        uy = np.linalg.svd(aug_y)[0][:, 0]
        # R_x = Γ^H Γ: its snapshots are the conjugated rows, conj(Γ)^T columns
        Gx = np.conj(G).T
        aug_x = np.concatenate([Gx, J @ np.conj(Gx)], axis=1)
        ux = np.linalg.svd(aug_x)[0][:, 0]
        v1 = np.conj(Vh[t, 0, :])          # first column of V
        assert abs(abs(np.vdot(uy, U[t, :, 0])) - 1) < 1e-9
        assert abs(abs(np.vdot(ux, v1)) - 1) < 1e-9
        # eigenvalues: λ(R_fb) = σ²(aug)/2
        s_aug = np.linalg.svd(aug_y, compute_uv=False)
        assert np.allclose(S[t] ** 2, s_aug ** 2 / 2, rtol=1e-9, atol=1e-9 * s_aug[0] ** 2)
        s_augx = np.linalg.svd(aug_x, compute_uv=False)
        assert np.allclose(Sx[t] ** 2, s_augx ** 2 / 2, rtol=1e-9, atol=1e-9 * s_augx[0] ** 2)


def test_fb_average_is_centro_hermitian():
    win = noisy_windows(7, 8, 5)
    Rf = R.fb_average(win @ np.conj(np.swapaxes(win, 1, 2)))
    J = R.exchange(7)
    assert np.allclose(Rf, np.conj(np.swapaxes(Rf, 1, 2)), atol=1e-12)
    assert np.allclose(Rf, J @ np.conj(Rf) @ J, atol=1e-12)


@pytest.mark.parametrize("M", [3, 4, 5, 8, 11, 16, 17, 24, 32])
def test_fb_plane_wave_exact(M):
    rng = np.random.default_rng(400 + M)
    n = 24
    wx = rng.uniform(-2.5, 2.5, n)
    wy = rng.uniform(-2.5, 2.5, n)
    a = rng.uniform(-math.pi, math.pi, n)
    o = R.window_offsets(M)
    win = np.exp(1j * (wx[:, None, None] * o[None, None, :] + wy[:, None, None] * o[None, :, None]
                       + a[:, None, None]))
    r = R.estimate_windows(win, "fb")
    assert np.max(np.abs(r["omega_x"] - wx)) < 1e-6
    assert np.max(np.abs(r["omega_y"] - wy)) < 1e-6
    tol = 1e-9 if M % 2 else 1e-6
    assert np.max(np.abs(R.wrap(r["alpha"] - a))) < tol
    assert not np.any(r["flags"] & R.PARITY_EXCLUDE_MASK)


@pytest.mark.parametrize("M", [5, 8, 11])
def test_fb_backward_window_symmetry(M):
    """Γ' = J Γ* J has the same FB covariances ⇒ identical ω; α' = −α − (ω_x + ω_y)·δ with
    δ = 0 (odd M, centred window) or 1 (even M: o_{M−1−i} = 1 − o_i, [R2])."""
    win = noisy_windows(M, 64, 500 + M)
    J = R.exchange(M)
    back = J @ np.conj(win) @ J
    f0, f1 = R.estimate_windows(win, "fb"), R.estimate_windows(back, "fb")
    ok = ((f0["flags"] | f1["flags"]) & R.PARITY_EXCLUDE_MASK) == 0
    assert ok.mean() > 0.8
    delta = 0.0 if M % 2 else 1.0
    assert np.max(np.abs(R.wrap(f1["omega_x"] - f0["omega_x"]))[ok]) < 1e-9
    assert np.max(np.abs(R.wrap(f1["omega_y"] - f0["omega_y"]))[ok]) < 1e-9
    pred = -f0["alpha"] - delta * (f0["omega_x"] + f0["omega_y"])
    assert np.max(np.abs(R.wrap(f1["alpha"] - pred))[ok]) < 1e-9
    # (root-MUSIC itself has this symmetry — the polynomial of J·conj(u) equals that of u —
    # so the paper variant passes it too; for FB it pins the J·R*·J term: an FB average that
    # drops the conjugate or one J breaks the equality of the two FB covariances)


@pytest.mark.parametrize("M", [3, 8])
def test_fb_metamorphic(M):
    win = noisy_windows(M, 64, 600 + M)
    base = R.estimate_windows(win, "fb")
    ok = (base["flags"] & R.PARITY_EXCLUDE_MASK) == 0
    tr = R.estimate_windows(np.swapaxes(win, 1, 2).copy(), "fb")
    assert np.max(np.abs(R.wrap(tr["alpha"] - base["alpha"]))[ok]) < 1e-9
    assert np.max(np.abs(R.wrap(tr["omega_x"] - base["omega_y"]))[ok]) < 1e-9
    sh = R.estimate_windows(2.5 * np.exp(0.77j) * win, "fb")
    assert np.max(np.abs(R.wrap(sh["alpha"] - base["alpha"] - 0.77))[ok]) < 1e-9


def test_fb_differs_from_paper_on_noise_but_agrees_statistically():
    """Both variants estimate the same plane: on 10 dB-like windows the two phase maps agree
    to well within the noise (not bit-identical: different subspace estimates)."""
    win = noisy_windows(11, 256, 700, sigma=0.2)
    a = R.estimate_windows(win, "paper")
    b = R.estimate_windows(win, "fb")
    d = np.abs(R.wrap(a["alpha"] - b["alpha"]))
    assert d.max() > 1e-8
    assert np.median(d) < 0.02


def test_fb_small_gap_uses_both_axes():
    """[R13]: a window whose columns are clamped copies (frame border) has a well-separated
    R_y but a near-degenerate FB R_x; SMALL_GAP must fire on the x axis alone."""
    rng = np.random.default_rng(3)
    M = 32
    o = R.window_offsets(M)
    win = np.exp(1j * (0.4 * o[None, :] + 0.7 * o[:, None]))
    win = win + 0.05 * (rng.standard_normal(win.shape) + 1j * rng.standard_normal(win.shape))
    win[:, M // 2:] = win[:, M // 2 - 1:M // 2]        # clamp at x = W−1 (M = 32 border pixel)
    U, S, Vh, Sx = R.fb_subspaces(win[None])
    gy, gx = (S[0, 0] / S[0, 1]) ** 2, (Sx[0, 0] / Sx[0, 1]) ** 2
    assert gy > R.GAMMA_MIN > gx
    assert R.estimate_windows(win[None], "fb")["flags"][0] & R.FLAG_SMALL_GAP
    assert not R.estimate_windows(win[None], "paper")["flags"][0] & R.FLAG_SMALL_GAP


def test_unknown_variant_rejected():
    with pytest.raises(ValueError):
        R.estimate_windows(noisy_windows(3, 1, 0), "spatial")


def test_demod_frame_variant_threading():
    rng = np.random.default_rng(9)
    f = (rng.standard_normal((20, 21)) + 1j * rng.standard_normal((20, 21))).astype(np.complex64)
    a1, f1 = R.demod_frame(f, 5, variant="fb", threads=1)
    a2, f2 = R.demod_frame(f, 5, variant="fb", threads=4)
    assert np.array_equal(a1, a2) and np.array_equal(f1, f2)


# --------------------------------------------------------------------------------------
# Spatial smoothing (subarray_len m < M), row f4 [R14]
# --------------------------------------------------------------------------------------
def test_ss_full_order_is_the_plain_covariance():
    """m = M: one subarray, the snapshots are the columns / conjugated rows → Γ_wΓ_w^H and
    Γ_w^HΓ_w exactly, whose top eigenvectors are the SVD's u_1, v_1."""
    win = noisy_windows(7, 8, 21)
    Ry, Rx = R.ss_covariances(win, 7)
    Wh = np.conj(np.swapaxes(win, 1, 2))
    assert np.allclose(Ry, win @ Wh, atol=1e-12) and np.allclose(Rx, Wh @ win, atol=1e-12)
    U, S, Vh, Sx = R.eig_subspaces(Ry, Rx)
    U2, S2, Vh2 = R.svd_subspaces(win)
    assert np.allclose(np.abs(np.einsum("ni,ni->n", np.conj(U[:, :, 0]), U2[:, :, 0])), 1.0, atol=1e-9)
    assert np.allclose(np.abs(np.einsum("ni,ni->n", Vh[:, 0, :], np.conj(Vh2[:, 0, :]))), 1.0, atol=1e-9)
    assert np.allclose(S, S2, rtol=1e-9) and np.allclose(Sx, S2, rtol=1e-9)


@pytest.mark.parametrize("M,m", [(8, 6), (11, 7), (16, 5)])
def test_ss_decorrelates_coherent_waves(M, m):
    """The textbook property of spatial smoothing (Shan, Wax & Kailath 1985): two coherent
    tones along y (identical in every column) give a rank-1 R_y, but a rank-2 smoothed R_y
    whose signal subspace contains both length-m steering vectors."""
    o = R.window_offsets(M)
    w1, w2 = 0.7, -0.4
    col = np.exp(1j * w1 * o) + 0.8 * np.exp(1j * (w2 * o + 0.3))
    win = np.repeat(col[:, None], M, axis=1)[None]
    lam_full = np.linalg.eigvalsh(win[0] @ np.conj(win[0]).T)[::-1]
    assert lam_full[1] < 1e-9 * lam_full[0]
    Ry, _ = R.ss_covariances(win, m)
    lam, U = np.linalg.eigh(Ry[0])
    lam, U = lam[::-1], U[:, ::-1]
    assert lam[1] > 1e-3 * lam[0] and lam[2] < 1e-9 * lam[0]
    Un = U[:, 2:]
    for w in (w1, w2):
        a = np.exp(1j * w * np.arange(m))
        assert np.linalg.norm(np.conj(Un).T @ a) < 1e-6 * np.linalg.norm(a)


@pytest.mark.parametrize("M,m", [(5, 3), (8, 3), (8, 5), (12, 8), (17, 9), (32, 16)])
def test_ss_plane_wave_exact(M, m):
    rng = np.random.default_rng(10 * M + m)
    n = 16
    wx = rng.uniform(-2.5, 2.5, n)
    wy = rng.uniform(-2.5, 2.5, n)
    a = rng.uniform(-math.pi, math.pi, n)
    o = R.window_offsets(M)
    win = np.exp(1j * (wx[:, None, None] * o[None, None, :] + wy[:, None, None] * o[None, :, None]
                       + a[:, None, None]))
    for variant in ("paper", "fb"):
        r = R.estimate_windows(win, variant, subarray_len=m)
        assert np.max(np.abs(r["omega_x"] - wx)) < 1e-6
        assert np.max(np.abs(r["omega_y"] - wy)) < 1e-6
        tol = 1e-9 if M % 2 else 1e-6
        assert np.max(np.abs(R.wrap(r["alpha"] - a))) < tol
        assert not np.any(r["flags"] & R.PARITY_EXCLUDE_MASK)


def test_ss_m3_noise_free_roots_closed_form():
    """m = 3 on a noise-free plane wave: the quartic's roots are the M = 3 template's
    {e^{jω} (double), −(2 ∓ √3)e^{jω}} (pinned in test_oracle_pins for Eq.(12) at M = 3)."""
    M, w = 9, 0.6
    o = R.window_offsets(M)
    win = np.exp(1j * (0.2 * o[None, :] + w * o[:, None]))[None]
    Ry, Rx = R.ss_covariances(win, 3)
    U, S, Vh, Sx = R.eig_subspaces(Ry, Rx)
    Cy, _ = R.noise_projectors(U, Vh)
    roots, _ = R.companion_roots(R.music_polynomial(Cy))
    expect = np.array([np.exp(1j * w), np.exp(1j * w), -(2 - math.sqrt(3)) * np.exp(1j * w),
                       -(2 + math.sqrt(3)) * np.exp(1j * w)])
    got = np.sort_complex(roots[0])
    for e in expect:
        assert np.min(np.abs(got - e)) < 1e-6


@pytest.mark.parametrize("M,m", [(8, 5), (11, 3)])
def test_ss_metamorphic(M, m):
    win = noisy_windows(M, 64, 800 + M)
    base = R.estimate_windows(win, "paper", subarray_len=m)
    ok = (base["flags"] & R.PARITY_EXCLUDE_MASK) == 0
    assert ok.mean() > 0.8
    tr = R.estimate_windows(np.swapaxes(win, 1, 2).copy(), "paper", subarray_len=m)
    assert np.max(np.abs(R.wrap(tr["alpha"] - base["alpha"]))[ok]) < 1e-9
    assert np.max(np.abs(R.wrap(tr["omega_x"] - base["omega_y"]))[ok]) < 1e-9
    cj = R.estimate_windows(np.conj(win), "paper", subarray_len=m)
    assert np.max(np.abs(R.wrap(cj["alpha"] + base["alpha"]))[ok]) < 1e-9
    sh = R.estimate_windows(2.5 * np.exp(0.77j) * win, "paper", subarray_len=m)
    assert np.max(np.abs(R.wrap(sh["alpha"] - base["alpha"] - 0.77))[ok]) < 1e-9


def test_ss_rejects_bad_order():
    with pytest.raises(ValueError):
        R.ss_covariances(noisy_windows(5, 1, 0), 6)
