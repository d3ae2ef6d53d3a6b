"""Pins of the FP64 oracle to things other than itself (paper closed forms, brute force,
invariants).  CPU only.  Citations: P:L<n> = PAPER.md line; [Rn] = DESIGN.md §3 readings."""

import math
import os

import numpy as np
import pytest

from oracle import rootmusic as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def plane_frame(H, W, wx, wy, a, amp=1.0):
    y, x = np.mgrid[0:H, 0:W]
    return amp * np.exp(1j * (wx * x + wy * y + a))


def steering(M, w):
    return np.exp(1j * w * np.arange(M))


# --------------------------------------------------------------------------------------
# Eq.(3) model exactness: a noise-free plane wave is recovered exactly (Eq.(15))
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 15, 16, 17, 24, 32, 33])
def test_plane_wave_exact(M):
    rng = np.random.default_rng(100 + M)
    n = 24
    wx = rng.uniform(-2.5, 2.5, n)
    wy = rng.uniform(-2.5, 2.5, n)
    a = rng.uniform(-math.pi, math.pi, n)
    o = R.window_offsets(M)
    # Window of the plane wave e^{j(wx x + wy y + a)} around the origin (rows <-> y, [R4]).
    win = np.exp(1j * (wx[:, None, None] * o[None, None, :] + wy[:, None, None] * o[None, :, None]
                       + a[:, None, None]))
    r = R.estimate_windows(win)
    assert np.max(np.abs(r["omega_x"] - wx)) < 1e-6
    assert np.max(np.abs(r["omega_y"] - wy)) < 1e-6
    # alpha = phase at the target pixel [R5]; even M is first-order sensitive to the
    # (√ε-limited) double-root ω error, odd M is not (centred window).
    tol = 1e-9 if M % 2 else 1e-6
    assert np.max(np.abs(R.wrap(r["alpha"] - a))) < tol
    assert not np.any(r["flags"] & R.PARITY_EXCLUDE_MASK)


def test_plane_wave_field_demod():
    """Whole-frame demod of a plane wave reproduces wrap(0.3x + 0.5y + 0.2) (SPEC S:L255 idea)."""
    H = W = 48
    f = plane_frame(H, W, 0.3, 0.5, 0.2).astype(np.complex64)
    ph, fl = R.demod_frame(f, 7)
    y, x = np.mgrid[0:H, 0:W]
    truth = 0.3 * x + 0.5 * y + 0.2
    interior = (fl & R.FLAG_BORDER) == 0
    # complex64 input quantisation (~6e-8) is the only error source
    assert np.max(np.abs(R.wrap(ph - truth))[interior]) < 1e-5


# --------------------------------------------------------------------------------------
# Eq.(8): noise-free window → dominant eigenvalue of R = Γ_wΓ_w^H is M²A² (M·A² per
# snapshot × M snapshots), all others 0; Eq.(9): u_1 ⟂ U_n.
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [3, 5, 8, 11, 17])
def test_eq8_eigenvalue_and_eq9_orthogonality(M):
    rng = np.random.default_rng(M)
    for _ in range(10):
        wx, wy, a = rng.uniform(-3, 3), rng.uniform(-3, 3), rng.uniform(-3, 3)
        A = rng.uniform(0.2, 3.0)
        o = R.window_offsets(M)
        win = A * np.exp(1j * (wx * o[None, :] + wy * o[:, None] + a))[None]
        U, S, Vh = R.svd_subspaces(win)
        assert abs(S[0, 0] ** 2 - M * M * A * A) <= 1e-10 * M * M * A * A
        assert np.all(S[0, 1:] < 1e-10 * A)
        Un = U[0, :, 1:]
        Vn = np.conj(Vh[0]).T[:, 1:]
        # Eq.(9) on both axes: a_y = [e^{jω_y i}], a_x = [e^{-jω_x k}] (z_x = e^{-jω_x})
        assert np.linalg.norm(Un.conj().T @ steering(M, wy)) < 1e-8
        assert np.linalg.norm(Vn.conj().T @ steering(M, -wx)) < 1e-8


# --------------------------------------------------------------------------------------
# Eqs.(12)-(13) polynomial: closed form of the noise-free coefficients and roots.
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [3, 4, 8, 11])
def test_noise_free_polynomial_closed_form(M):
    """For u_1 = a(ω)/√M, C = I - u_1u_1^H and the diagonal sums are
    s_d = M·δ_d - (M-|d|)/M · e^{-jωd}  (coefficient of z^{d+M-1})."""
    w = 0.77
    u = steering(M, w) / math.sqrt(M)
    C = np.eye(M) - np.outer(u, u.conj())
    a = R.music_polynomial(C[None])[0]
    d = np.arange(-(M - 1), M)
    expect = M * (d == 0) - (M - np.abs(d)) / M * np.exp(-1j * w * d)
    assert np.max(np.abs(a - expect)) < 1e-13
    # conjugate-palindromic (C Hermitian)
    assert np.max(np.abs(a - np.conj(a[::-1]))) < 1e-13
    # the double root sits at z = e^{jω} on the unit circle (Eq.(12) at the true z_y)
    roots, _ = R.companion_roots(a[None])
    dist = np.sort(np.abs(roots[0] - np.exp(1j * w)))
    assert dist[0] < 1e-6 and dist[1] < 1e-6


def test_m3_template_roots():
    """M=3 closed form: P(z) ∝ (z - e^{jω})² (z + (2∓√3)e^{jω}) (derived from the s_d above:
    -2/3·e^{jω}… ; roots e^{jω} (double), -(2-√3)e^{jω}, -(2+√3)e^{jω})."""
    w = -1.3
    u = steering(3, w) / math.sqrt(3)
    C = np.eye(3) - np.outer(u, u.conj())
    roots, _ = R.companion_roots(R.music_polynomial(C[None]))
    expect = np.array([1, 1, -(2 - math.sqrt(3)), -(2 + math.sqrt(3))]) * np.exp(1j * w)
    got = roots[0]
    for e in expect:
        k = np.argmin(np.abs(got - e))
        assert abs(got[k] - e) < 1e-6
        got = np.delete(got, k)


# --------------------------------------------------------------------------------------
# Brute force: the root multiset equals the zeros of f(z) = z^{M-1} u^H(z) C u(z) evaluated
# straight from Eq.(12)'s definition (no coefficients), found on a polar grid.
# --------------------------------------------------------------------------------------
def _direct_f(C, z):
    """z^{M-1} Σ_{i,k} C[i][k] z^{k-i} and its derivative, evaluated from the matrix."""
    M = C.shape[0]
    f = np.zeros_like(z)
    df = np.zeros_like(z)
    for i in range(M):
        for k in range(M):
            p = k - i + M - 1
            f = f + C[i, k] * z ** p
            if p > 0:
                df = df + C[i, k] * p * z ** (p - 1)
    return f, df


def brute_force_roots(C, n_r=300, n_t=2048):
    M = C.shape[0]
    # Cauchy bound from the Eq.(12) diagonal sums (roots pair as z ↔ 1/z̄)
    a = np.array([np.trace(C, offset=d) for d in range(-(M - 1), M)])
    rho = 1.0 + np.max(np.abs(a[:-1] / a[-1]))
    r = np.exp(np.linspace(-math.log(rho) * 1.05, math.log(rho) * 1.05, n_r))
    t = np.linspace(-math.pi, math.pi, n_t, endpoint=False)
    z = r[:, None] * np.exp(1j * t[None, :])
    mag = np.abs(_direct_f(C, z)[0])
    loc = np.ones_like(mag, dtype=bool)
    for dr in (-1, 0, 1):
        for dt in (-1, 0, 1):
            if dr == 0 and dt == 0:
                continue
            sh = np.roll(np.roll(mag, dr, axis=0), dt, axis=1)
            if dr == 1:
                sh[0, :] = np.inf
            if dr == -1:
                sh[-1, :] = np.inf
            loc &= mag < sh
    cands = z[loc]
    found = []
    for z0 in cands:
        zz = np.clongdouble(z0)
        Cl = C.astype(np.clongdouble)
        for _ in range(60):
            f, df = _direct_f(Cl, np.array([zz]))
            step = f[0] / df[0]
            zz = zz - step
            if abs(step) < 1e-18:
                break
        zz = complex(zz)
        if all(abs(zz - q) > 1e-7 for q in found):
            found.append(zz)
    return np.array(found)


@pytest.mark.parametrize("M", [3, 4, 5])
def test_roots_match_brute_force(M):
    rng = np.random.default_rng(7 + M)
    o = R.window_offsets(M)
    for trial in range(6):
        wx, wy = rng.uniform(-2, 2, 2)
        tone = np.exp(1j * (wx * o[None, :] + wy * o[:, None]))
        noise = (rng.standard_normal((M, M)) + 1j * rng.standard_normal((M, M))) / math.sqrt(2)
        win = tone + (0.6 if trial % 2 else 2.0) * noise
        U, S, Vh = R.svd_subspaces(win[None])
        Cy, Cx = R.noise_projectors(U, Vh)
        for C in (Cy[0], Cx[0]):
            roots, _ = R.companion_roots(R.music_polynomial(C[None]))
            bf = brute_force_roots(C)
            assert len(bf) == 2 * M - 2, (len(bf), roots)
            for q in roots[0]:
                assert np.min(np.abs(bf - q)) < 1e-7 * max(1.0, abs(q))


def test_companion_roots_constructed():
    """(z - e^{j0.5})(z - 0.8e^{j0.5}) and z² - 1 (SPEC S:L174-175 examples)."""
    z1, z2 = np.exp(0.5j), 0.8 * np.exp(0.5j)
    a = np.array([[z1 * z2, -(z1 + z2), 1.0], [-1.0, 0.0, 1.0]], dtype=np.complex128)
    roots, deg = R.companion_roots(a)
    assert not deg.any()
    assert np.allclose(sorted(roots[0], key=abs), [z2, z1], atol=1e-12)
    assert np.allclose(sorted(roots[1], key=lambda q: q.real), [-1, 1], atol=1e-12)


# --------------------------------------------------------------------------------------
# Selection rule P:L208 — golden examples
# --------------------------------------------------------------------------------------
def test_select_root_golden():
    with open(os.path.join(GOLDEN, "spec_select_root_examples.txt")) as fh:
        lines = [ln for ln in fh if ln.strip() and not ln.startswith("#")]
    for ln in lines:
        lhs, rhs = ln.split("->")
        roots = []
        for item in lhs.split(";"):
            m, a = (float(v) for v in item.split(","))
            roots.append(m * np.exp(1j * a))
        em, ea = (float(v) for v in rhs.split(","))
        z, _, found = R.select_root(np.array([roots]))
        assert found[0]
        assert abs(z[0] - em * np.exp(1j * ea)) < 1e-12


def test_select_root_none_inside():
    z, _, found = R.select_root(np.array([[2.0 + 0j, 3.0j]]))
    assert not found[0] and np.isnan(z[0])


# --------------------------------------------------------------------------------------
# Eq.(15): α is the least-squares complex-amplitude phase given (ω_x, ω_y) — brute force
# over α; and brute-force frequency search on tiny windows.
# --------------------------------------------------------------------------------------
def test_alpha_is_least_squares_fit():
    rng = np.random.default_rng(3)
    M = 5
    o = R.window_offsets(M)
    win = np.exp(1j * (0.4 * o[None, :] - 0.9 * o[:, None] + 1.1))
    win = win + 0.3 * (rng.standard_normal((M, M)) + 1j * rng.standard_normal((M, M)))
    r = R.estimate_windows(win[None])
    wx, wy = r["omega_x"][0], r["omega_y"][0]
    grid = np.linspace(-math.pi, math.pi, 200001)
    basis = np.exp(1j * (wx * o[None, :] + wy * o[:, None]))
    # ‖Γ_w - A e^{jα} basis‖² minimised over α (A ≥ 0 free) ⇔ maximise Re(e^{-jα} Σ Γ conj(basis))
    s = np.sum(win * np.conj(basis))
    best = grid[np.argmax(np.real(np.exp(-1j * grid) * s))]
    assert abs(R.wrap(best - r["alpha"][0])) < 1e-4


@pytest.mark.parametrize("M", [3, 4, 5])
def test_frequency_matches_brute_force_search(M):
    """Noise-free tone: the oracle's (ω_x, ω_y) equal the argmax of a brute-force 2-D search of
    |Σ Γ_w e^{-j(ω_x x + ω_y y)}| (coarse grid + golden-section refinement)."""
    rng = np.random.default_rng(50 + M)
    o = R.window_offsets(M)
    for _ in range(5):
        wx, wy = rng.uniform(-2.8, 2.8, 2)
        win = np.exp(1j * (wx * o[None, :] + wy * o[:, None] + rng.uniform(-3, 3)))
        g = np.linspace(-math.pi, math.pi, 721)
        P = np.abs(np.einsum("ik,ai,bk->ab", win, np.exp(-1j * g[:, None] * o[None, :]),
                             np.exp(-1j * g[:, None] * o[None, :])))
        ia, ib = np.unravel_index(np.argmax(P), P.shape)
        bx, by = g[ib], g[ia]
        # refine with a local dense search
        for span in (0.02, 2e-3, 2e-4, 2e-5, 2e-6):
            gx = bx + np.linspace(-span, span, 41)
            gy = by + np.linspace(-span, span, 41)
            P = np.abs(np.einsum("ik,ai,bk->ab", win, np.exp(-1j * gy[:, None] * o[None, :]),
                                 np.exp(-1j * gx[:, None] * o[None, :])))
            ia, ib = np.unravel_index(np.argmax(P), P.shape)
            bx, by = gx[ib], gy[ia]
        r = R.estimate_windows(win[None])
        assert abs(r["omega_x"][0] - bx) < 1e-6 and abs(r["omega_y"][0] - by) < 1e-6


# --------------------------------------------------------------------------------------
# Quadratic-phase closed form (first order in curvature), pins window centring + Eq.(15):
# α - φ(0) = (a+c)(M²-1)/24 (odd M),  (a+c)(M²-4)/24 - b/4 (even M, offsets -M/2+1..M/2)
# for φ = φ0 + g·r + ½(aX² + 2bXY + cY²).
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [5, 8, 9, 11, 16, 17])
def test_quadratic_phase_bias_closed_form(M):
    o = R.window_offsets(M).astype(float)
    X, Y = o[None, :], o[:, None]
    ca, cb, cc = 2e-4, 0.7e-4, -1.1e-4
    phi0, gx, gy = 0.3, 0.45, -0.8
    phi = phi0 + gx * X + gy * Y + 0.5 * (ca * X * X + 2 * cb * X * Y + cc * Y * Y)
    r = R.estimate_windows(np.exp(1j * phi)[None])
    if M % 2:
        pred = (ca + cc) * (M * M - 1) / 24.0
    else:
        pred = (ca + cc) * (M * M - 4) / 24.0 - cb / 4.0
    got = R.wrap(r["alpha"][0] - phi0)
    assert abs(got - pred) < 0.03 * abs(pred) + 2e-7, (got, pred)


# --------------------------------------------------------------------------------------
# Metamorphic symmetries (exact for the algorithm): transpose swaps ω_x↔ω_y and keeps α;
# conjugation negates ω and α; e^{jc} shifts α by c; real scaling changes nothing.
# --------------------------------------------------------------------------------------
@pytest.mark.parametrize("M", [3, 8, 11])
def test_metamorphic_invariants(M):
    rng = np.random.default_rng(200 + M)
    o = R.window_offsets(M)
    N = 64
    wx = rng.uniform(-2, 2, N)
    wy = rng.uniform(-2, 2, N)
    win = np.exp(1j * (wx[:, None, None] * o[None, None, :] + wy[:, None, None] * o[None, :, None]))
    win = win + 0.7 * (rng.standard_normal(win.shape) + 1j * rng.standard_normal(win.shape))
    base = R.estimate_windows(win)
    ok = (base["flags"] & R.PARITY_EXCLUDE_MASK) == 0
    assert ok.mean() > 0.8

    tr = R.estimate_windows(np.swapaxes(win, 1, 2).copy())
    assert np.max(np.abs(R.wrap(tr["alpha"] - base["alpha"]))[ok]) < 1e-9
    assert np.max(np.abs(R.wrap(tr["omega_x"] - base["omega_y"]))[ok]) < 1e-9

    cj = R.estimate_windows(np.conj(win))
    assert np.max(np.abs(R.wrap(cj["alpha"] + base["alpha"]))[ok]) < 1e-9
    assert np.max(np.abs(R.wrap(cj["omega_y"] + base["omega_y"]))[ok]) < 1e-9

    sh = R.estimate_windows(2.5 * np.exp(0.77j) * win)
    assert np.max(np.abs(R.wrap(sh["alpha"] - base["alpha"] - 0.77))[ok]) < 1e-9
    assert np.max(np.abs(sh["omega_x"] - base["omega_x"])[ok]) < 1e-9


# --------------------------------------------------------------------------------------
# Flags / borders / degenerate inputs
# --------------------------------------------------------------------------------------
def test_border_clamp_window():
    """Corner pixel window replicates edge samples ([R1]; SPEC S:L221 example)."""
    f = (np.arange(36).reshape(6, 6) + 1j * np.arange(36).reshape(6, 6)[::-1]).astype(np.complex128)
    win, border = R.extract_windows(f, np.array([0]), np.array([0]), 5)
    o = R.window_offsets(5)
    yy = np.clip(o, 0, 5)
    assert border[0]
    assert np.array_equal(win[0], f[np.ix_(yy, yy)])
    win, border = R.extract_windows(f, np.array([3]), np.array([2]), 5)
    assert not border[0]


def test_constant_window_dc():
    """ω = 0 degenerate tone: α = arg of the constant."""
    win = np.full((1, 7, 7), np.exp(1.0j))
    r = R.estimate_windows(win)
    assert abs(r["omega_x"][0]) < 1e-6 and abs(r["omega_y"][0]) < 1e-6
    assert abs(r["alpha"][0] - 1.0) < 1e-9


def test_nonfinite_and_flags():
    H = W = 24
    f = plane_frame(H, W, 0.4, 0.2, 0.0).astype(np.complex64)
    f[10, 10] = np.nan
    ph, fl = R.demod_frame(f, 5)
    assert np.isnan(ph[10, 10]) and fl[10, 10] & R.FLAG_NONFINITE
    assert np.isnan(ph[8, 12]) and fl[8, 12] & R.FLAG_NONFINITE   # window covers (10,10)
    assert np.isfinite(ph[3, 3]) and fl[3, 3] == 0
    assert fl[0, 0] & R.FLAG_BORDER and fl[23, 12] & R.FLAG_BORDER
    z = np.zeros((H, W), np.complex64)
    ph, fl = R.demod_frame(z, 5)
    assert np.all(fl & R.FLAG_LOW_AMPLITUDE)


def test_reference_difference_identical_frames_zero():
    rng = np.random.default_rng(0)
    f = (plane_frame(32, 32, 0.4, 0.8, 0.0) + 0.3 * rng.standard_normal((32, 32))).astype(np.complex64)
    out, fl = R.demod_stack(np.stack([f, f]), 8)
    assert np.all(out[np.isfinite(out)] == 0.0)


def test_carrier_cancels_in_difference():
    """Carrier-only reference vs carrier + plane-wave flow: the difference is the flow
    phase exactly (a linear phase has no curvature bias)."""
    H = W = 40
    ref = plane_frame(H, W, 2 * math.pi / 16, 2 * math.pi / 8, 0.0)
    flow = plane_frame(H, W, 2 * math.pi / 16 + 0.05, 2 * math.pi / 8 - 0.1, 0.3)
    out, fl = R.demod_stack(np.stack([ref, flow]), 8)
    y, x = np.mgrid[0:H, 0:W]
    interior = (fl[1] & R.FLAG_BORDER) == 0      # clamped windows are not plane waves
    assert interior.sum() == (H - 7) * (W - 7)
    assert np.max(np.abs(R.wrap(out[1] - (0.05 * x - 0.1 * y + 0.3)))[interior]) < 1e-6


def test_threads_deterministic():
    rng = np.random.default_rng(5)
    f = (rng.standard_normal((40, 40)) + 1j * rng.standard_normal((40, 40))).astype(np.complex64)
    a1, f1 = R.demod_frame(f, 6, threads=1)
    a8, f8 = R.demod_frame(f, 6, threads=8)
    assert np.array_equal(a1, a8) and np.array_equal(f1, f8)


def test_wrap_range():
    d = np.array([-3 * math.pi, -math.pi, -1.0, 0.0, math.pi, 3 * math.pi, 7.0])
    w = R.wrap(d)
    assert np.all(w > -math.pi) and np.all(w <= math.pi)
    assert np.allclose(np.exp(1j * w), np.exp(1j * d))
    assert w[1] == math.pi and w[4] == math.pi


def test_paper_tables_golden_parse():
    t1 = np.loadtxt(os.path.join(GOLDEN, "paper_table1_rmse_vs_L.txt"))
    assert t1.shape == (8, 3) and np.all(t1[:, 1] == 2 * t1[:, 0] + 1)
    assert t1[np.argmin(t1[:, 2]), 0] == 4          # P:L323 minimum at L=4
    t2 = np.loadtxt(os.path.join(GOLDEN, "paper_table2_timing.txt"))
    assert np.allclose(t2[:, 1] / t2[:, 2], [29.5, 33.8, 35.1, 35.3], atol=0.1)


def test_eq17_index_gradient_example():
    """Eq.(17) with the SPEC example geometry: φ = 1 rad, μ = 1, f_x = 1e4 /m,
    n0 = 1.333, L = 10 mm (the cell path length) → 0.6665 /m; linear in φ and n0,
    inverse in μ and f_x, inverse-square in L."""
    assert abs(R.index_gradient(1.0, 1.333, 1.0, 1e4, 0.01) - 0.6665) < 1e-12
    base = R.index_gradient(2.0, 1.333, 1.0, 1e4, 0.01)
    assert abs(base - 2 * 0.6665) < 1e-12
    assert abs(R.index_gradient(1.0, 1.333, 2.0, 1e4, 0.01) - 0.6665 / 2) < 1e-12
    assert abs(R.index_gradient(1.0, 1.333, 1.0, 1e4, 0.02) - 0.6665 / 4) < 1e-12


def test_vertical_profile_closed_forms():
    """Row f3 / SPEC stack_series: column-averaged φ per row.  Separable map
    f(y) + g(x) with Σ_x g = 0 → exactly f; NaN pixels skipped; an all-NaN row → NaN;
    identical frames → identical profiles."""
    H, W = 17, 24
    y = np.arange(H, dtype=np.float64)
    x = np.arange(W, dtype=np.float64)
    f = np.sin(0.3 * y) + 0.01 * y * y
    g = np.cos(2 * np.pi * x / W)                       # sums to 0 over a full period
    ph = f[:, None] + g[None, :]
    assert np.allclose(R.vertical_profile(ph), f, atol=1e-12)
    ph2 = ph.copy()
    ph2[3, 5] = np.nan
    ph2[4, :] = np.inf
    prof = R.vertical_profile(ph2)
    assert abs(prof[3] - (ph[3].sum() - ph[3, 5]) / (W - 1)) < 1e-12
    assert np.isnan(prof[4])
    st = np.stack([ph, ph])
    p2 = R.vertical_profile(st)
    assert p2.shape == (2, H) and np.array_equal(p2[0], p2[1])


def test_vertical_profile_fick_phantom():
    """SPEC S:L401 [DERIVED]: profiles of the Fick phase (∝ ∂c/∂y of the erfc step solution,
    a Gaussian of variance 2Dt, Eq.(16)) at t = 120 s and 600 s: the peak falls by
    √(600/120) and the width grows by the same factor."""
    D, dy = 1.5e-9, 9.1e-6
    H, W = 2001, 8
    yy = (np.arange(H) - H // 2) * dy

    def phi(t):
        prof = np.exp(-yy * yy / (4 * D * t)) / np.sqrt(np.pi * D * t)
        return np.repeat(prof[:, None], W, axis=1)

    p1, p2 = R.vertical_profile(phi(120.0)), R.vertical_profile(phi(600.0))
    assert abs(p1.max() / p2.max() - np.sqrt(5.0)) < 1e-9

    def fwhm(p):
        above = np.nonzero(p >= p.max() / 2)[0]
        return (above[-1] - above[0]) * dy

    assert abs(fwhm(p2) / fwhm(p1) - np.sqrt(5.0)) < 0.02
