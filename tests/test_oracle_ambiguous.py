"""Pins of the oracle's AMBIGUOUS rule and of its candidate sets ([R8], [R15]) — both
directions: the flag MUST fire where two distinct-frequency root pairs are equally close to
the unit circle ("closest to the unit circle" is then not unique), and must NOT fire
once their distance gap exceeds τ_sel = 1e-3.  Ties are constructed exactly from a symmetry
of the algorithm (no oracle value is used to build an expectation); margins are checked
against roots found by brute force from the matrix definition of Eq.(12).  CPU only."""

import math

import numpy as np
import pytest

from oracle import rootmusic as R

from .test_oracle_pins import brute_force_roots


def two_tone_window(M, w0, delta, wx, eps=0.0, phase=0.0):
    """Γ_w = s t^T: every column is s = a(w0+δ) + (1+ε)e^{jφ}... (rows ↔ y, [R4]); t is an
    x-tone.  For ε = 0 and φ = 0, s_i = e^{j w0 o_i}·2cos(δ o_i): e^{-j w0 ·} times a REAL
    vector, so R_y = M s s^H is rank 1, u_1 ∝ s, and the Eq.(12) coefficients are
    e^{-j w0 d}·(real): the polynomial in w = z e^{-j w0} has real coefficients, its roots come
    in conjugate pairs (w, w̄) with equal |w| — two frequencies w0 ± θ exactly equally close
    to the circle.  ε ≠ 0 breaks the tie."""
    o = R.window_offsets(M).astype(np.float64)
    s = np.exp(1j * (w0 + delta) * o) + (1.0 + eps) * np.exp(1j * phase) * np.exp(1j * (w0 - delta) * o)
    t = np.exp(1j * wx * o)
    return np.outer(s, t)[None]


def _margin_brute_force(C):
    """Selection margin from brute-force roots (polar-grid minima of |f(z)| evaluated from the
    matrix, long-double Newton polish): distance gap between the closest root and the closest
    root of a different frequency."""
    r = brute_force_roots(C)
    d = np.abs(np.log(np.abs(r)))
    b = int(np.argmin(d))
    dang = np.abs(R.wrap(np.angle(r) - np.angle(r[b])))
    other = d[dang > R.TAU_OMEGA]
    return float(other.min() - d[b]), r


@pytest.mark.parametrize("M,w0,delta", [(5, 0.4, 0.9), (6, -1.0, 0.8), (8, 0.7, 0.6), (11, 0.2, 0.45)])
def test_exact_two_tone_tie_fires_ambiguous(M, w0, delta):
    win = two_tone_window(M, w0, delta, wx=0.3)
    r = R.estimate_windows(win)
    assert r["flags"][0] & R.FLAG_AMBIGUOUS, r["margin"]
    assert r["margin"][0] < 1e-9
    # the two tied candidates are mirror images about w0 (the symmetry that made the tie)
    cy = R.root_candidates(r["roots_y"][0])
    assert len(cy) >= 2
    a1, a2 = (float(R.wrap(np.angle(z) - w0)) for z in cy[:2])
    assert abs(a1 + a2) < 1e-6 and abs(a1) > R.TAU_OMEGA
    # the x axis is a clean tone (exact double root on the circle): one candidate, ω_x exact
    cx = R.root_candidates(r["roots_x"][0])
    assert len(cx) == 1 and abs(-np.angle(cx[0]) - 0.3) < 1e-6
    # the rank-1 window has no SMALL_GAP (σ2 = 0) and a non-vanishing amplitude
    assert not (r["flags"][0] & (R.FLAG_SMALL_GAP | R.FLAG_LOW_AMPLITUDE | R.FLAG_NONCONVERGED))


@pytest.mark.parametrize("M,w0,delta", [(5, 0.4, 0.9), (6, -1.0, 0.8)])
def test_tie_margin_matches_brute_force_roots(M, w0, delta):
    """Independent of the companion-matrix path: the brute-force root set of Eq.(12) from the
    matrix has the same tie (margin ≈ 0) and, with the tie broken, the oracle margin equals the
    brute-force margin."""
    for eps, phase in ((0.0, 0.0), (0.2, 0.0), (0.0, 0.5), (0.05, 0.3)):
        win = two_tone_window(M, w0, delta, 0.3, eps, phase)
        U, S, Vh = R.svd_subspaces(win)
        Cy, _ = R.noise_projectors(U, Vh)
        mb, _ = _margin_brute_force(Cy[0])
        r = R.estimate_windows(win)
        assert abs(r["margin"][0] - mb) < 1e-7, (eps, phase, r["margin"][0], mb)
        if eps == 0.0 and phase == 0.0:
            assert mb < 1e-9


@pytest.mark.parametrize("M,w0,delta", [(8, 0.7, 0.6), (5, 0.4, 0.9)])
def test_ambiguous_fires_iff_margin_below_tau_sel(M, w0, delta):
    """Sweep the tie-breaking amplitude ε: the flag fires exactly when the (brute-force
    checked) margin is below τ_sel = 1e-3, and the sweep crosses τ_sel (so a rule that never
    fires, or one that always fires, fails here)."""
    fired, not_fired = 0, 0
    for eps in (0.0, 1e-5, 1e-4, 3e-4, 1e-3, 3e-3, 1e-2, 3e-2, 0.1, 0.3):
        r = R.estimate_windows(two_tone_window(M, w0, delta, 0.3, eps))
        m = float(r["margin"][0])
        f = bool(r["flags"][0] & R.FLAG_AMBIGUOUS)
        assert f == (m < R.TAU_SEL), (eps, m, f)
        fired += f
        not_fired += not f
    assert fired >= 2 and not_fired >= 2


def test_selection_margin_units_constructed_roots():
    """The margin rule on hand-made root sets (units: |ln|z|| and radians):
    distinct frequencies (args 0.05 rad apart > τ_ω = 1e-2) at radii giving a gap of 2e-4 →
    margin 2e-4 (fires); the same radii with args 0.005 rad apart are one frequency → the
    margin comes from the next distinct root."""
    r_a, r_b = math.exp(-0.0100), math.exp(-0.0102)
    far = 0.5 * np.exp(2.0j)
    roots = np.array([[r_a * np.exp(0.30j), 1 / r_a * np.exp(0.30j), r_b * np.exp(0.35j), far]])
    z, _, _ = R.select_root(roots)
    m = R.selection_margin(roots, z)[0]
    assert abs(m - 2e-4) < 1e-12
    roots2 = np.array([[r_a * np.exp(0.30j), 1 / r_a * np.exp(0.30j), r_b * np.exp(0.305j), far]])
    z2, _, _ = R.select_root(roots2)
    m2 = R.selection_margin(roots2, z2)[0]
    assert abs(m2 - (math.log(2.0) - 0.0100)) < 1e-12
    # args straddling ±π are compared wrapped (a pair at ≈ ±π is one frequency)
    roots3 = np.array([[r_a * np.exp(3.139j), r_b * np.exp(-3.139j), far]])
    z3, _, _ = R.select_root(roots3)
    m3 = R.selection_margin(roots3, z3)[0]
    assert abs(m3 - (math.log(2.0) - 0.0100)) < 1e-12


def test_root_candidates_and_candidate_estimates_on_tie():
    """[R15] On an exact tie the candidate set holds both frequencies; each candidate's α is
    Eq.(15) at its (ω_x, ω_y), checked against the brute-force least-squares phase; with the
    tie broken beyond the band, one candidate remains: Algorithm 1's output."""
    M, w0, delta = 8, 0.7, 0.6
    o = R.window_offsets(M)
    H = W = 3 * M
    y, x = np.mgrid[0:H, 0:W]
    frame = np.exp(1j * 0.3 * x) * (np.exp(1j * (w0 + delta) * y) + np.exp(1j * (w0 - delta) * y))
    py, px = np.array([H // 2, H // 2 + 1]), np.array([W // 2, W // 2 - 2])
    cands = R.candidate_estimates(frame, py, px, M)
    for p, cs in enumerate(cands):
        assert cs.shape[0] == 2
        # the two frequencies are mirror images about w0 (up to the window shift's phase, the
        # same real-vector symmetry holds at every pixel)
        assert abs(R.wrap((cs[0, 1] - w0) + (cs[1, 1] - w0))) < 1e-6
        assert np.allclose(cs[:, 0], 0.3, atol=1e-6)
        win, _ = R.extract_windows(frame, py[p:p + 1], px[p:p + 1], M)
        for wx, wy, a in cs:
            # brute-force least-squares phase: maximise Re(e^{-jα} Σ Γ_w conj(basis)) over α
            basis = np.exp(1j * (wx * o[None, :] + wy * o[:, None]))
            al = np.linspace(-math.pi, math.pi, 20001)
            proj = np.real(np.exp(-1j * al) * np.sum(win[0] * np.conj(basis)))
            assert abs(R.wrap(a - al[int(np.argmax(proj))])) < 1e-3
    # tie broken well beyond the band: one candidate, equal to the estimate
    win = two_tone_window(M, w0, delta, 0.3, eps=0.3)
    r = R.estimate_windows(win)
    assert len(R.root_candidates(r["roots_y"][0])) == 1
