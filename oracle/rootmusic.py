"""Plain FP64 CPU oracle: windowed root-MUSIC phase estimation, step by step as in the paper.

TEST INFRASTRUCTURE, NOT PRODUCT CODE (see ``oracle/__init__.py``).  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs may call it.

Paper: Ramaiah, Ajithaprasad, Rajshekhar, Ambrosini, "Fast and robust method for flow
analysis using GPU assisted DOE based background oriented schlieren", arxiv 1910.11872.
Citations ``P:L<n>`` are line numbers of ``PAPER.md`` (the LaTeX source); equation numbers
follow the paper.  Readings of silent/ambiguous passages are listed in ``DESIGN.md`` §3 and
tagged here as ``[R<n>]``.

The oracle follows Algorithm 1 literally, for every pixel independently:

  line 3  Γ_w ← (M×M) window around (px,py)                   extract_windows   Eq.(2)
  line 4  U, S, V^H ← SVD of Γ_w                                svd_subspaces
  line 5-6 U_n = [u_2..u_M], V_n = [v_2..v_M]                   noise_projectors  Eqs.(11),(14)
  line 7-8 y_poly, x_poly = u_1^H(z) U_n U_n^H u_1(z), ...       music_polynomial  Eqs.(12),(13)
          roots ← eigenvalues of the companion matrix            companion_roots
  line 9-10 root inside and closest to the unit circle          select_root
  line 11 φ(px,py) ← Eq.(15)                                    estimate_windows  Eq.(15)

plus the time-lapse reference difference wrap(φ_t − φ_ref) (BASELINE north_star, [R7]).
Variant "fb" (NOT in the paper, [R13]): line 4 uses the eigenvectors of the
forward–backward averaged covariances instead of the SVD (fb_subspaces); everything else is
unchanged.  ``subarray_len`` m < M (row f4, [R14]): line 4 uses the eigenvectors of the
spatially smoothed covariances of order m (ss_covariances, degree-(2m−2) polynomials).
Library primitives used as single steps: ``numpy.linalg.svd`` (LAPACK zgesdd) for the SVD
and ``numpy.linalg.eigvals`` (LAPACK zgeev: balancing + Hessenberg + shifted QR) for the
companion-matrix eigenvalues.  No blocking, fusion or reordering beyond the paper's steps.
Arithmetic is complex128 throughout; inputs (complex64 frames) are promoted exactly.

Pins (tests/test_oracle_*.py): plane-wave exactness (Eq.(3) model), Eq.(8) eigenvalue,
Eq.(9) orthogonality, brute-force polar-grid root search, quadratic-phase closed form,
metamorphic symmetries (transpose, conjugation, global phase, real scale), and the
SPEC selection examples.  The exact Table 1 values are parity-unpinned (phantom unknown).
"""

from __future__ import annotations

import math
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# ----------------------------------------------------------------------------------------
# Per-pixel status bits (DESIGN.md §3 [R8]; the paper never discusses failures).
# ----------------------------------------------------------------------------------------
FLAG_NONCONVERGED = 1 << 0   # no root inside the tolerance band / LAPACK failure / degree drop
FLAG_AMBIGUOUS = 1 << 1      # two distinct-frequency root pairs equally close to the circle
FLAG_SMALL_GAP = 1 << 2      # σ1²/σ2² < GAMMA_MIN: signal subspace not separated
FLAG_LOW_AMPLITUDE = 1 << 3  # |Σ Γ_w e^{-j(...)}| < LOW_AMP · M · ‖Γ_w‖_F: α ill-defined
FLAG_NONFINITE = 1 << 4      # window contains NaN/Inf: output NaN
FLAG_BORDER = 1 << 5         # informational: window was clamped at the frame edge
PARITY_EXCLUDE_MASK = 0x1F   # bits 0-4 exclude a pixel from GPU parity

TAU_CIRCLE = 1e-6    # unit-circle tolerance band |z| < 1 + τ   [R6]
TAU_SEL = 1e-3       # ambiguity margin in |ln|z||            [R8]
TAU_OMEGA = 1e-2     # two roots are "distinct" if their args differ by more than this
GAMMA_MIN = 1.3      # SMALL_GAP threshold on σ1²/σ2²         [R8]
LOW_AMP = 1e-4       # LOW_AMPLITUDE threshold                 [R8]


def window_offsets(M: int) -> np.ndarray:
    """Local coordinates o_i of window row/column i, target pixel at 0.

    Eq.(2): a (2L+1)×(2L+1) window, M = 2L+1, so o = -L..L.
    Even M is not in the paper [R2]: o = -⌊(M-1)/2⌋ .. ⌊M/2⌋ (e.g. M=8 → -3..4).
    """
    if M < 2:
        raise ValueError("window_len must be >= 2")
    return np.arange(M, dtype=np.int64) - (M - 1) // 2


def wrap(d):
    """Wrap radians into (-π, π]:  wrap(d) = d - 2π·ceil((d - π) / 2π)."""
    d = np.asarray(d, dtype=np.float64)
    return d - 2.0 * np.pi * np.ceil((d - np.pi) / (2.0 * np.pi))


def extract_windows(frame: np.ndarray, py: np.ndarray, px: np.ndarray, M: int):
    """Algorithm 1 line 3 / Eq.(2): Γ_w[i][k] = Γ[clamp(py+o_i)][clamp(px+o_k)].

    Rows of Γ_w follow y, columns follow x [R4]; out-of-frame samples replicate the
    nearest edge sample [R1] (the paper computes every pixel, but states no
    border rule).  Returns (windows [N,M,M] complex128, border_mask [N] bool).
    """
    H, W = frame.shape
    o = window_offsets(M)
    yy = py[:, None] + o[None, :]
    xx = px[:, None] + o[None, :]
    border = (yy.min(axis=1) < 0) | (yy.max(axis=1) > H - 1) | \
             (xx.min(axis=1) < 0) | (xx.max(axis=1) > W - 1)
    yy = np.clip(yy, 0, H - 1)
    xx = np.clip(xx, 0, W - 1)
    win = frame[yy[:, :, None], xx[:, None, :]].astype(np.complex128)
    return win, border


def svd_subspaces(win: np.ndarray):
    """Algorithm 1 line 4: U, S, V^H ← SVD of Γ_w ("singular value
    decomposition approach").  Columns of U are eigenvectors of Γ_wΓ_w^H = R_y (Eq.(4)),
    columns of V eigenvectors of Γ_w^HΓ_w = R_x; S descending.  Full U, V even when Γ_w
    is rank deficient (noise-free rank-1 windows)."""
    U, S, Vh = np.linalg.svd(win, full_matrices=True)
    return U, S, Vh


def exchange(M: int) -> np.ndarray:
    """J, the M×M exchange (anti-identity) matrix: (J x)_i = x_{M-1-i}."""
    return np.eye(M)[::-1]


def fb_average(R: np.ndarray) -> np.ndarray:
    """Forward–backward average ½(R + J R* J) of covariances [N,M,M] (variant f4, NOT in the
    paper): the covariance of the forward snapshots together with the backward snapshots
    J·conj(x) (Pillai & Kwon 1989; standard in root-MUSIC/ESPRIT)."""
    J = exchange(R.shape[-1])
    return 0.5 * (R + J @ np.conj(R) @ J)


def fb_subspaces(win: np.ndarray):
    """Variant f4 replacement of Algorithm 1 line 4 (NOT in the paper): eigenvectors of the
    forward–backward averaged R_y = Γ_wΓ_w^H and R_x = Γ_w^HΓ_w (Eq.(4) and its x-axis
    counterpart), eigenvalues descending (numpy.linalg.eigh, LAPACK
    zheevd, as a single step).  Returned like svd_subspaces, (U, S, V^H) with S = √λ(R_y,fb),
    plus S_x = √λ(R_x,fb): unlike the SVD, the two axes have different spectra."""
    Wh = np.conj(np.swapaxes(win, 1, 2))
    Ry = fb_average(win @ Wh)
    Rx = fb_average(Wh @ win)
    ly, U = np.linalg.eigh(Ry)
    lx, V = np.linalg.eigh(Rx)
    U = U[:, :, ::-1]
    V = V[:, :, ::-1]
    S = np.sqrt(np.maximum(ly[:, ::-1], 0.0))
    Sx = np.sqrt(np.maximum(lx[:, ::-1], 0.0))
    return U, S, np.conj(np.swapaxes(V, 1, 2)), Sx


def ss_covariances(win: np.ndarray, m: int):
    """Spatially smoothed (reduced-order) covariances of order m ≤ M (variant f4, NOT in the
    paper; Shan, Wax & Kailath 1985): the snapshots of R_y are all length-m segments of the
    columns of Γ_w, x_{s,k} = Γ_w[s:s+m, k]; those of R_x are the conjugated length-m segments
    of the rows, y_{s,i} = conj(Γ_w[i, s:s+m]) (so that m = M gives Γ_wΓ_w^H and Γ_w^HΓ_w):
        R_y = Σ_{s=0}^{M−m} Σ_k x_{s,k} x_{s,k}^H,   R_x = Σ_{s=0}^{M−m} Σ_i y_{s,i} y_{s,i}^H."""
    N, M, _ = win.shape
    if not 2 <= m <= M:
        raise ValueError("subarray length must be in [2, M]")
    Ry = np.zeros((N, m, m), dtype=np.complex128)
    Rx = np.zeros((N, m, m), dtype=np.complex128)
    for s in range(M - m + 1):
        X = win[:, s:s + m, :]                                  # columns = snapshots
        Y = np.swapaxes(np.conj(win[:, :, s:s + m]), 1, 2)      # [N, m, M]: columns = conj rows
        Ry += X @ np.conj(np.swapaxes(X, 1, 2))
        Rx += Y @ np.conj(np.swapaxes(Y, 1, 2))
    return Ry, Rx


def eig_subspaces(Ry: np.ndarray, Rx: np.ndarray, fb: bool = False):
    """Eigenvectors (descending) of the two axes' covariances, optionally FB-averaged; returned
    like fb_subspaces: (U, S, V^H, S_x) with S = √λ(R_y), S_x = √λ(R_x)."""
    if fb:
        Ry, Rx = fb_average(Ry), fb_average(Rx)
    ly, U = np.linalg.eigh(Ry)
    lx, V = np.linalg.eigh(Rx)
    U, V = U[:, :, ::-1], V[:, :, ::-1]
    S = np.sqrt(np.maximum(ly[:, ::-1], 0.0))
    Sx = np.sqrt(np.maximum(lx[:, ::-1], 0.0))
    return U, S, np.conj(np.swapaxes(V, 1, 2)), Sx


VARIANTS = ("paper", "fb")


def noise_projectors(U: np.ndarray, Vh: np.ndarray):
    """Algorithm 1 lines 5-6, Eqs.(11),(14):
    U_n = [u_2 … u_M], V_n = [v_2 … v_M] (signal subspace dimension 1, Eqs.(7)-(10), [R3]);
    returns C_y = U_n U_n^H and C_x = V_n V_n^H (the matrices inside Eqs.(12),(13))."""
    Un = U[:, :, 1:]
    V = np.conj(np.swapaxes(Vh, 1, 2))
    Vn = V[:, :, 1:]
    Cy = Un @ np.conj(np.swapaxes(Un, 1, 2))
    Cx = Vn @ np.conj(np.swapaxes(Vn, 1, 2))
    return Cy, Cx


def music_polynomial(C: np.ndarray) -> np.ndarray:
    """Eqs.(12),(13), Algorithm 1 lines 7-8.

    f(z) = u_1^H(z) C u_1(z) with u_1(z) = [1, z, …, z^{M-1}]^T and u_1^H(z) read as
    [1, z^{-1}, …, z^{-(M-1)}] off the unit circle (standard root-MUSIC, [R3c]):
        f(z) = Σ_{i,k} C[i][k] z^{k-i} = Σ_d s_d z^d,   s_d = Σ_i C[i][i+d].
    Multiplying by z^{M-1} gives a polynomial of degree 2M-2 ([R3b]: the paper's
    "(2M-1) possible roots", counts coefficients).
    Returns coefficients a[:, n], n = 0..2M-2 (ascending powers), a_n = s_{n-M+1}.
    """
    N, M, _ = C.shape
    a = np.empty((N, 2 * M - 1), dtype=np.complex128)
    for n in range(2 * M - 1):
        a[:, n] = np.trace(C, offset=n - (M - 1), axis1=1, axis2=2)
    return a


def _roots_one(a: np.ndarray) -> np.ndarray:
    """Single polynomial with possibly vanishing leading coefficients: trim, then the
    companion-matrix eigenvalues (degree drops mean roots at infinity, returned as inf)."""
    n = a.shape[0] - 1
    nz = np.nonzero(a)[0]
    out = np.full(n, np.inf + 0j, dtype=np.complex128)
    if nz.size == 0:
        return out
    top = nz[-1]
    if top == 0:
        return out
    comp = np.zeros((top, top), dtype=np.complex128)
    comp[1:, :-1] = np.eye(top - 1)
    comp[:, -1] = -a[:top] / a[top]
    out[:top] = np.linalg.eigvals(comp)
    return out


def companion_roots(a: np.ndarray):
    """roots as eigenvalues of the companion matrix (Chapra & Canale).

    For p(z) = Σ_n a_n z^n of degree n, the monic companion matrix has ones on the
    subdiagonal and last column -a_{0..n-1}/a_n; its characteristic polynomial is
    p(z)/a_n.  Eigenvalues by LAPACK zgeev (balancing + Hessenberg + shifted QR).
    Returns (roots [N, n], degenerate [N] bool: leading coefficient vanished)."""
    N, n1 = a.shape
    n = n1 - 1
    lead = a[:, -1]
    degenerate = lead == 0
    roots = np.empty((N, n), dtype=np.complex128)
    ok = ~degenerate
    if ok.any():
        comp = np.zeros((int(ok.sum()), n, n), dtype=np.complex128)
        comp[:, 1:, :-1] = np.eye(n - 1)
        comp[:, :, -1] = -a[ok, :-1] / lead[ok, None]
        roots[ok] = np.linalg.eigvals(comp)
    for idx in np.nonzero(degenerate)[0]:
        roots[idx] = _roots_one(a[idx])
    return roots, degenerate


def select_root(roots: np.ndarray, tau: float = TAU_CIRCLE):
    """P:L208 / Algorithm 1 lines 9-10: "the one which is closest to the unit circle with
    magnitude less than 1".  Noise-free double roots sit on the circle, so the strict
    inequality is relaxed to |z| < 1 + τ [R6]; among the candidates the largest |z| is
    the closest to the circle from inside.  Ties: smallest arg in (-π, π], then input
    order.  Returns (z [N], index [N], found [N] bool)."""
    N, n = roots.shape
    mag = np.abs(roots)
    cand = np.isfinite(mag) & (mag < 1.0 + tau)
    key_mag = np.where(cand, -mag, np.inf)
    key_arg = np.where(cand, np.angle(roots), np.inf)
    key_idx = np.broadcast_to(np.arange(n), (N, n))
    order = np.lexsort((key_idx, key_arg, key_mag), axis=-1)
    idx = order[:, 0]
    found = cand[np.arange(N), idx]
    z = roots[np.arange(N), idx]
    z = np.where(found, z, np.nan + 0j)
    return z, idx, found


def selection_margin(roots: np.ndarray, z_sel: np.ndarray) -> np.ndarray:
    """[R8] margin between the selected pair and the best root pair of a *different*
    frequency: d = |ln|z||, margin = min_{|wrap(arg z - arg z_sel)| > τ_ω} d - d(z_sel).
    Members of one (z, 1/z̄) pair share arg (P:L208 selects within a pair; ω is unique),
    so only distinct-frequency pairs make the selection ambiguous."""
    with np.errstate(divide="ignore", invalid="ignore"):
        d = np.abs(np.log(np.abs(roots)))
        d_sel = np.abs(np.log(np.abs(z_sel)))
        dang = np.abs(wrap(np.angle(roots) - np.angle(z_sel)[:, None]))
        other = np.where((dang > TAU_OMEGA) & np.isfinite(d), d, np.inf)
        return other.min(axis=1) - d_sel


def estimate_windows(win: np.ndarray, variant: str = "paper", subarray_len: int | None = None):
    """Algorithm 1 lines 4-11 on a batch of windows [N,M,M] (complex128, finite).
    Row f4 (not in the paper): variant "fb" replaces line 4 by fb_subspaces; subarray_len
    m < M replaces it by the eigenvectors of the spatially smoothed covariances of order m
    (ss_covariances; polynomials of degree 2m−2; FB-averaged too for "fb").  Eq.(15) always
    uses the whole M×M window.

    Returns dict: alpha (Eq.(15) phase), omega_x, omega_y, flags (bits 0-3), plus the
    intermediate z_y, z_x, S, margins for tests."""
    N, M, _ = win.shape
    if variant not in VARIANTS:
        raise ValueError(f"unknown variant {variant!r}")
    if subarray_len is not None and subarray_len != M:
        U, S, Vh, Sx = eig_subspaces(*ss_covariances(win, int(subarray_len)), fb=variant == "fb")
    elif variant == "paper":
        U, S, Vh = svd_subspaces(win)
        Sx = S                       # one spectrum: σ of Γ_w serves both axes
    else:
        U, S, Vh, Sx = fb_subspaces(win)
    Cy, Cx = noise_projectors(U, Vh)
    ay = music_polynomial(Cy)
    ax = music_polynomial(Cx)
    ry, degy = companion_roots(ay)
    rx, degx = companion_roots(ax)
    zy, _, fy = select_root(ry)
    zx, _, fx = select_root(rx)

    # Eq.(15): ω_y = arg z_y, ω_x = -arg z_x (z_x = e^{-jω_x})
    omega_y = np.angle(zy)
    omega_x = -np.angle(zx)
    alpha, c = eq15_phase(win, omega_x, omega_y)

    flags = np.zeros(N, dtype=np.uint8)
    flags |= np.where(~(fy & fx) | degy | degx, FLAG_NONCONVERGED, 0).astype(np.uint8)
    marg = np.minimum(selection_margin(ry, zy), selection_margin(rx, zx))
    flags |= np.where(marg < TAU_SEL, FLAG_AMBIGUOUS, 0).astype(np.uint8)
    with np.errstate(divide="ignore", invalid="ignore"):
        # [R8]/[R13]: the smaller eigenvalue ratio of the two axes' covariances
        gap = np.minimum(np.where(S[:, 1] > 0, (S[:, 0] / S[:, 1]) ** 2, np.inf),
                         np.where(Sx[:, 1] > 0, (Sx[:, 0] / Sx[:, 1]) ** 2, np.inf))
    flags |= np.where(gap < GAMMA_MIN, FLAG_SMALL_GAP, 0).astype(np.uint8)
    fro = np.sqrt(np.sum(np.abs(win) ** 2, axis=(1, 2)))
    low = (fro == 0) | (np.abs(c) * M * M < LOW_AMP * M * fro)
    flags |= np.where(low, FLAG_LOW_AMPLITUDE, 0).astype(np.uint8)
    return dict(alpha=alpha, omega_x=omega_x, omega_y=omega_y, flags=flags,
                z_y=zy, z_x=zx, S=S, margin=marg, c=c, roots_y=ry, roots_x=rx)


def eq15_phase(win: np.ndarray, omega_x, omega_y):
    """Eq.(15), Algorithm 1 line 11: α = ∠ mean(Γ_w e^{-j(ω_x x + ω_y y)}) with
    the window's local coordinates (target pixel at the origin, [R5]).  The mean of the
    demodulated window is the least-squares complex amplitude of the Eq.(3) model for the
    given (ω_x, ω_y).  Returns (α [N], c [N] complex)."""
    N, M, _ = win.shape
    omega_x = np.broadcast_to(np.asarray(omega_x, dtype=np.float64), (N,))
    omega_y = np.broadcast_to(np.asarray(omega_y, dtype=np.float64), (N,))
    o = window_offsets(M).astype(np.float64)
    phase = omega_x[:, None, None] * o[None, None, :] + omega_y[:, None, None] * o[None, :, None]
    c = np.mean(win * np.exp(-1j * phase), axis=(1, 2))
    return np.angle(c), c


# [R15] Where several outputs are correct (P:L208 leaves the choice between two distinct root
# pairs equally close to the unit circle open), the valid outputs are the candidates below.
TAU_CAND = 2.0 * TAU_SEL   # candidate band in |ln|z|| above the closest root (2 × the AMBIGUOUS margin)


def root_candidates(roots: np.ndarray, band: float = TAU_CAND):
    """[R15] For one polynomial's roots [n]: the distinct frequencies among the roots whose
    distance |ln|z|| to the unit circle is within ``band`` of the closest root (P:L208's
    candidates when the rule is ambiguous).  Roots whose args differ by ≤ τ_ω are one
    frequency (the members of a (z, 1/z̄) pair share arg); each frequency is represented by
    its closest root.  Returns a list of complex roots, closest first."""
    r = np.asarray(roots)
    with np.errstate(divide="ignore", invalid="ignore"):
        d = np.abs(np.log(np.abs(r)))
    ok = np.isfinite(d)
    if not ok.any():
        return []
    order = np.argsort(np.where(ok, d, np.inf), kind="stable")
    dmin = d[order[0]]
    out = []
    for i in order:
        if not ok[i] or d[i] > dmin + band:
            break
        if all(abs(float(wrap(np.angle(r[i]) - np.angle(q)))) > TAU_OMEGA for q in out):
            out.append(r[i])
    return out


def candidate_estimates(frame: np.ndarray, py, px, M: int, band: float = TAU_CAND, variant: str = "paper",
                        subarray_len: int | None = None):
    """[R15] The set of valid (ω_x, ω_y, α) at each pixel: every combination of the y- and
    x-axis root candidates (root_candidates) with α from Eq.(15) at that (ω_x, ω_y).  For an
    unambiguous pixel the set has one member, Algorithm 1's output.  Returns a list (one entry
    per pixel) of arrays [k, 3]."""
    py = np.asarray(py, dtype=np.int64).ravel()
    px = np.asarray(px, dtype=np.int64).ravel()
    win, _ = extract_windows(np.asarray(frame), py, px, M)
    res = estimate_windows(win, variant, subarray_len)
    out = []
    for p in range(py.size):
        cy = root_candidates(res["roots_y"][p], band)
        cx = root_candidates(res["roots_x"][p], band)
        rows = []
        for zy in cy:
            for zx in cx:
                wy, wx = float(np.angle(zy)), float(-np.angle(zx))
                a, _ = eq15_phase(win[p:p + 1], wx, wy)
                rows.append((wx, wy, float(a[0])))
        out.append(np.array(rows, dtype=np.float64).reshape(-1, 3))
    return out


def eq15_at(frame: np.ndarray, py, px, M: int, omega_x, omega_y):
    """Eq.(15) at given frequencies for the windows of pixels (py, px) (clamped as in
    extract_windows): returns (α [N], |c| [N], ‖Γ_w‖_F [N])."""
    py = np.asarray(py, dtype=np.int64).ravel()
    px = np.asarray(px, dtype=np.int64).ravel()
    win, _ = extract_windows(np.asarray(frame), py, px, M)
    a, c = eq15_phase(win, np.asarray(omega_x, np.float64).ravel(), np.asarray(omega_y, np.float64).ravel())
    fro = np.sqrt(np.sum(np.abs(win) ** 2, axis=(1, 2)))
    return a, np.abs(c), fro


def default_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return max(1, os.cpu_count() or 1)


def _estimate_pixels(frame, py, px, M, variant="paper", subarray_len=None):
    win, border = extract_windows(frame, py, px, M)
    finite = np.isfinite(win.real).all(axis=(1, 2)) & np.isfinite(win.imag).all(axis=(1, 2))
    safe = np.where(finite[:, None, None], win, 0.0)
    res = estimate_windows(safe, variant, subarray_len)
    alpha = np.where(finite, res["alpha"], np.nan)
    flags = res["flags"].copy()
    flags[~finite] = FLAG_NONFINITE
    flags |= np.where(border, FLAG_BORDER, 0).astype(np.uint8)
    return alpha, flags


def demod_frame(frame: np.ndarray, window_len: int, model_order: int = 3, ref_phase=None,
                pixels=None, threads: int | None = None, chunk: int | None = None, variant: str = "paper",
                subarray_len: int | None = None):
    """Phase map of one frame: Algorithm 1 at every pixel (or at ``pixels=(py, px)``).

    ref_phase: None → raw α (wrapped); else out = wrap(α - ref_phase) [R7], where
    ref_phase has the frame's shape [H,W] (or is already sampled to ``pixels``).
    Returns (phase float64, flags uint8) shaped [H,W] (or [N] for ``pixels``).
    Multi-threaded over static pixel chunks; each pixel is computed independently, so the
    result does not depend on ``threads`` or ``chunk``.
    """
    if model_order != 3:
        raise NotImplementedError("model_order must be 3: Eq.(3) plane model [R3]")
    frame = np.asarray(frame)
    H, W = frame.shape
    M = int(window_len)
    if M < 2 or H < M or W < M:
        raise ValueError("frame smaller than the window")
    if pixels is None:
        yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        py, px = yy.ravel(), xx.ravel()
    else:
        py, px = (np.asarray(p, dtype=np.int64).ravel() for p in pixels)
    n = py.size
    nthreads = threads or default_threads()
    if chunk is None:   # static partition depending on n only (not on the thread count)
        chunk = int(min(2048, max(128, -(-n // 32))))
    alpha = np.empty(n, dtype=np.float64)
    flags = np.empty(n, dtype=np.uint8)
    bounds = list(range(0, n, chunk)) + [n]

    def work(j):
        s, e = bounds[j], bounds[j + 1]
        alpha[s:e], flags[s:e] = _estimate_pixels(frame, py[s:e], px[s:e], M, variant, subarray_len)

    if nthreads == 1 or len(bounds) <= 2:
        for j in range(len(bounds) - 1):
            work(j)
    else:
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(work, range(len(bounds) - 1)))

    if ref_phase is not None:
        ref = np.asarray(ref_phase, dtype=np.float64)
        ref = ref.ravel() if pixels is None else (ref[py, px] if ref.shape == (H, W) else ref.ravel())
        alpha = wrap(alpha - ref)
    if pixels is None:
        return alpha.reshape(H, W), flags.reshape(H, W)
    return alpha, flags


def demod_stack(frames: np.ndarray, window_len: int, model_order: int = 3, ref_index: int = 0,
                pixels=None, frame_indices=None, threads: int | None = None, variant: str = "paper",
                subarray_len: int | None = None):
    """Time-lapse stack [T,H,W]: φ_ref = α(frames[ref_index]); out[t] = wrap(α_t - φ_ref).

    ``frame_indices`` restricts the output to those frames (sampled parity on big stacks);
    the reference flags are OR-ed into every output frame's flags (a bad reference pixel
    makes every difference at that pixel ill-conditioned)."""
    frames = np.asarray(frames)
    T = frames.shape[0]
    ts = range(T) if frame_indices is None else frame_indices
    ref, ref_flags = demod_frame(frames[ref_index], window_len, model_order, None, pixels, threads,
                                 variant=variant, subarray_len=subarray_len)
    outs, fls = [], []
    for t in ts:
        a, f = demod_frame(frames[t], window_len, model_order, None, pixels, threads, variant=variant,
                           subarray_len=subarray_len)
        outs.append(wrap(a - ref))
        fls.append(f | ref_flags)
    return np.stack(outs), np.stack(fls)


def rms_max_wrapped(a, b, valid=None):
    """Parity statistic: e = wrap(a - b) over valid entries → (rms, max, count)."""
    e = wrap(np.asarray(a, np.float64) - np.asarray(b, np.float64))
    if valid is not None:
        e = e[valid]
    e = e[np.isfinite(e)]
    if e.size == 0:
        return 0.0, 0.0, 0
    return float(math.sqrt(np.mean(e * e))), float(np.max(np.abs(e))), int(e.size)


def index_gradient(phase, n0: float, mu: float, f_x: float, cell_len: float):
    """Eq.(17): ∂n/∂x = (1/(2 μ f_x)) · (n0 / L²) · φ, pointwise (FP64)."""
    return (1.0 / (2.0 * mu * f_x)) * (n0 / (cell_len * cell_len)) * np.asarray(phase, dtype=np.float64)


def vertical_profile(phase):
    """Row f3, SPEC ``stack_series``: per-frame vertical profile, the
    column-averaged phase as a function of the row y (the paper's time-evolution comparison,
    Figs. 6-8).  phase [..., H, W] → [..., H] (FP64); non-finite pixels are
    skipped, a row without finite pixels gives NaN."""
    p = np.asarray(phase, dtype=np.float64)
    fin = np.isfinite(p)
    n = fin.sum(axis=-1)
    s = np.where(fin, p, 0.0).sum(axis=-1)
    with np.errstate(invalid="ignore", divide="ignore"):
        return np.where(n > 0, s / np.maximum(n, 1), np.nan)

