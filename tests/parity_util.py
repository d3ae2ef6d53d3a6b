"""Shared parity assertions: CUDA path vs FP64 oracle (BASELINE north_star tolerance).

Two checks:
* assert_parity — the north_star bar (RMS ≤ 1e-3, max ≤ 1e-2 rad of the wrapped error) over the
  pixels the oracle does not flag (bits 0-4), no GPU NaN there, and at most 5 % flagged pixels
  among the INTERIOR windows ([R15]: clamped border windows repeat edge rows/columns [R1], are
  not the Eq.(3) plane model and may be flagged at any rate; their outputs are checked by
  assert_excluded_valid instead).  NONFINITE pixels have an exact check of their own (NaN out).
* assert_excluded_valid — [R15] where several outputs are correct, or the oracle flags the
  pixel ill-conditioned, the GPU output must still be VALID: finite; α equal to Eq.(15) at the
  GPU's own (ω_x, ω_y) (FP64, from the oracle); and, for AMBIGUOUS pixels, (ω_x, ω_y, α) equal
  to one of the oracle's candidates (oracle.rootmusic.candidate_estimates); for LOW_AMPLITUDE
  pixels (α ill-defined, ω not) ω equal to the oracle's.
"""

import math

import numpy as np

from oracle import rootmusic as R

RMS_TOL = 1e-3   # rad, RMS of wrapped error over oracle-unflagged pixels (north_star)
MAX_TOL = 1e-2   # rad, max |wrapped error| over the same pixels
INTERIOR_EXCLUDED_MAX = 0.05   # [R15] flagged fraction bound over interior, finite windows


def parity_stats(gpu, ref, ref_flags, gpu_flags=None):
    gpu = np.asarray(gpu, np.float64).ravel()
    ref = np.asarray(ref, np.float64).ravel()
    rf = np.asarray(ref_flags).ravel()
    valid = (rf & R.PARITY_EXCLUDE_MASK) == 0
    e = R.wrap(gpu - ref)
    ev = e[valid]
    n_nan = int(np.sum(~np.isfinite(ev)))
    evf = ev[np.isfinite(ev)]
    rms = float(math.sqrt(np.mean(evf * evf))) if evf.size else 0.0
    mx = float(np.max(np.abs(evf))) if evf.size else 0.0
    interior = ((rf & R.FLAG_BORDER) == 0) & ((rf & R.FLAG_NONFINITE) == 0)
    n_int = int(interior.sum())
    out = dict(n=int(valid.sum()), excluded=int((~valid).sum()), rms=rms, max=mx, gpu_nan=n_nan,
               flagged_frac=float((~valid).mean()),
               interior_n=n_int,
               interior_flagged_frac=float((~valid & interior).sum() / n_int) if n_int else 0.0)
    if gpu_flags is not None:      # report the GPU-only-flagged fraction too
        gf = np.asarray(gpu_flags).ravel()
        out["gpu_only_flagged_frac"] = float((((gf & R.PARITY_EXCLUDE_MASK) != 0) & valid).mean())
    return out


def assert_parity(gpu, ref, ref_flags, what="", rms_tol=RMS_TOL, max_tol=MAX_TOL,
                  max_interior_excluded_frac=INTERIOR_EXCLUDED_MAX, gpu_flags=None):
    s = parity_stats(gpu, ref, ref_flags, gpu_flags)
    msg = f"{what}: {s}"
    assert s["gpu_nan"] == 0, msg
    assert s["rms"] <= rms_tol, msg
    assert s["max"] <= max_tol, msg
    assert s["interior_flagged_frac"] <= max_interior_excluded_frac, msg
    return s


def _eq15_tol(M, cabs, fro):
    """FP32 bound on |α_gpu − Eq.(15)(ω_gpu)| (rad): the GPU sums M² FP32 products of
    magnitude |Γ| with twiddles from powers of ẑ, |δc| ≲ 8·M·u·Σ|Γ_w| ≤ 8·M²·u·‖Γ_w‖_F
    (u = 2⁻²⁴), over |Σ| = M²|c|; plus 1e-3 for the ω rounding of the reported maps (ω is
    float32, α's sensitivity ≤ M/2·δω) and the FP64/FP32 Eq.(15) basis differences."""
    u = 2.0 ** -24
    with np.errstate(divide="ignore"):
        return 1e-3 + 8.0 * u * fro / np.maximum(cabs, 1e-300)


def excluded_validity(frame, M, alpha, omega_x, omega_y, ref_flags, pixels=None, variant="paper", subarray_len=None):
    """[R15] Validity of the GPU output (raw α, no reference difference) on the pixels the
    oracle excludes from parity.  frame [H,W]; alpha/omega_* the GPU maps [H,W] (or sampled at
    ``pixels`` = (py, px), matching ref_flags).  Returns a dict of counts and the failures."""
    frame = np.asarray(frame)
    H, W = frame.shape
    rf = np.asarray(ref_flags).ravel()
    if pixels is None:
        yy, xx = np.meshgrid(np.arange(H), np.arange(W), indexing="ij")
        py, px = yy.ravel(), xx.ravel()
    else:
        py, px = (np.asarray(p, np.int64).ravel() for p in pixels)
    a = np.asarray(alpha, np.float64).ravel()
    wx = np.asarray(omega_x, np.float64).ravel()
    wy = np.asarray(omega_y, np.float64).ravel()
    ex = ((rf & R.PARITY_EXCLUDE_MASK) != 0) & ((rf & R.FLAG_NONFINITE) == 0)
    idx = np.nonzero(ex)[0]
    fails = []
    stats = dict(checked=int(idx.size), ambiguous=0, low_amp=0, eq15=0)
    if idx.size == 0:
        return stats, fails
    fin = np.isfinite(a[idx]) & np.isfinite(wx[idx]) & np.isfinite(wy[idx])
    for k in idx[~fin]:
        fails.append(("nonfinite", int(py[k]), int(px[k]), int(rf[k])))
    idx = idx[fin]
    # Eq.(15) at the GPU's own frequencies (every excluded pixel whose α is defined)
    a15, cabs, fro = R.eq15_at(frame, py[idx], px[idx], M, wx[idx], wy[idx])
    low = (cabs * M * M < R.LOW_AMP * M * fro) | (fro == 0)
    tol = _eq15_tol(M, cabs, fro)
    err = np.abs(R.wrap(a[idx] - a15))
    for j in np.nonzero(~low & (err > tol))[0]:
        k = idx[j]
        fails.append(("eq15", int(py[k]), int(px[k]), int(rf[k]), float(err[j]), float(tol[j])))
    stats["eq15"] = int((~low).sum())
    # AMBIGUOUS (well-separated subspace): the GPU's (ω_x, ω_y, α) is one of the candidates;
    # LOW_AMPLITUDE only: ω is unique (Algorithm 1's)
    amb = idx[((rf[idx] & R.FLAG_AMBIGUOUS) != 0) & ((rf[idx] & (R.FLAG_SMALL_GAP | R.FLAG_NONCONVERGED)) == 0)]
    lowonly = idx[(rf[idx] & R.PARITY_EXCLUDE_MASK) == R.FLAG_LOW_AMPLITUDE]
    for group, name in ((amb, "ambiguous"), (lowonly, "low_amp")):
        if group.size == 0:
            continue
        cands = R.candidate_estimates(frame, py[group], px[group], M, variant=variant, subarray_len=subarray_len)
        for k, cs in zip(group, cands):
            if cs.shape[0] == 0:
                fails.append((name + ":no-candidate", int(py[k]), int(px[k]), int(rf[k])))
                continue
            dw = np.maximum(np.abs(R.wrap(cs[:, 0] - wx[k])), np.abs(R.wrap(cs[:, 1] - wy[k])))
            da = np.abs(R.wrap(cs[:, 2] - a[k]))
            ok = dw <= R.TAU_OMEGA
            if name == "ambiguous":
                ok &= da <= MAX_TOL
            if not ok.any():
                j = int(np.argmin(dw))
                fails.append((name, int(py[k]), int(px[k]), int(rf[k]), float(dw[j]), float(da[j]),
                              (float(wx[k]), float(wy[k]), float(a[k])), cs.tolist()))
        stats[name] = int(group.size)
    return stats, fails


def assert_excluded_valid(frame, M, alpha, omega_x, omega_y, ref_flags, what="", pixels=None, variant="paper",
                          subarray_len=None):
    stats, fails = excluded_validity(frame, M, alpha, omega_x, omega_y, ref_flags, pixels, variant, subarray_len)
    assert not fails, f"{what}: {stats} {len(fails)} invalid outputs, first: {fails[:5]}"
    return stats
