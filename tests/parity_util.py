"""Shared parity assertions: CUDA path vs FP64 oracle (BASELINE north_star tolerance)."""

import math

import numpy as np

from oracle import rootmusic as R

RMS_TOL = 1e-3   # rad, RMS of wrapped error over oracle-unflagged pixels (north_star)
MAX_TOL = 1e-2   # rad, max |wrapped error| over the same pixels


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
    out = dict(n=int(valid.sum()), excluded=int((~valid).sum()), rms=rms, max=mx, gpu_nan=n_nan,
               flagged_frac=float((~valid).mean()))
    if gpu_flags is not None:      # report the GPU-only-flagged fraction too
        gf = np.asarray(gpu_flags).ravel()
        out["gpu_only_flagged_frac"] = float((((gf & R.PARITY_EXCLUDE_MASK) != 0) & valid).mean())
    return out


def assert_parity(gpu, ref, ref_flags, what="", rms_tol=RMS_TOL, max_tol=MAX_TOL, max_excluded_frac=0.05,
                  gpu_flags=None):
    s = parity_stats(gpu, ref, ref_flags, gpu_flags)
    msg = f"{what}: {s}"
    assert s["gpu_nan"] == 0, msg
    assert s["rms"] <= rms_tol, msg
    assert s["max"] <= max_tol, msg
    assert s["flagged_frac"] <= max_excluded_frac, msg
    return s
