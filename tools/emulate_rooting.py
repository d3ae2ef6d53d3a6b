"""Development tool (not product, not oracle): numpy FP32 emulation of the CUDA kernel's
rooting stage (symmetric Gauss–Seidel Aberth from rotated templates), to iterate on
convergence rules on the CPU.  Compares α against the FP64 oracle on the same windows.

    python tools/emulate_rooting.py C1 8      # workload, window_len
"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "paper_1910_11872_b200", "csrc"))

from gen_template_roots import template  # noqa: E402

f32 = np.float32
c64 = np.complex64


def coeffs(q):
    N, M = q.shape
    c = np.zeros((N, 2 * M - 1), c64)
    c[:, M - 1] = M - np.sum(np.abs(q) ** 2, axis=1)
    r1 = None
    for d in range(1, M):
        r = np.sum(q[:, :M - d] * np.conj(q[:, d:]), axis=1).astype(c64)
        c[:, M - 1 + d] = -r
        c[:, M - 1 - d] = -np.conj(r)
        if d == 1:
            r1 = r
    rot = np.conj(r1) / np.abs(r1)
    return c, rot.astype(c64)


def newton_ratio(c, z):
    n = c.shape[1] - 1
    m2 = np.abs(z) ** 2
    out = m2 > 1
    v = np.where(out, z / m2, z).astype(c64)
    p = c[:, n].copy()
    dp = np.zeros_like(p)
    for k in range(n - 1, -1, -1):
        dp = dp * v + p
        p = p * v + c[:, k]
    q, dq, u = np.conj(p), np.conj(dp), np.conj(v)
    num = np.where(out, z * q, p)
    den = np.where(out, q * n - u * dq, dp)
    with np.errstate(all="ignore"):
        return (num / den).astype(c64)


def newton_dp(c, z):
    """P'(z)/P''(z): Newton on P' (a near-double root of P is a simple root of P')."""
    n = c.shape[1] - 1
    p = c[:, n].copy()
    dp = np.zeros_like(p)
    ddp = np.zeros_like(p)
    for k in range(n - 1, -1, -1):
        ddp = ddp * z + dp
        dp = dp * z + p
        p = p * z + c[:, k]
    with np.errstate(all="ignore"):
        return (dp / (2 * ddp)).astype(c64)


def aberth_sym(c, z, near_tol=2e-3, tol2=1e-12, maxit=40, verbose=False, dp_mode=True):
    N, K = z.shape
    z = z.copy()
    zm = (z / np.abs(z) ** 2).astype(c64)
    its = np.zeros(N, int)
    done = np.zeros(N, bool)
    prev = np.full(N, np.inf, f32)
    for it in range(maxit):
        maxw = np.zeros(N, f32)
        for r in range(K):
            zi = z[:, r]
            ratio = newton_ratio(c, zi)
            near = np.abs(1 - np.abs(zi) ** 2) < near_tol
            with np.errstate(all="ignore"):
                s = np.where(near, 0, 1 / (zi - zm[:, r]))
                for j in range(K):
                    if j != r:
                        s = s + 1 / (zi - z[:, j]) + 1 / (zi - zm[:, j])
                w = ratio / (1 - ratio * s)
                if dp_mode:
                    w = np.where(near, newton_dp(c, zi), w)
            w2 = np.abs(w) ** 2
            bad = ~(w2 < 1e30)
            w = np.where(bad, 0, w)
            w2 = np.where(bad, 0, w2)
            w = np.where(done, 0, w)
            zn = (zi - w).astype(c64)
            z[:, r] = zn
            zm[:, r] = zn / np.abs(zn) ** 2
            maxw = np.maximum(maxw, np.where(done, 0, w2))
        active = ~done
        its[active] += 1
        conv = (maxw < tol2) | ((it >= 4) & (maxw < 1e-6) & (maxw > 0.9 * prev))
        done |= conv & active
        prev = maxw
        if done.all():
            break
    return z, its


def select(z):
    r2 = np.abs(z) ** 2
    d = np.abs(r2 - 1) / (r2 + 1)
    i = np.argmin(d, axis=1)
    return z[np.arange(z.shape[0]), i]


def run(win, M, **kw):
    """win [N,M,M] complex128 → alpha (emulated FP32 rooting; eigvecs via FP64 eigh)."""
    w32 = win.astype(c64)
    R = w32 @ np.conj(np.swapaxes(w32, 1, 2))
    _, V = np.linalg.eigh(R.astype(np.complex128))
    u = V[:, :, -1].astype(c64)
    v = np.einsum("nik,ni->nk", np.conj(w32), u)
    v = (v / np.linalg.norm(v, axis=1, keepdims=True)).astype(c64)
    T = template(M).astype(c64)[: M - 1]
    zs = []
    its = []
    for q in (u, v):
        c, rot = coeffs(q)
        z, it = aberth_sym(c, T[None, :] * rot[:, None], **kw)
        zs.append(select(z))
        its.append(it)
    zy, zx = zs
    o = np.arange(M) - (M - 1) // 2
    hx, hy = zx / np.abs(zx), zy / np.abs(zy)
    basis = hx[:, None, None] ** o[None, None, :] * np.conj(hy)[:, None, None] ** o[None, :, None]
    cs = np.sum(win * basis, axis=(1, 2))
    return np.angle(cs), its


if __name__ == "__main__":
    import torch  # noqa: F401
    from oracle import rootmusic as R
    from paper_1910_11872_b200 import synth
    name = sys.argv[1] if len(sys.argv) > 1 else "C1"
    M = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    near = float(sys.argv[3]) if len(sys.argv) > 3 else 2e-3
    w = synth.workload(name)
    t = 0 if name.startswith("C1") else 1
    f = synth.make_frame(w, t).numpy()
    rng = np.random.default_rng(0)
    n = 4000
    py, px = rng.integers(M, w.H - M, n), rng.integers(M, w.W - M, n)
    win, _ = R.extract_windows(f, py, px, M)
    ref = R.estimate_windows(win)
    a, its = run(win, M, near_tol=near)
    e = R.wrap(a - ref["alpha"])
    ok = (ref["flags"] & R.PARITY_EXCLUDE_MASK) == 0
    print(f"{name} M={M} near={near}: rms {math.sqrt(np.mean(e[ok]**2)):.2e} max {np.max(np.abs(e[ok])):.2e} "
          f"sweeps y {its[0].mean():.2f} (max {its[0].max()}) x {its[1].mean():.2f}")
