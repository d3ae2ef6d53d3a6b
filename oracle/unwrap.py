"""FP64 oracle for SURVEY §8 row f2: 2-D phase unwrapping by reliability sorting (Herráez).

TEST INFRASTRUCTURE, NOT PRODUCT CODE (see ``oracle/__init__.py``).

P:L218: "The above process is repeated for all blocks and followed by an unwrapping
operation [Herráez et al. 2002] to obtain the overall phase map."  The paper gives no
details; the reading ([R12]) is the cited algorithm as SPEC S:L285-322 states
it, step by step:

1. reliability of pixel (i,j): R = 1/D, D = sqrt(H² + V² + D1² + D2²) with the wrapped second
   differences H = γ(φ(i,j−1) − φ(i,j)) − γ(φ(i,j) − φ(i,j+1)), V (rows), D1, D2 (diagonals);
   neighbours outside the frame replicate the edge pixel; γ = wrap into (−π, π];
2. edges between 4-neighbours, reliability R(p) + R(q); edge id 2p (p → p+1, horizontal),
   2p+1 (p → p+W, vertical);
3. edges processed by decreasing reliability, ties by increasing edge id; when an
   edge joins two groups, the group with fewer pixels (ties: q's group) is shifted by the
   multiple of 2π that makes the unwrapped difference across the edge equal γ(φ(q) − φ(p));
4. the result is shifted by one global multiple of 2π so that the most reliable pixel
   (ties: lowest index) keeps its wrapped value.

All arithmetic in float64 with the same operation order as the CUDA kernels' FP64 steps
(reliability ordering must agree exactly); the 2π multiples are carried as integers.
Non-finite input pixels are treated as 0 in the arithmetic and returned as NaN.
"""

from __future__ import annotations

import numpy as np

TWO_PI = 2.0 * np.pi


def gamma(d):
    """wrap into (−π, π]:  d − 2π·ceil((d − π)/2π)."""
    return d - TWO_PI * np.ceil((d - np.pi) / TWO_PI)


def reliability(phase: np.ndarray) -> np.ndarray:
    """Step 1: R = 1/D (float64 [H,W]); D = 0 gives +inf."""
    p = np.asarray(phase, np.float64)
    p = np.where(np.isfinite(p), p, 0.0)
    H, W = p.shape
    pad = np.pad(p, 1, mode="edge")
    c = pad[1:H + 1, 1:W + 1]

    def at(di, dj):
        return pad[1 + di:H + 1 + di, 1 + dj:W + 1 + dj]

    h = gamma(at(0, -1) - c) - gamma(c - at(0, 1))
    v = gamma(at(-1, 0) - c) - gamma(c - at(1, 0))
    d1 = gamma(at(-1, -1) - c) - gamma(c - at(1, 1))
    d2 = gamma(at(-1, 1) - c) - gamma(c - at(1, -1))
    D = np.sqrt(h * h + v * v + d1 * d1 + d2 * d2)
    with np.errstate(divide="ignore"):
        return 1.0 / D


def edges(H: int, W: int, rel: np.ndarray):
    """Step 2: (ids, p, q, reliability) of every 4-neighbour edge."""
    idx = np.arange(H * W).reshape(H, W)
    ph, qh = idx[:, :-1].ravel(), idx[:, 1:].ravel()
    pv, qv = idx[:-1, :].ravel(), idx[1:, :].ravel()
    p = np.concatenate([ph, pv])
    q = np.concatenate([qh, qv])
    ids = np.concatenate([2 * ph, 2 * pv + 1])
    r = rel.ravel()
    return ids, p, q, r[p] + r[q]


def unwrap_k(phase: np.ndarray) -> np.ndarray:
    """Steps 1-4; returns the integer 2π multiples k (int64 [H,W]): unwrapped = φ + 2πk."""
    p = np.asarray(phase, np.float64)
    H, W = p.shape
    w = np.where(np.isfinite(p), p, 0.0).ravel()
    rel = reliability(p)
    ids, ep, eq, er = edges(H, W, rel)
    order = np.lexsort((ids, -er))                       # decreasing reliability, then id
    n = H * W
    k = np.zeros(n, np.int64)
    group = np.arange(n)
    members = {i: [i] for i in range(n)}
    for e in order:
        a, b = int(ep[e]), int(eq[e])
        ga, gb = group[a], group[b]
        if ga == gb:
            continue
        # k(b) − k(a) must equal e_ab = (γ(w_b − w_a) − (w_b − w_a)) / 2π
        dw = w[b] - w[a]
        e_ab = int(np.rint((gamma(dw) - dw) / TWO_PI))
        shift = k[a] + e_ab - k[b]                       # add to group b (or −shift to group a)
        if len(members[ga]) < len(members[gb]):
            small, big, delta = ga, gb, -shift
        else:
            small, big, delta = gb, ga, shift
        ms = members.pop(small)
        k[ms] += delta
        group[ms] = big
        members[big].extend(ms)
    top = int(np.argmax(rel.ravel()))                      # most reliable pixel, lowest index on ties
    k -= k[top]
    return k.reshape(H, W)


def unwrap(phase: np.ndarray) -> np.ndarray:
    """Unwrapped phase (float64 [H,W]); NaN where the input is not finite."""
    p = np.asarray(phase, np.float64)
    out = np.where(np.isfinite(p), p, 0.0) + TWO_PI * unwrap_k(p)
    return np.where(np.isfinite(p), out, np.nan)
