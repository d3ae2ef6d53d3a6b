"""Pins of the row-f2 oracle (Herráez reliability-sorted unwrapping), CPU only."""

import math
from collections import deque

import numpy as np
import pytest

from oracle import unwrap as U


def wrap(x):
    return U.gamma(np.asarray(x, np.float64))


def test_ramp_recovered():
    """wrap(0.3x) on 64×64 → 0.3x + one global 2πk."""
    y, x = np.mgrid[0:64, 0:64]
    truth = 0.3 * x
    u = U.unwrap(wrap(truth))
    d = u - truth
    assert np.allclose(d, d[0, 0], atol=1e-9)
    assert abs(d[0, 0] / (2 * math.pi) - round(d[0, 0] / (2 * math.pi))) < 1e-12


@pytest.mark.parametrize("seed", range(6))
def test_smooth_surfaces_exact(seed):
    """Any surface whose true neighbour differences are < π is recovered up to one global 2πk
    (S:L309); includes the wrapped 12-rad Gaussian peak of S:L304."""
    rng = np.random.default_rng(seed)
    H, W = 40 + seed, 52
    y, x = np.mgrid[0:H, 0:W]
    truth = 12.0 * np.exp(-((x - W / 2) ** 2 + (y - H / 2) ** 2) / (2 * 9.0 ** 2))
    truth += rng.uniform(-0.4, 0.4) * x + rng.uniform(-0.4, 0.4) * y
    assert np.max(np.abs(np.diff(truth, axis=0))) < math.pi and np.max(np.abs(np.diff(truth, axis=1))) < math.pi
    u = U.unwrap(wrap(truth))
    d = u - truth
    assert np.max(np.abs(d - d.flat[0])) < 1e-9
    assert abs(d.flat[0] / (2 * math.pi) - round(d.flat[0] / (2 * math.pi))) < 1e-9


def test_congruence_and_anchor_on_noise():
    rng = np.random.default_rng(9)
    w = wrap(rng.uniform(-4, 4, (30, 33)))
    u = U.unwrap(w)
    assert np.max(np.abs(wrap(u) - w)) < 1e-12
    top = np.argmax(U.reliability(w).ravel())
    assert u.flat[top] == w.flat[top]                   # the anchor keeps its wrapped value


def _kruskal_bfs_k(w):
    """Independent construction: maximum spanning tree by Kruskal (same edge order), then
    integrate the wrapped differences along the tree by BFS from the anchor."""
    H, W = w.shape
    rel = U.reliability(w)
    ids, ep, eq, er = U.edges(H, W, rel)
    order = np.lexsort((ids, -er))
    parent = list(range(H * W))

    def find(a):
        while parent[a] != a:
            parent[a] = parent[parent[a]]
            a = parent[a]
        return a

    adj = [[] for _ in range(H * W)]
    for e in order:
        a, b = int(ep[e]), int(eq[e])
        ra, rb = find(a), find(b)
        if ra != rb:
            parent[ra] = rb
            adj[a].append(b)
            adj[b].append(a)
    flat = w.ravel()
    top = int(np.argmax(rel.ravel()))
    k = np.full(H * W, np.iinfo(np.int64).min, np.int64)
    k[top] = 0
    dq = deque([top])
    while dq:
        a = dq.popleft()
        for b in adj[a]:
            if k[b] == np.iinfo(np.int64).min:
                dw = flat[b] - flat[a]
                k[b] = k[a] + int(np.rint((U.gamma(dw) - dw) / (2 * math.pi)))
                dq.append(b)
    return k.reshape(H, W)


@pytest.mark.parametrize("seed", range(4))
def test_group_merging_equals_spanning_tree_integration(seed):
    """Herráez's group shifting is integration of the wrapped differences along the maximum
    spanning tree of the reliability-ordered edges: an independent Kruskal+BFS gives the same
    2π multiples on noisy maps (the property the GPU Borůvka build relies on)."""
    rng = np.random.default_rng(100 + seed)
    H, W = 23, 31
    y, x = np.mgrid[0:H, 0:W]
    truth = 0.9 * x - 0.5 * y + 3 * np.sin(x / 5.0)
    w = wrap(truth + rng.normal(0, 0.6 + 0.3 * seed, (H, W)))
    assert np.array_equal(U.unwrap_k(w), _kruskal_bfs_k(w))


def test_nonfinite_pixels_are_nan():
    w = wrap(np.linspace(0, 20, 15 * 17).reshape(15, 17))
    w[4, 5] = np.nan
    u = U.unwrap(w)
    assert np.isnan(u[4, 5]) and np.isfinite(np.delete(u.ravel(), 4 * 17 + 5)).all()
