"""Independent checks for the Galerkin pair quadrature: numpy restatements of
the reference's TEST-side oracles (proj/tests/oracles.cpp:140-290), which do
not use the production coordinate transforms:

  gauss_pair / recurse_pair / bruteforce_pair_integral  (oracles.cpp:140-207)
  analytic_triangle_potential                            (oracles.cpp:209-232)
  outer_graded / vdelta_singular_oracle                  (oracles.cpp:236-281)

Test infrastructure only.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc

_R6 = orc.gauss_rule(6)  # (a, b, w) of the 12-point order-6 rule


def _area(t):
    return 0.5 * np.linalg.norm(np.cross(t[1] - t[0], t[2] - t[0]))


def _pts(t, a, b):
    return t[0] + a[:, None] * (t[1] - t[0]) + b[:, None] * (t[2] - t[0])


def gauss_pair(tx, ty, kernel):
    """plain tensor Gauss (order 6 x order 6) on a pair (oracles.cpp:140-158)."""
    a, b, w = _R6
    X = _pts(tx, a, b)
    Y = _pts(ty, a, b)
    K = kernel(X[:, None, :], Y[None, :, :])
    return 4.0 * _area(tx) * _area(ty) * float(w @ K @ w)


def _diam(t):
    return max(np.linalg.norm(t[0] - t[1]), np.linalg.norm(t[1] - t[2]),
               np.linalg.norm(t[0] - t[2]))


def _dist(a, b):
    return min(np.linalg.norm(p - q) for p in a for q in b)


def split4(t):
    m01 = 0.5 * (t[0] + t[1])
    m12 = 0.5 * (t[1] + t[2])
    m02 = 0.5 * (t[0] + t[2])
    return [np.array([t[0], m01, m02]), np.array([m01, t[1], m12]),
            np.array([m02, m12, t[2]]), np.array([m01, m12, m02])]


def bruteforce_pair_integral(tx, ty, kernel, max_depth=14):
    """recursive uniform subdivision, Gauss on separated sub-pairs
    (oracles.cpp:178-207)."""
    tx, ty = np.asarray(tx, float), np.asarray(ty, float)
    if _dist(tx, ty) > 1.0 * max(_diam(tx), _diam(ty)) or max_depth == 0:
        return gauss_pair(tx, ty, kernel)
    acc = 0.0
    for sx in split4(tx):
        for sy in split4(ty):
            acc += bruteforce_pair_integral(sx, sy, kernel, max_depth - 1)
    return acc


def analytic_triangle_potential(P, tri):
    """int_T 1/|p - y| dA_y, per-edge log/atan formula (oracles.cpp:209-232);
    P is (k, 3)."""
    tri = np.asarray(tri, float)
    P = np.atleast_2d(P)
    nrm = np.cross(tri[1] - tri[0], tri[2] - tri[0])
    nrm = nrm / np.linalg.norm(nrm)
    d = (P - tri[0]) @ nrm
    proj = P - d[:, None] * nrm
    acc = np.zeros(len(P))
    ad = np.abs(d)
    for e in range(3):
        a, b = tri[e], tri[(e + 1) % 3]
        s_hat = (b - a) / np.linalg.norm(b - a)
        m_hat = np.cross(s_hat, nrm)
        t = (a - proj) @ m_hat
        s1 = (a - proj) @ s_hat
        s2 = (b - proj) @ s_hat
        r1 = np.linalg.norm(P - a, axis=1)
        r2 = np.linalg.norm(P - b, axis=1)
        r0sq = t * t + d * d
        ok = (r1 + s1 > 0) & (r2 + s2 > 0)
        with np.errstate(divide="ignore", invalid="ignore"):
            lg = np.where(ok, t * np.log(np.where(ok, (r2 + s2) / np.where(ok, r1 + s1, 1.0), 1.0)), 0.0)
        acc += lg
        acc -= ad * (np.arctan2(t * s2, r0sq + ad * r2) - np.arctan2(t * s1, r0sq + ad * r1))
    return acc


def _dist_to_segment(p, a, b):
    ab = b - a
    t = np.clip(ab @ (p - a) / (ab @ ab), 0.0, 1.0)
    return np.linalg.norm(a + t * ab - p)


def vdelta_singular_oracle(tri_x, tri_y, depth=12):
    """V_Delta entry of touching pairs: analytic inner potential, outer Gauss
    graded towards the trial boundary (oracles.cpp:236-281), iterative."""
    tri_x, tri_y = np.asarray(tri_x, float), np.asarray(tri_y, float)
    a, b, w = _R6
    cells = [(tri_x, depth)]
    total = 0.0
    leaves = []
    while cells:
        cell, dep = cells.pop()
        h = _diam(cell)
        front = min(_dist_to_segment(c, tri_y[e], tri_y[(e + 1) % 3])
                    for c in cell for e in range(3))
        if dep == 0 or front > 0.5 * h:
            leaves.append(cell)
        else:
            cells.extend((s, dep - 1) for s in split4(cell))
    for i in range(0, len(leaves), 4096):
        chunk = np.array(leaves[i:i + 4096])
        X = (chunk[:, 0, None, :] + a[None, :, None] * (chunk[:, 1] - chunk[:, 0])[:, None, :]
             + b[None, :, None] * (chunk[:, 2] - chunk[:, 0])[:, None, :])
        pot = analytic_triangle_potential(X.reshape(-1, 3), tri_y).reshape(len(chunk), -1)
        areas = 0.5 * np.linalg.norm(np.cross(chunk[:, 1] - chunk[:, 0],
                                              chunk[:, 2] - chunk[:, 0]), axis=1)
        total += float(np.sum(2.0 * areas * (pot @ w)))
    return total / (4.0 * np.pi)


def integrate_with_rule(tx, ty, case, order, kernel):
    """production pair rule on physical triangles (test_quadrature.cpp:119-133)."""
    xr1, xr2, yr1, yr2, w = orc.pair_rule(case, order)
    tx, ty = np.asarray(tx, float), np.asarray(ty, float)
    X = _pts(tx, xr1, xr2)
    Y = _pts(ty, yr1, yr2)
    return 4.0 * _area(tx) * _area(ty) * float(np.sum(w * kernel(X, Y)))


def newton_kernel(X, Y):
    return 1.0 / np.linalg.norm(X - Y, axis=-1)


def smooth_kernel(X, Y):
    return np.cos(X @ np.array([1.0, 2.0, 3.0])) * np.exp(-0.3 * np.sum((Y - X) ** 2, axis=-1))
