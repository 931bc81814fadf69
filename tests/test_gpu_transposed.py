"""Transposed H-matvec on the device (HMatrix::matvec_transposed,
proj/src/hmatrix.cpp:47-72) against the oracle's
transposed product, the dense transpose and the adjoint identity."""
import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc
from tests.helpers import centroid_points_and_boxes, cube_mesh

pytestmark = pytest.mark.gpu
RV = orc.random_vector


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_kdelta_transposed_vs_oracle():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    eps = 1e-5
    g = hm.HMatrix.kdelta(mesh, b_min=32, eta=1.0, device=0)
    g.assemble(eps=eps, beta=0.8, lookahead=2)
    o = orc.Problem.kdelta(a["vertices"], a["triangles"], b_min=32, eta=1.0)
    o.assemble(eps=eps, beta=0.8, lookahead=2)
    x = RV(g.rows, 3)
    y = g.matvec_transposed(x)
    assert y.shape == (g.cols,)
    assert rel(y, o.matvec_transposed(x)) <= 1e-12
    assert rel(y, o.dense(0).T @ x) <= 10 * eps
    yl = g.matvec_transposed(x, hm.Mode.Lookahead)
    assert rel(yl, o.matvec_transposed(x, 1)) <= 1e-12
    X = np.stack([RV(g.rows, s) for s in range(2)], axis=1)
    Y = g.matvec_transposed(X)
    for q in range(2):
        assert rel(Y[:, q], g.matvec_transposed(X[:, q])) <= 1e-13


def test_newton_transposed_vs_oracle():
    mesh = cube_mesh(4)
    pts, boxes = centroid_points_and_boxes(mesh)
    g = hm.HMatrix.newton(pts, boxes, diag=2.0, b_min=10, eta=0.8, device=0)
    g.assemble(eps=1e-6, beta=0.8)
    o = orc.Problem.newton(pts, boxes, 2.0, b_min=10, eta=0.8)
    o.assemble(eps=1e-6, beta=0.8)
    x = RV(g.rows, 5)
    assert rel(g.matvec_transposed(x), o.matvec_transposed(x)) <= 1e-12


def test_kelvin_grid_transposed_adjoint_and_dense():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    eps = 1e-4
    g = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
    g.assemble(eps=eps, beta=0.8)
    x, z = RV(g.rows, 1), RV(g.cols, 2)
    yt = g.matvec_transposed(x)
    # <A^T x, z> = <x, A z> up to rounding (the same stored factors)
    lhs, rhs = float(yt @ z), float(x @ g.matvec(z))
    assert abs(lhs - rhs) <= 1e-12 * np.linalg.norm(yt) * np.linalg.norm(z)
    o = orc.Problem.kelvin(a["vertices"], a["triangles"], 1.0, 0.3, b_min=32, eta=1.0)
    assert rel(yt, o.dense_grid().T @ x) <= 10 * eps
