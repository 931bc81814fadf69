"""The single-layer grid of evaluate_interior (proj/src/baca.cpp:625-687):
Kelvin collocation at interior points (CollocSingleOracle, kernels.hpp:
107-126) on the device vs the oracle -- partition, entries, ACA factors and
the matvec bit for bit / to rounding."""
import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc

RV = orc.random_vector


def interior_points(n, seed, radius=0.8):
    rng = np.random.default_rng(seed)
    p = rng.normal(size=(n, 3))
    return p / np.linalg.norm(p, axis=1)[:, None] * rng.uniform(0.0, radius, (n, 1))


def test_partition_and_rejection_host():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    P = interior_points(700, 0)
    h = hm.HMatrix.kelvin_points(mesh, P, b_min=32, eta=1.0, device=-1)
    o = orc.Problem.kelvin_points(a["vertices"], a["triangles"], P, b_min=32, eta=1.0)
    assert (h.rows, h.cols) == (3 * 700, 3 * 1280)
    assert h.partition_json() == o.partition_json()
    with pytest.raises(hm.Error):  # baca.cpp:632-643
        hm.HMatrix.kelvin_points(mesh, np.array([[0.99, 0.0, 0.0]]), device=-1)


@pytest.mark.gpu
def test_interior_single_layer_matches_oracle():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    P = interior_points(700, 0)
    eps = 1e-5
    g = hm.HMatrix.kelvin_points(mesh, P, b_min=32, eta=1.0, device=0)
    g.assemble(eps=eps, beta=0.8, lookahead=2)
    o = orc.Problem.kelvin_points(a["vertices"], a["triangles"], P, b_min=32, eta=1.0)
    o.assemble(eps=eps, beta=0.8, lookahead=2)
    rn, cn = g.tree(0).nodes, g.tree(1).nodes
    blocks = g.partition_blocks()
    for comp in (0, 1, 4):
        for b, (r, c, adm, _) in enumerate(blocks):
            if adm:
                continue
            m, n = rn[r, 1] - rn[r, 0], cn[c, 1] - cn[c, 0]
            assert (g.dense_block(comp, b) == o.dense_block(comp, b, m, n)).all()
    gk, gl, gc, _ = g.ranks()
    ok, ol, oc, _ = o.ranks()
    assert (gk == ok).all() and (gl == ol).all() and (gc == oc).all()
    t = RV(g.cols, 4)
    y = g.matvec(t)
    assert np.linalg.norm(y - o.matvec(t)) <= 1e-12 * np.linalg.norm(y)
    A = o.dense_grid()
    assert np.linalg.norm(y - A @ t) <= 10 * eps * np.linalg.norm(A @ t)


def kelvin_traction(x, n, E=1.0, nu=0.3):
    """kelvin_traction (kernels.cpp:30-55), literal, test side."""
    lam = E * nu / ((1 + nu) * (1 - 2 * nu))
    mu = E / (2 * (1 + nu))
    c = (1 + nu) / (8 * np.pi * E * (1 - nu))
    r = np.linalg.norm(x)
    r3, r5 = r ** 3, r ** 5
    k34 = 3 - 4 * nu

    def dU(k, i, j):
        v = -k34 * (x[k] / r3 if i == j else 0.0)
        v += ((x[j] if i == k else 0.0) + (x[i] if j == k else 0.0)) / r3
        v -= 3 * x[i] * x[j] * x[k] / r5
        return c * v

    t = np.zeros((3, 3))
    for j in range(3):
        div_j = -2 * c * (1 - 2 * nu) * x[j] / r3
        for i in range(3):
            t[i, j] = lam * n[i] * div_j + sum(mu * n[k] * (dU(k, i, j) + dU(i, k, j))
                                               for k in range(3))
    return t


@pytest.mark.gpu
def test_double_layer_cell_matches_oracle():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    P = interior_points(500, 1)
    eps = 1e-6
    for (r, c) in ((0, 1), (2, 2)):
        g = hm.HMatrix.kelvin_double(mesh, P, r, c, b_min=32, eta=1.0, device=0)
        g.assemble(eps=eps, beta=0.8, lookahead=2)
        o = orc.Problem.kelvin_double(a["vertices"], a["triangles"], P, r, c, b_min=32,
                                      eta=1.0)
        o.assemble(eps=eps, beta=0.8, lookahead=2)
        assert g.partition_json() == o.partition_json()
        rn, cn = g.tree(0).nodes, g.tree(1).nodes
        for b, (rr, cc, adm, _) in enumerate(g.partition_blocks()):
            if adm:
                continue
            m, n = rn[rr, 1] - rn[rr, 0], cn[cc, 1] - cn[cc, 0]
            assert (g.dense_block(0, b) == o.dense_block(0, b, m, n)).all()
        gk, gl, _, _ = g.ranks()
        ok, ol, _, _ = o.ranks()
        assert (gk == ok).all() and (gl == ol).all()
        u = RV(g.cols, 6)
        y = g.matvec(u)
        assert np.linalg.norm(y - o.matvec(u)) <= 1e-12 * np.linalg.norm(y)
        D = o.dense(0)
        assert np.linalg.norm(y - D @ u) <= 10 * eps * np.linalg.norm(D @ u)


@pytest.mark.gpu
def test_interior_representation_reproduces_manufactured_field():
    """test_kernels.cpp:278-308 through the H-matrices: u(x) = S(x - p) a with
    p outside; v = V~ t - W~ u with the exact Cauchy data reproduces u."""
    mesh = hm.Mesh.voxel_cube(6, -1.0, 1.0)
    ar = mesh.arrays()
    V, T, Cc, N = ar["vertices"], ar["triangles"], ar["centroids"], ar["normals"]
    p = np.array([5.0, 5.0, 5.0])
    av = np.ones(3) / np.sqrt(3.0)
    nt, nv = len(T), len(V)
    t_tot = np.zeros(3 * nt)
    for i in range(nt):
        t_tot[[i, nt + i, 2 * nt + i]] = kelvin_traction(Cc[i] - p, N[i]) @ av
    u_tot = np.zeros(3 * nv)
    for v in range(nv):
        u_tot[[v, nv + v, 2 * nv + v]] = orc.kelvin_tensor(V[v] - p) @ av
    X = np.array([[0.2, -0.1, 0.3], [-0.4, 0.5, 0.0]])
    ev = hm.InteriorEvaluator(mesh, X, b_min=8, eta=1.0, device=0, disjoint_order=5)
    ev.assemble(eps=1e-8)
    got = ev.evaluate(t_tot, u_tot).reshape(3, -1).T
    for k, x in enumerate(X):
        want = orc.kelvin_tensor(x - p) @ av
        assert np.linalg.norm(got[k] - want) <= 2e-2 * np.linalg.norm(want)
