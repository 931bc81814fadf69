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
