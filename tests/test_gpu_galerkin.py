"""GPU parity of the Galerkin scalar kernels: V_Delta
and the six V_kl over triangle pairs with the reference's pair quadrature
(disjoint tensor rules and Sauter-Schwab transforms for touching pairs,
proj/src/kernels.cpp:95-149, quadrature.cpp:127-338), assembled by the same
ACA / near-field / matvec engine, against the CPU oracle; and the Lame
single-layer composition V_h (compose_Vh, operators.cpp:97-105)."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
RV = orc.random_vector
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module", params=[0, 1], ids=["vkl", "vdelta"])
def gal(request):
    which = request.param
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    eps = 1e-5
    g = hm.HMatrix.galerkin(mesh, which, b_min=32, eta=1.0, device=0)
    st = g.assemble(eps=eps, beta=0.8, lookahead=2)
    o = orc.Problem.galerkin(a["vertices"], a["triangles"], which, b_min=32, eta=1.0)
    o.assemble(eps=eps, beta=0.8, lookahead=2)
    return dict(g=g, o=o, eps=eps, which=which, st=st, nc=6 if which == 0 else 1)


def test_partition_identical(gal):
    assert gal["g"].partition_json() == gal["o"].partition_json()


def test_nearfield_entries_bit_identical(gal):
    g, o = gal["g"], gal["o"]
    nodes = g.tree().nodes
    blocks = g.partition_blocks()
    n_touch = 0
    for comp in range(gal["nc"]):
        for b, (rn, cn, adm, _) in enumerate(blocks):
            if adm:
                continue
            m = nodes[rn, 1] - nodes[rn, 0]
            n = nodes[cn, 1] - nodes[cn, 0]
            want = o.dense_block(comp, b, m, n)
            got = g.dense_block(comp, b)
            assert (got == want).all(), (comp, b, np.abs(got - want).max())
            n_touch += rn == cn
    assert n_touch > 0  # diagonal blocks (identical / edge / vertex pairs) covered


def test_ranks_and_factors_bit_identical(gal):
    g, o = gal["g"], gal["o"]
    gk, gl, gc, _ = g.ranks()
    ok, ol, oc, _ = o.ranks()
    assert (gk == ok).all() and (gl == ol).all() and (gc == oc).all()
    blocks = g.partition_blocks()
    adm = np.nonzero(blocks[:, 2])[0]
    for b in adm[:: max(1, len(adm) // 30)]:
        for comp in range(0, gal["nc"], 2):
            fg, fo = g.factor(comp, b), o.factor(comp, b)
            assert (fg["pivots"] == fo["pivots"]).all()
            assert (fg["U"] == fo["U"]).all() and (fg["V"] == fo["V"]).all()
            assert fg["frob_sq"] == fo["frob_sq"]


def test_matvec_vs_oracle_and_dense(gal):
    g, o, eps = gal["g"], gal["o"], gal["eps"]
    x = RV(g.cols, 0)
    y = g.matvec(x)
    assert rel(y, o.matvec(x)) <= 1e-12
    assert rel(y, o.dense_grid() @ x) <= 10 * eps
    X = np.stack([RV(g.cols, s) for s in range(3)], axis=1)
    Y = g.matvec(X)
    for q in range(3):
        assert rel(Y[:, q], g.matvec(X[:, q])) <= 1e-12


def test_lame_single_layer_composition():
    """V_h through the package against the dense composition of the oracle's
    V_Delta and V_kl matrices (compose_Vh, operators.cpp:97-105)."""
    mesh = hm.Mesh.icosphere(2)
    a = mesh.arrays()
    E, nu, eps = 1.0, 0.3, 1e-6
    vh = hm.LameSingleLayer(mesh, E, nu, b_min=16, eta=1.0, device=0)
    vh.assemble(eps=eps, beta=0.8)
    nt = len(a["triangles"])
    grid = orc.Problem.galerkin(a["vertices"], a["triangles"], 0, b_min=16, eta=1.0)
    vd = orc.Problem.galerkin(a["vertices"], a["triangles"], 1, b_min=16, eta=1.0)
    A = 0.5 / E * (1.0 + nu) / (1.0 - nu) * (
        (3.0 - 4.0 * nu) * np.kron(np.eye(3), vd.dense(0)) + grid.dense_grid())
    x = RV(3 * nt, 7)
    assert rel(vh.matvec(x), A @ x) <= 10 * eps
    # symmetric positive definite (the single-layer operator is elliptic)
    assert np.allclose(A, A.T, rtol=0, atol=1e-15 * np.abs(A).max())
    assert np.linalg.eigvalsh(A).min() > 0


def test_cta_mode_bit_identical(gal):
    """Items run CTA-cooperatively (HMGPU_ACA_CTA_MIN) give the warp mode's
    bits: a subprocess with every item of m+n >= 64 in CTA mode reproduces
    this process's ranks and matvec exactly."""
    if gal["which"] != 0:
        pytest.skip("one instance is enough")
    g = gal["g"]
    x = RV(g.cols, 3)
    y = g.matvec(x)
    code = ("import sys, numpy as np; sys.path.insert(0, %r);"
            "import paper_2205_04752_b200 as hm; from oracle import oracle as orc;"
            "g = hm.HMatrix.galerkin(hm.Mesh.icosphere(3), 0, b_min=32, eta=1.0, device=0);"
            "g.assemble(eps=1e-5, beta=0.8, lookahead=2);"
            "y = g.matvec(orc.random_vector(g.cols, 3)); k = g.ranks()[1];"
            "sys.stdout.write(y.tobytes().hex() + ' ' + k.tobytes().hex())" % ROOT)
    env = dict(os.environ, HMGPU_ACA_CTA_MIN="64")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                         text=True, check=True).stdout.split()
    assert out[0] == y.tobytes().hex()
    assert out[1] == g.ranks()[1].tobytes().hex()


@pytest.fixture(scope="module")
def kdelta():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    eps = 1e-5
    g = hm.HMatrix.kdelta(mesh, b_min=32, eta=1.0, device=0)
    g.assemble(eps=eps, beta=0.8, lookahead=2)
    o = orc.Problem.kdelta(a["vertices"], a["triangles"], b_min=32, eta=1.0)
    o.assemble(eps=eps, beta=0.8, lookahead=2)
    return dict(g=g, o=o, eps=eps)


def test_kdelta_partition_and_nearfield(kdelta):
    g, o = kdelta["g"], kdelta["o"]
    assert g.partition_json() == o.partition_json()
    rnodes, cnodes = g.tree(0).nodes, g.tree(1).nodes
    for b, (rn, cn, adm, _) in enumerate(g.partition_blocks()):
        if adm:
            continue
        m = rnodes[rn, 1] - rnodes[rn, 0]
        n = cnodes[cn, 1] - cnodes[cn, 0]
        assert (g.dense_block(0, b) == o.dense_block(0, b, m, n)).all(), b


def test_kdelta_ranks_factors_matvec(kdelta):
    g, o, eps = kdelta["g"], kdelta["o"], kdelta["eps"]
    gk, gl, gc, _ = g.ranks()
    ok, ol, oc, _ = o.ranks()
    assert (gk == ok).all() and (gl == ol).all() and (gc == oc).all()
    adm = np.nonzero(g.partition_blocks()[:, 2])[0]
    for b in adm[:: max(1, len(adm) // 30)]:
        fg, fo = g.factor(0, b), o.factor(0, b)
        assert (fg["U"] == fo["U"]).all() and (fg["V"] == fo["V"]).all()
    x = RV(g.cols, 2)
    y = g.matvec(x)
    assert rel(y, o.matvec(x)) <= 1e-12
    assert rel(y, o.dense(0) @ x) <= 10 * eps
