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


# ---------------------------------------------------------------------------
# operator algebra: V_h, K_h, D_h on the device vs the
# dense compositions of the oracle's matrices (operators.cpp:97-158)
@pytest.fixture(scope="module")
def opset():
    mesh = hm.Mesh.icosphere(2)
    a = mesh.arrays()
    E, nu, eps = 1.0, 0.3, 1e-7
    ops = hm.OperatorSet(mesh, E, nu, b_min=16, eta=1.0, device=0)
    ops.assemble(eps=eps, beta=0.8)
    V, T = a["vertices"], a["triangles"]
    m, n = len(T), len(V)
    lam, mu = hm.lame_constants(E, nu)
    vd = orc.Problem.galerkin(V, T, 1, b_min=16, eta=1.0).dense(0)
    vg = orc.Problem.galerkin(V, T, 0, b_min=16, eta=1.0).dense_grid()
    kd = orc.Problem.kdelta(V, T, b_min=16, eta=1.0).dense(0)
    t12, t13, t23 = (orc.sparse_op(V, T, w) for w in range(3))
    Z = np.zeros((m, n))
    Th = np.block([[Z, t12, t13], [-t12, Z, t23], [-t13, -t23, Z]])
    D3 = np.kron(np.eye(3), vd)
    Vh = 0.5 / E * (1 + nu) / (1 - nu) * ((3 - 4 * nu) * D3 + vg)
    Kh = np.kron(np.eye(3), kd) - D3 @ Th + 2 * mu * Vh @ Th
    S = [np.kron(np.eye(3), -t23), np.kron(np.eye(3), t13), np.kron(np.eye(3), t12)]
    Dh = sum(mu * Sk.T @ D3 @ Sk for Sk in S) + 2 * mu * Th.T @ D3 @ Th \
        - 4 * mu * mu * Th.T @ Vh @ Th
    tl = {(0, 1): t12, (0, 2): t13, (1, 2): t23}
    def ts(k, l):
        return None if k == l else (1.0 if k < l else -1.0) * tl[(min(k, l), max(k, l))]
    G = np.zeros((3 * n, 3 * n))
    for i in range(3):
        for j in range(3):
            for k in range(3):
                if k in (i, j):
                    continue
                G[i * n:(i + 1) * n, j * n:(j + 1) * n] += ts(k, j).T @ vd @ ts(k, i)
    Dh = Dh + mu * G
    return dict(ops=ops, Vh=Vh, Kh=Kh, Dh=Dh, m=m, n=n, eps=eps, t=(t12, t13, t23))


def test_sparse_ops_match_oracle(opset):
    ops, t = opset["ops"], opset["t"]
    torch = pytest.importorskip("torch")
    n = opset["n"]
    x = RV(n, 11)
    xd = torch.tensor(x, device="cuda")
    for w in range(3):
        y = ops._spmv(w, xd).cpu().numpy()
        assert np.allclose(y, t[w] @ x, rtol=1e-13, atol=1e-13 * np.abs(t[w] @ x).max())
        z = RV(opset["m"], 12)
        yt = ops._spmv(w, torch.tensor(z, device="cuda"), transpose=True).cpu().numpy()
        assert np.allclose(yt, t[w].T @ z, rtol=1e-13, atol=1e-13 * np.abs(t[w].T @ z).max())


def test_composed_operators_match_dense(opset):
    ops, eps = opset["ops"], opset["eps"]
    m, n = opset["m"], opset["n"]
    xm, xn = RV(3 * m, 13), RV(3 * n, 14)
    assert rel(ops.vh(xm), opset["Vh"] @ xm) <= 10 * eps
    assert rel(ops.kh(xn), opset["Kh"] @ xn) <= 100 * eps
    assert rel(ops.dh(xn), opset["Dh"] @ xn) <= 100 * eps
    zm = RV(3 * m, 15)
    assert rel(ops.kh_t(zm), opset["Kh"].T @ zm) <= 100 * eps
    # D_h is symmetric; constants are in its kernel (rigid translations)
    Dh = opset["Dh"]
    assert np.allclose(Dh, Dh.T, rtol=0, atol=1e-10 * np.abs(Dh).max())
    ones = np.concatenate([np.ones(n), np.zeros(2 * n)])
    assert np.linalg.norm(ops.dh(ones)) <= 1e-6 * np.linalg.norm(Dh) * np.sqrt(n)
