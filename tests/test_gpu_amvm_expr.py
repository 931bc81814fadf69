"""The adaptive matvec over a composite operator (amvm_multiply on an
expression, proj/src/amvm.cpp:199-268 over flatten_occurrences,
proj/src/expr.cpp:424-510): assemble_rhs with opt.amvm (baca.cpp:57-76),
i.e. the rows [Dirichlet triangles; Neumann nodes] of
[-V_h, M/2 + K_h; M'/2 - K_h', -D_h] [g_N; g_D] over the device V_Delta, V_kl
and K_Delta H-matrices -- the paper's Table 3 workload -- checked against
the reference's AMVM properties (test_amvm.cpp) and dense algebra on the
oracle's matrices, and the generic machinery against the single-operator
device AMVM."""
import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc

pytestmark = pytest.mark.gpu

E, NU = 1.0, 0.3


def _mesh():
    mesh = hm.Mesh.voxel_cube(4, -1.0, 1.0)
    mesh.label_dirichlet("x1>=1|x2<=-1|x3>=1")
    return mesh


def _system(eps):
    pytest.importorskip("torch")
    mesh = _mesh()
    ops = hm.OperatorSet(mesh, E, NU, b_min=8, eta=1.0, device=0)
    ops.assemble(eps=eps, beta=0.8, lookahead=2)
    return mesh, ops, hm.SaddleSystem(ops, hm.DofLayout(mesh))


def _data(mesh, seed=11):
    m, n = mesh.num_triangles, mesh.num_vertices
    return orc.random_vector(3 * m, seed), orc.random_vector(3 * n, seed + 1)


def _dense_rhs(mesh, gn, gd):
    """rhs_operator from the oracle's dense V_Delta, V_kl, K_Delta and the
    sparse operators (compose_Vh / Kh / Dh, operators.cpp:95-159)."""
    a = mesh.arrays()
    V, T = a["vertices"], a["triangles"]
    m, n = len(T), len(V)
    lam, mu = hm.lame_constants(E, NU)
    vd = orc.Problem.galerkin(V, T, 1, b_min=8, eta=1.0).dense(0)
    vg = orc.Problem.galerkin(V, T, 0, b_min=8, eta=1.0).dense_grid()
    kd = orc.Problem.kdelta(V, T, b_min=8, eta=1.0).dense(0)
    t12, t13, t23 = (orc.sparse_op(V, T, w) for w in range(3))
    mass = orc.sparse_op(V, T, 3)
    Z = np.zeros((m, n))
    Th = np.block([[Z, t12, t13], [-t12, Z, t23], [-t13, -t23, Z]])
    D3 = np.kron(np.eye(3), vd)
    Vh = 0.5 / E * (1 + NU) / (1 - NU) * ((3 - 4 * NU) * D3 + vg)
    Kh = np.kron(np.eye(3), kd) - D3 @ Th + 2 * mu * Vh @ Th
    S = [np.kron(np.eye(3), -t23), np.kron(np.eye(3), t13), np.kron(np.eye(3), t12)]
    Dh = sum(mu * Sk.T @ D3 @ Sk for Sk in S) + 2 * mu * Th.T @ D3 @ Th \
        - 4 * mu * mu * Th.T @ Vh @ Th
    tl = {(0, 1): t12, (0, 2): t13, (1, 2): t23}
    ts = lambda k, l: None if k == l else (1.0 if k < l else -1.0) * tl[(min(k, l), max(k, l))]
    G = np.zeros((3 * n, 3 * n))
    for i in range(3):
        for j in range(3):
            for k in range(3):
                if k not in (i, j):
                    G[i * n:(i + 1) * n, j * n:(j + 1) * n] += ts(k, j).T @ vd @ ts(k, i)
    Dh = Dh + mu * G
    M3 = np.kron(np.eye(3), mass)
    layout = hm.DofLayout(mesh)
    top = -Vh @ gn + 0.5 * M3 @ gd + Kh @ gd
    bottom = 0.5 * M3.T @ gn - Kh.T @ gn - Dh @ gd
    return np.concatenate([top[layout.t_dofs], bottom[layout.u_dofs]])


def test_rhs_without_sweeps_is_the_current_product():
    mesh, ops, sys = _system(1e-3)
    gn, gd = _data(mesh)
    f, rep = hm.assemble_rhs(sys, gn, gd, amvm=True,
                             amvm_cfg=hm.AmvmConfig(max_iterations=0))
    assert (f == sys.rhs(gn, gd)).all()
    assert rep.iterations[0].gamma > 0 and rep.termination == "max_iterations"
    f0, none = hm.assemble_rhs(sys, gn, gd)
    assert none is None and (f0 == f).all()


def test_rhs_estimator_is_the_lookahead_gap():
    """gamma = ||(A_lookahead - A_current) x|| of the composite operator: after
    promoting every block with a tail (no extension) the product moves by
    exactly the estimator's difference vector."""
    mesh, ops, sys = _system(1e-3)
    gn, gd = _data(mesh)
    f, rep = hm.assemble_rhs(sys, gn, gd, amvm=True,
                             amvm_cfg=hm.AmvmConfig(max_iterations=0))
    gamma = rep.iterations[0].gamma
    for h in (ops.vdelta, ops.vkl, ops.kdelta):
        kc, kl, _, _ = h.ranks()
        pairs = [(q, b) for q in range(kc.shape[0]) for b in range(kc.shape[1])
                 if kc[q, b] >= 0 and kl[q, b] > kc[q, b]]
        h.promote(pairs)
    f_look = sys.rhs(gn, gd)
    assert np.linalg.norm(f_look - f) == pytest.approx(gamma, rel=1e-10)


def test_rhs_amvm_converges_to_the_dense_product():
    mesh, ops, sys = _system(1e-2)
    gn, gd = _data(mesh)
    f_dense = _dense_rhs(mesh, gn, gd)
    f0 = sys.rhs(gn, gd)
    theta = 0.7
    f, rep = hm.assemble_rhs(sys, gn, gd, amvm=True,
                             amvm_cfg=hm.AmvmConfig(theta=theta, eps_amvm=1e-7,
                                                    max_iterations=40))
    its = rep.iterations
    assert rep.converged and its[-1].gamma <= 1e-7
    assert sum(it.marked for it in its) > 0
    for it in its[:-1]:
        # Doerfler marking: the unmarked remainder is within (1 - theta) gamma
        # (or every term was taken)
        assert it.gamma_pk <= (1 - theta) * it.gamma * (1 + 1e-9) or it.marked > 0
        assert it.cumulative_pivots <= its[-1].cumulative_pivots
    # e_hat tracks the change of the look-ahead product between sweeps
    assert all(it.e_hat >= 0 for it in its[:-1])
    err0 = np.linalg.norm(f0 - f_dense) / np.linalg.norm(f_dense)
    err = np.linalg.norm(f - f_dense) / np.linalg.norm(f_dense)
    assert err < 0.2 * err0, (err0, err)  # refined blocks: 10x closer here


def test_rhs_amvm_zero_data():
    mesh, ops, sys = _system(1e-2)
    m, n = mesh.num_triangles, mesh.num_vertices
    f, rep = hm.assemble_rhs(sys, np.zeros(3 * m), np.zeros(3 * n), amvm=True)
    assert (f == 0).all() and rep.converged and rep.iterations[0].gamma == 0.0
    assert len(rep.iterations) == 1


def test_single_h_expression_equals_device_amvm():
    """The generic expression machinery on the expression `h` alone gives the
    device AMVM's record (gamma, marked count, cumulative pivots of every
    sweep) bit for bit."""
    mesh = hm.Mesh.ellipsoid(3, 2.0, 1.0, 0.5)
    c = mesh.arrays()["centroids"]
    bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.1 ** 2))
    x = np.tile(bump, 3) + 1e-3 * hm.random_vector(3 * len(c), 3)
    hs = []
    for _ in range(2):
        h = hm.HMatrix.kelvin(mesh, b_min=16, eta=1.0, device=0)
        h.assemble(eps=1e-2, beta=0.8, lookahead=2)
        hs.append(h)
    cfg = hm.AmvmConfig(theta=0.7, eps_amvm=1e-6, max_iterations=6)
    b1, r1 = hs[0].amvm_multiply(x, cfg)
    b2, r2 = hm.amvm_multiply_occurrences([(hs[1], False, 1.0, None, None)], hs[1].matvec,
                                          x, hs[1].rows, hs[1].cols, cfg)
    assert len(r1.iterations) == len(r2.iterations)
    for a, e in zip(r1.iterations, r2.iterations):
        assert (a.gamma, a.marked, a.cumulative_pivots) == (e.gamma, e.marked,
                                                            e.cumulative_pivots)
        assert a.gamma_pk == pytest.approx(e.gamma_pk, rel=1e-13)
    assert np.linalg.norm(b1 - b2) <= 1e-13 * np.linalg.norm(b1)
