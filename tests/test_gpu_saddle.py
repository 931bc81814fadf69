"""The mixed Lame saddle system on the GPU H-matrices (
assemble_saddle / assemble_rhs / bpcg_solve, proj/src/baca.cpp:12-76,
227-399) with the reference's BPCG tests (proj/tests/test_baca.cpp:50-153)
on the cube with the experiments' labelling, against dense algebra on the
oracle's matrices."""
import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc
from tests.test_gpu_interior import kelvin_traction

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fx():
    torch = pytest.importorskip("torch")
    mesh = hm.Mesh.voxel_cube(4, -1.0, 1.0)
    mesh.label_dirichlet("x1>=1|x2<=-1|x3>=1")  # make_cube_mesh (oracles.cpp:113-119)
    a = mesh.arrays()
    V, T, Cc, N = a["vertices"], a["triangles"], a["centroids"], a["normals"]
    m, n = len(T), len(V)
    E, nu = 1.0, 0.3
    ops = hm.OperatorSet(mesh, E, nu, b_min=8, eta=1.0, device=0)
    ops.assemble(eps=1e-8, beta=0.8)
    layout = hm.DofLayout(mesh)
    sys = hm.SaddleSystem(ops, layout)
    # dense truth from the oracle's matrices (compose_Vh / Kh / Dh)
    lam, mu = hm.lame_constants(E, nu)
    vd = orc.Problem.galerkin(V, T, 1, b_min=8, eta=1.0).dense(0)
    vg = orc.Problem.galerkin(V, T, 0, b_min=8, eta=1.0).dense_grid()
    kd = orc.Problem.kdelta(V, T, b_min=8, eta=1.0).dense(0)
    t12, t13, t23 = (orc.sparse_op(V, T, w) for w in range(3))
    mass = orc.sparse_op(V, T, 3)
    Z = np.zeros((m, n))
    Th = np.block([[Z, t12, t13], [-t12, Z, t23], [-t13, -t23, Z]])
    D3 = np.kron(np.eye(3), vd)
    Vh = 0.5 / E * (1 + nu) / (1 - nu) * ((3 - 4 * nu) * D3 + vg)
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
    td, ud = layout.t_dofs, layout.u_dofs
    A = np.block([[Vh[np.ix_(td, td)], -Kh[np.ix_(td, ud)]],
                  [Kh[np.ix_(td, ud)].T, Dh[np.ix_(ud, ud)]]])
    # manufactured data (oracles.cpp:401-413): u = S(x - p) a, p outside
    p = np.array([5.0, 5.0, 5.0])
    av = np.ones(3) / np.sqrt(3.0)
    g_n = np.zeros(3 * m)
    g_d = np.zeros(3 * n)
    for t in range(m):
        g_n[[t, m + t, 2 * m + t]] = kelvin_traction(Cc[t] - p, N[t]) @ av
    for v in range(n):
        g_d[[v, n + v, 2 * n + v]] = orc.kelvin_tensor(V[v] - p) @ av
    for t in layout.dirichlet_triangle_ids:
        g_n[[t, m + t, 2 * m + t]] = 0.0
    for v in layout.neumann_interior_nodes:
        g_d[[v, n + v, 2 * n + v]] = 0.0
    M3 = np.kron(np.eye(3), mass)
    full = np.block([[-Vh, 0.5 * M3 + Kh], [0.5 * M3.T - Kh.T, -Dh]])
    rows = np.concatenate([td, 3 * m + ud])
    f_dense = full[rows] @ np.concatenate([g_n, g_d])
    # the current (H-matrix) system, densified through the device operator
    I = torch.eye(sys.dim, dtype=torch.float64, device="cuda")
    A_cur = torch.stack([sys.a(I[j]) for j in range(sys.dim)], dim=1).cpu().numpy()
    return dict(sys=sys, A=A, A_cur=A_cur, f=f_dense, g_n=g_n, g_d=g_d, prec=sys.preconditioner())


def test_rhs_agrees_with_dense(fx):  # test_baca.cpp:50-72
    sys = fx["sys"]
    f = sys.rhs(fx["g_n"], fx["g_d"])
    assert np.linalg.norm(f - fx["f"]) <= 1e-6 * np.linalg.norm(fx["f"])
    assert np.linalg.norm(sys.rhs(0 * fx["g_n"], 0 * fx["g_d"])) == 0.0
    assert np.abs(fx["A_cur"] - fx["A"]).max() <= 1e-6 * np.abs(fx["A"]).max()


def test_bpcg_zero_rhs(fx):  # test_baca.cpp:108-115
    x, st = hm.bpcg_solve(fx["sys"], fx["prec"], np.zeros(fx["sys"].dim), 1e-10)
    assert np.linalg.norm(x) == 0.0 and st.iterations == 0


def test_bpcg_matches_direct_solve(fx):  # test_baca.cpp:117-128
    f = fx["f"]
    want = np.linalg.solve(fx["A_cur"], f)
    x, st = hm.bpcg_solve(fx["sys"], fx["prec"], f, 1e-10 * np.linalg.norm(f))
    assert st.converged and not st.used_fallback
    assert np.linalg.norm(x - want) <= 1e-7 * np.linalg.norm(want)


def test_minres_path_matches(fx):  # test_baca.cpp:130-141
    f = fx["f"]
    want = np.linalg.solve(fx["A_cur"], f)
    x, st = hm.bpcg_solve(fx["sys"], fx["prec"], f, 1e-9 * np.linalg.norm(f), use_bpcg=False)
    assert st.converged
    assert np.linalg.norm(x - want) <= 1e-6 * np.linalg.norm(want)


def test_warm_starts_beat_cold(fx):  # test_baca.cpp:143-152
    f = fx["f"]
    nf = np.linalg.norm(f)
    x1, _ = hm.bpcg_solve(fx["sys"], fx["prec"], f, 1e-1 * nf)
    _, warm = hm.bpcg_solve(fx["sys"], fx["prec"], f, 1e-3 * nf, x1)
    _, cold = hm.bpcg_solve(fx["sys"], fx["prec"], f, 1e-3 * nf)
    assert warm.iterations < cold.iterations


@pytest.fixture(scope="module")
def coarse():
    """BacaFixture-like coarse system (test_baca.cpp:11-48): full-mode ACA at
    a loose tolerance so that the look-ahead tails are large."""
    mesh = hm.Mesh.voxel_cube(4, -1.0, 1.0)
    mesh.label_dirichlet("x1>=1|x2<=-1|x3>=1")
    ops = hm.OperatorSet(mesh, 1.0, 0.3, b_min=8, eta=1.0, device=0)
    ops.assemble(eps=1e-2, beta=0.8, lookahead=2)
    return mesh, ops, hm.SaddleSystem(ops, hm.DofLayout(mesh))


def test_estimator_aggregates_family_terms(coarse):  # test_baca.cpp:155-178
    torch = pytest.importorskip("torch")
    mesh, ops, sys = coarse
    x = orc.random_vector(sys.dim, 31)
    ek, terms, diff = hm.SaddleEstimator(sys).estimate(x)
    assert ek == pytest.approx(np.sqrt(sum(t[4] for t in terms)), rel=1e-12)
    xd = torch.tensor(x, device="cuda")
    cur = sys.a(xd).cpu().numpy()
    ops.mode = hm.Mode.Lookahead
    try:
        look = sys.a(xd).cpu().numpy()
    finally:
        ops.mode = hm.Mode.Current
    want = look - cur
    assert np.linalg.norm(diff - want) <= 1e-10 * (np.linalg.norm(want) + 1.0)
    assert {t[0] for t in terms} == {"V", "K", "D"}  # all three families on a mixed mesh


def test_baca_saddle_drives_estimator_below_tolerance(coarse, fx):  # test_baca.cpp:195-227
    mesh, ops, sys = coarse
    f = sys.rhs(fx["g_n"], fx["g_d"])
    cfg = hm.BacaConfig(theta=0.8, alpha=10.0, eps_baca=3e-7, inner_tol0=1e-1)
    x, rep = hm.baca_solve_saddle(sys, f, cfg)
    assert rep.converged and rep.iterations[-1]["ek"] <= cfg.eps_baca
    want = np.linalg.solve(fx["A"], fx["f"])
    assert np.linalg.norm(x - want) <= 1e-3 * np.linalg.norm(want)
    for it in rep.iterations:
        if cfg.alpha * it["tail_norm"] > 1e-12 * np.linalg.norm(f):
            assert it["residual"] <= max(cfg.alpha * it["tail_norm"], it["inner_tol"]) * (1 + 1e-10)
        ph = it["phases"]
        assert all(ph[i - 1] < ph[i] for i in range(1, len(ph)))  # D before K before V
        if it["marked_d"] > 0:
            assert ph and ph[0] == 1
    assert len(rep.iterations) > 1
