"""BPCG / BACA of the reduced all-Dirichlet system V_h t = f on the GPU
H-matrices (proj/src/baca.cpp:104-600), checked with
the reference's own property tests (proj/tests/test_baca.cpp:82-101,
195-271) against dense solves of the oracle's matrices."""
import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc

pytestmark = pytest.mark.gpu
RV = orc.random_vector


def dense_vh(mesh, E, nu, b_min):
    a = mesh.arrays()
    V, T = a["vertices"], a["triangles"]
    vd = orc.Problem.galerkin(V, T, 1, b_min=b_min, eta=1.0).dense(0)
    vg = orc.Problem.galerkin(V, T, 0, b_min=b_min, eta=1.0).dense_grid()
    return 0.5 / E * (1 + nu) / (1 - nu) * ((3 - 4 * nu) * np.kron(np.eye(3), vd) + vg)


@pytest.fixture(scope="module")
def sys2():
    mesh = hm.Mesh.icosphere(2)
    ops = hm.OperatorSet(mesh, 1.0, 0.3, b_min=16, eta=1.0, device=0)
    ops.assemble(eps=1e-3, beta=0.8, lookahead=2)
    return mesh, ops, dense_vh(mesh, 1.0, 0.3, 16)


def test_preconditioner_below_single_layer(sys2):  # test_baca.cpp:82-101
    torch = pytest.importorskip("torch")
    mesh, ops, A = sys2
    prec = hm.VddPreconditioner(ops)
    assert prec.eta > 0
    n = A.shape[0]
    I = torch.eye(n, dtype=torch.float64, device="cuda")
    C = torch.stack([prec.apply(I[j]) for j in range(n)], dim=1).cpu().numpy()
    assert np.linalg.eigvalsh(A - C).min() > 0
    r = torch.tensor(RV(n, 23), device="cuda")
    assert float((prec.apply(prec.solve(r)) - r).norm()) <= 1e-10 * float(r.norm())


def test_doerfler_marking_minimal(sys2):  # test_baca.cpp:229-250
    mesh, ops, A = sys2
    x = RV(A.shape[0], 41)
    ek, terms, _ = hm.estimator_vh(ops, x)
    assert ek > 0
    theta = 0.8
    marked = hm.doerfler_mark(terms, ek, theta)
    acc = sum(terms[i][3] for i in marked)
    assert acc >= theta * theta * ek * ek
    assert acc - terms[marked[-1]][3] < theta * theta * ek * ek
    # greedy: the marked terms are the largest ones
    rest = [terms[i][3] for i in range(len(terms)) if i not in set(marked)]
    assert not rest or min(terms[i][3] for i in marked) >= max(rest)


def test_baca_drives_estimator_below_tolerance():  # test_baca.cpp:195-227
    mesh = hm.Mesh.icosphere(2)
    ops = hm.OperatorSet(mesh, 1.0, 0.3, b_min=16, eta=1.0, device=0)
    ops.assemble(eps=1e-2, beta=0.8, lookahead=2)
    A = dense_vh(mesh, 1.0, 0.3, 16)
    f = A @ RV(A.shape[0], 5)
    cfg = hm.BacaConfig(theta=0.8, alpha=10.0, eps_baca=3e-7, inner_tol0=1e-1)
    x, rep = hm.baca_solve(ops, f, cfg)
    assert rep.converged and rep.iterations[-1].ek <= cfg.eps_baca
    want = np.linalg.solve(A, f)
    assert np.linalg.norm(x - want) <= 1e-3 * np.linalg.norm(want)
    _, _, c_sp = ops.vdelta.partition_info()
    depth = ops.vdelta.tree(0).depth
    bound = np.sqrt(27.0 * c_sp * depth)
    for it in rep.iterations:
        assert it.tail_norm <= bound * it.ek * (1 + 1e-12)  # reliability surrogate
        if cfg.alpha * it.tail_norm > 1e-12 * np.linalg.norm(f):
            assert it.residual <= max(cfg.alpha * it.tail_norm, it.inner_tol) * (1 + 1e-10)
    assert len(rep.iterations) > 1  # the loop refined


def test_reduced_system_solves_single_layer():  # test_baca.cpp:252-271
    mesh = hm.Mesh.icosphere(1)
    ops = hm.OperatorSet(mesh, 1.0, 0.3, b_min=8, eta=1.0, device=0)
    ops.assemble(eps=1e-4, beta=0.8, lookahead=2)
    f = RV(3 * mesh.num_triangles, 9)
    x, rep = hm.baca_solve(ops, f, hm.BacaConfig(eps_baca=1e-10))
    assert rep.converged
    assert np.linalg.norm(ops.vh(x) - f) <= 1e-8 * np.linalg.norm(f)
