"""Oracle H-matrix and AMVM property tests: the reference's
test_hmatrix.cpp / test_amvm.cpp cases on the CentroidKernelOracle fixture
(Newton kernel on cube(4) centroids, diagonal 2.0, b_min 10, beta 0.8)."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import centroid_points_and_boxes, cube_mesh

RV = orc.random_vector


@pytest.fixture(scope="module")
def fixture_pts():
    return centroid_points_and_boxes(cube_mesh(4))


def newton(fixture_pts):
    pts, boxes = fixture_pts
    return orc.Problem.newton(pts, boxes, diag=2.0, b_min=10, eta=0.8)


def test_full_mode_approximates_dense(fixture_pts):  # test_hmatrix.cpp:76-90
    p = newton(fixture_pts)
    p.assemble(eps=1e-6)
    a = p.dense(0)
    x = RV(p.n, 17)
    y = p.matvec(x)
    assert np.linalg.norm(y - a @ x) <= 1e-5 * np.linalg.norm(a @ x)
    yt = p.matvec_transposed(x)
    assert np.linalg.norm(yt - a.T @ x) <= 1e-5 * np.linalg.norm(a.T @ x)


def test_coarse_mode_caps_ranks(fixture_pts):  # test_hmatrix.cpp:92-112
    p = newton(fixture_pts)
    p.assemble(initial_rank=2, lookahead=2)
    kc, kl, co, _ = p.ranks()
    adm = kc[0] >= 0
    assert adm.any()
    assert (kc[0][adm] <= 2).all() and (kl[0][adm] <= 4).all()


def test_lookahead_dominates(fixture_pts):  # test_hmatrix.cpp:114-140
    p = newton(fixture_pts)
    p.assemble(initial_rank=3, lookahead=2)
    a = p.dense(0)
    nodes, _, perm, _ = p.tree()
    kc, kl, co, _ = p.ranks()
    for b, (rn, cn, adm, _) in enumerate(p.blocks()):
        if not adm:
            continue
        r = perm[nodes[rn, 0]:nodes[rn, 1]]
        c = perm[nodes[cn, 0]:nodes[cn, 1]]
        ab = a[np.ix_(r, c)]
        f = p.factor(0, b)
        lo, hi = kc[0, b], kl[0, b]
        e_lo = np.linalg.norm(ab - f["U"][:, :lo] @ f["V"][:, :lo].T)
        e_hi = np.linalg.norm(ab - f["U"][:, :hi] @ f["V"][:, :hi].T)
        assert e_hi <= e_lo * (1 + 1e-12)
        if co[0, b] < len(r):
            assert e_hi < e_lo


def test_storage_kat():  # test_hmatrix.cpp:288-301
    pts = np.array([[i, 0.0, 0.0] for i in range(100)])
    p = orc.Problem.dense_matrix(np.ones((100, 100)), pts, pts, b_min=128, eta=0.8)
    p.assemble()
    assert p.storage()["mb_current"] == pytest.approx(0.0762939453125)


def test_permutation_correctness():  # test_hmatrix.cpp:142-164
    n = 60
    pts = RV(3 * n, 77).reshape(n, 3)
    d = pts[:, None, :] - pts[None, :, :]
    r = np.sqrt((d[..., 0] ** 2 + d[..., 1] ** 2) + d[..., 2] ** 2)
    base = np.where(np.eye(n, dtype=bool), 1.5, 1.0 / np.where(r == 0, 1, r))
    p = orc.Problem.dense_matrix(base, pts, pts, b_min=8, eta=1.2)
    p.assemble(eps=1e-10)
    y = p.matvec(np.eye(n)[:, 5])
    assert np.linalg.norm(y - base[:, 5]) <= 1e-9 * np.linalg.norm(base)


# ---- test_amvm.cpp (plain H-leaf operator instead of the sparse sandwich)
def test_gamma_matches_dense_gap(fixture_pts):  # test_amvm.cpp:74-103
    p = newton(fixture_pts)
    p.assemble(initial_rank=2, lookahead=2)
    g, diff, terms = p.gamma(np.zeros(p.n))
    assert g == 0.0 and all(t["norm_sq"] == 0.0 for t in terms)
    x = RV(p.n, 3)
    g, diff, terms = p.gamma(x)
    want = p.matvec(x, 1) - p.matvec(x, 0)
    assert np.linalg.norm(diff - want) <= 1e-12 * (np.linalg.norm(want) + 1)
    assert g == pytest.approx(np.linalg.norm(want), rel=1e-10)
    acc = np.zeros(p.n)
    for t in terms:
        acc[t["idx"]] += t["val"]
        assert np.sum(t["val"] ** 2) == pytest.approx(t["norm_sq"])
    assert np.linalg.norm(acc - diff) <= 1e-13 * (np.linalg.norm(want) + 1)


def test_marking_theta_condition(fixture_pts):  # test_amvm.cpp:105-132
    p = newton(fixture_pts)
    p.assemble(initial_rank=2, lookahead=2)
    x = RV(p.n, 5)
    g, diff, terms = p.gamma(x)
    c_sp = p.partition_info()[2]
    for theta in (0.3, 0.7, 0.9):
        marked, gpk = p.mark(theta, c_sp, p.n, p.n, len(terms))
        assert len(marked) > 0
        assert gpk <= (1 - theta) * g * (1 + 1e-12)
        res = diff.copy()
        for t in marked:
            res[terms[t]["idx"]] -= terms[t]["val"]
        assert np.linalg.norm(res) == pytest.approx(gpk, rel=1e-12)
    marked, _ = p.mark(0.999999, c_sp, p.n, p.n, len(terms))
    assert len(marked) == sum(1 for t in terms if t["norm_sq"] > 0)


def test_amvm_refines_to_tolerance(fixture_pts):  # test_amvm.cpp:162-193
    p = newton(fixture_pts)
    p.assemble(initial_rank=2, lookahead=2)
    x = RV(p.n, 11)
    b_true = p.dense(0) @ x
    eps = 1e-7 * np.linalg.norm(b_true)
    b, it, conv = p.amvm(x, theta=0.7, eps_amvm=eps, max_iterations=100)
    assert conv and it[-1, 1] <= eps
    assert np.linalg.norm(b - b_true) <= 50 * eps
    for k in range(len(it) - 1):
        assert it[k, 2] <= 0.3 * it[k, 1] * (1 + 1e-12) and it[k, 3] > 0
        g0, g1, eh = it[k, 1], it[k + 1, 1], it[k, 6]
        assert eh >= 0
        assert g1 * g1 <= 0.5 * g0 * g0 + (1 / 0.82) * eh * eh + 1e-18


def test_amvm_zero_and_exhausted(fixture_pts):  # test_amvm.cpp:195-215
    p = newton(fixture_pts)
    p.assemble(initial_rank=2, lookahead=2)
    piv = p.storage()["total_pivots"]
    b, it, conv = p.amvm(np.zeros(p.n))
    assert np.linalg.norm(b) == 0 and conv and len(it) == 1 and it[0, 3] == 0
    assert p.storage()["total_pivots"] == piv
    p2 = newton(fixture_pts)
    p2.assemble(initial_rank=1000, lookahead=2)
    b, it, conv = p2.amvm(RV(p2.n, 13))
    assert conv and len(it) == 1 and it[0, 1] == 0.0


def test_amvm_deterministic(fixture_pts):  # test_amvm.cpp:217-232
    x = RV(192, 17)
    runs = []
    for _ in range(2):
        p = newton(fixture_pts)
        p.assemble(initial_rank=2, lookahead=2)
        runs.append(p.amvm(x, eps_amvm=1e-6))
    (b1, i1, _), (b2, i2, _) = runs
    assert (b1 == b2).all() and (i1[:, :5] == i2[:, :5]).all()
