"""Pins the oracle's Galerkin pair quadrature and V_Delta / V_kl entries
 with the reference's own known-answer and property
tests (proj/tests/test_quadrature.cpp:83-191, test_kernels.cpp:132-254),
checked against the reference's test-side oracles restated in
tests/galerkin_ref.py."""
import numpy as np
import pytest

from oracle import oracle as orc
from tests import galerkin_ref as ref
from tests.helpers import cube_mesh, doctest_approx

T0 = np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]])


def test_pair_rule_weights_cover_pair_measure():  # test_quadrature.cpp:83-90
    for c in range(4):
        w = orc.pair_rule(c, 4)[4]
        assert doctest_approx(w.sum(), 0.25, 1e-12)


def test_pair_rule_sizes():  # quadrature.cpp:296-313
    assert len(orc.pair_rule(0, 2)[4]) == 9
    assert len(orc.pair_rule(0, 5)[4]) == 49
    assert len(orc.pair_rule(1, 7)[4]) == 2 * 7 ** 4
    assert len(orc.pair_rule(2, 7)[4]) == 5 * 7 ** 4
    assert len(orc.pair_rule(3, 9)[4]) == 6 * 9 ** 4


def test_classify_pair():  # test_quadrature.cpp:92-115
    c, rt, rs, pa, pb = orc.classify_pair([0, 1, 2], [0, 1, 2])
    assert c == 3
    c, rt, rs, pa, pb = orc.classify_pair([0, 1, 2], [2, 1, 3])
    assert c == 2
    a, b = [0, 1, 2], [2, 1, 3]
    assert a[pa[0]] == b[pb[0]] and a[pa[1]] == b[pb[1]]
    c, rt, rs, pa, pb = orc.classify_pair([0, 1, 2], [3, 4, 2])
    assert c == 1
    assert [0, 1, 2][pa[0]] == [3, 4, 2][pb[0]]
    assert orc.classify_pair([0, 1, 2], [3, 4, 5])[0] == 0


def test_singular_transforms_integrate_smooth_kernels():  # test_quadrature.cpp:142-151
    want = ref.bruteforce_pair_integral(T0, T0, ref.smooth_kernel, 3)
    for c in (3, 2, 1):
        got = ref.integrate_with_rule(T0, T0, c, 6, ref.smooth_kernel)
        assert doctest_approx(got, want, 1e-8)


@pytest.fixture(scope="module")
def coincident_want():
    return 4.0 * np.pi * ref.vdelta_singular_oracle(T0, T0)


def test_coincident_newton_integral(coincident_want):  # test_quadrature.cpp:153-164
    got6 = ref.integrate_with_rule(T0, T0, 3, 6, ref.newton_kernel)
    assert doctest_approx(got6, coincident_want, 1e-5)
    got8 = ref.integrate_with_rule(T0, T0, 3, 8, ref.newton_kernel)
    assert doctest_approx(got8, coincident_want, 2e-7)


def test_edge_adjacent_newton_integral():  # test_quadrature.cpp:166-181
    ty = np.array([[1.0, 0, 0], [0, 0, 0], [0.3, -0.5, 0.4]])
    c, rt, rs, pa, pb = orc.classify_pair([0, 1, 2], [1, 0, 3])
    assert c == 2
    got = ref.integrate_with_rule(T0[pa], ty[pb], 2, 5, ref.newton_kernel)
    want = 4.0 * np.pi * ref.vdelta_singular_oracle(T0, ty)
    assert doctest_approx(got, want, 1e-6)


def test_vertex_adjacent_newton_integral():  # test_quadrature.cpp:183-191
    ty = np.array([[0.0, 0, 0], [-1, 0.2, 0.1], [-0.4, -0.8, 0.3]])
    got = ref.integrate_with_rule(T0, ty, 1, 5, ref.newton_kernel)
    want = 4.0 * np.pi * ref.vdelta_singular_oracle(T0, ty)
    assert doctest_approx(got, want, 1e-6)


@pytest.fixture(scope="module")
def cube3():
    m = cube_mesh(3)
    a = m.arrays()
    grid = orc.Problem.galerkin(a["vertices"], a["triangles"], which=0, b_min=8, eta=1.0)
    vd = orc.Problem.galerkin(a["vertices"], a["triangles"], which=1, b_min=8, eta=1.0)
    return a, grid, vd


def test_separated_entries_match_subdivision(cube3):  # test_kernels.cpp:132-171
    a, grid, vd = cube3
    V, T = a["vertices"], a["triangles"]
    pairs = []
    for j in range(1, len(T), 7):
        if orc.classify_pair(T[0], T[j])[0] == 0:
            pairs.append(j)
        if len(pairs) == 10:
            break
    assert len(pairs) == 10
    for j in pairs:
        want = ref.bruteforce_pair_integral(V[T[0]], V[T[j]], ref.newton_kernel) / (4 * np.pi)
        assert doctest_approx(vd.entry(0, 0, j), want, 1e-6)
        k01 = lambda X, Y: (X - Y)[..., 0] * (X - Y)[..., 1] / np.linalg.norm(X - Y, axis=-1) ** 3
        want12 = ref.bruteforce_pair_integral(V[T[0]], V[T[j]], k01) / (4 * np.pi)
        if abs(want12) > 1e-12:
            assert doctest_approx(grid.entry(1, 0, j), want12, 1e-6)


def test_touching_vdelta_entries_match_analytic(cube3):  # test_kernels.cpp:207-233
    a, grid, vd = cube3
    V, T = a["vertices"], a["triangles"]
    assert doctest_approx(vd.entry(0, 0, 0), ref.vdelta_singular_oracle(V[T[0]], V[T[0]]),
                          1e-5)
    edge_j = vertex_j = -1
    for j in range(1, len(T)):
        c = orc.classify_pair(T[0], T[j])[0]
        if c == 2 and edge_j < 0:
            edge_j = j
        if c == 1 and vertex_j < 0:
            vertex_j = j
    assert edge_j > 0 and vertex_j > 0
    assert doctest_approx(vd.entry(0, 0, edge_j),
                          ref.vdelta_singular_oracle(V[T[0]], V[T[edge_j]]), 1e-5)
    assert doctest_approx(vd.entry(0, 0, vertex_j),
                          ref.vdelta_singular_oracle(V[T[0]], V[T[vertex_j]]), 1e-6)


def test_exact_symmetry(cube3):  # test_kernels.cpp:235-240
    a, grid, vd = cube3
    assert vd.entry(0, 3, 11) == vd.entry(0, 11, 3)
    assert grid.entry(2, 5, 9) == grid.entry(2, 9, 5)  # vkl(0,2,5,9) == vkl(2,0,9,5)


def test_canonical_order_matches_literal(cube3):
    a, grid, vd = cube3
    rng = np.random.default_rng(0)
    nt = len(a["triangles"])
    for _ in range(40):
        i, j = (int(v) for v in rng.integers(0, nt, 2))
        x, y = vd.entry(0, i, j), vd.entry_literal(0, i, j)
        assert abs(x - y) <= 1e-13 * abs(y)
        for c in range(6):
            x, y = grid.entry(c, i, j), grid.entry_literal(c, i, j)
            assert abs(x - y) <= 1e-13 * max(abs(y), 1e-3 * abs(vd.entry(0, i, j)))


def test_galerkin_hmatrix_vs_dense(cube3):  # test_hmatrix.cpp:76-90 on V_Delta / V_kl
    a, grid, vd = cube3
    eps = 1e-6
    for p in (grid, vd):
        p.assemble(eps=eps, beta=0.8)
        x = orc.random_vector(p.rows, 5)
        y = p.matvec(x)
        yd = p.dense_grid() @ x
        assert np.linalg.norm(y - yd) <= 10 * eps * np.linalg.norm(yd)


# ---------------------------------------------------------------------------
# K_Delta (triangles x nodes, kernels.cpp:151-167)
@pytest.fixture(scope="module")
def kd3():
    m = cube_mesh(3)
    a = m.arrays()
    return a, orc.Problem.kdelta(a["vertices"], a["triangles"], b_min=8, eta=1.0)


def _vertex_triangles(T, nv):
    vt = [[] for _ in range(nv)]
    for t, tri in enumerate(T):
        for v in tri:
            vt[v].append(t)
    return vt


def _kdelta_bruteforce(V, T, i, node, vt):  # test_kernels.cpp:103-118
    acc = 0.0
    for tau in vt[node]:
        if tau == i:
            continue
        local = list(T[tau]).index(node)
        c = V[T[tau]]
        e0, e1 = c[1] - c[0], c[2] - c[0]
        nrm = np.cross(e0, e1)
        nrm = nrm / np.linalg.norm(nrm)
        a00, a01, a11 = e0 @ e0, e0 @ e1, e1 @ e1
        det = a00 * a11 - a01 * a01

        def k(X, Y, c=c, e0=e0, e1=e1, nrm=nrm, local=local):
            d = X - Y
            r = np.linalg.norm(d, axis=-1)
            rel_ = Y - c[0]
            b1 = (a11 * (rel_ @ e0) - a01 * (rel_ @ e1)) / det
            b2 = (a00 * (rel_ @ e1) - a01 * (rel_ @ e0)) / det
            bary = [1.0 - b1 - b2, b1, b2][local]
            return (d @ nrm) / (4.0 * np.pi * r ** 3) * bary

        acc += ref.bruteforce_pair_integral(V[T[i]], c, k, 8)
    return acc


def test_kdelta_separated_matches_subdivision(kd3):  # test_kernels.cpp:150-170
    a, kd = kd3
    V, T = a["vertices"], a["triangles"]
    vt = _vertex_triangles(T, len(V))
    checked = 0
    for v in range(len(V)):
        if checked >= 4:
            break
        if any(t == 0 or orc.classify_pair(T[0], T[t])[0] != 0 for t in vt[v]):
            continue
        want = _kdelta_bruteforce(V, T, 0, v, vt)
        if abs(want) < 1e-12:
            continue
        assert doctest_approx(kd.entry(0, 0, v), want, 1e-6)
        checked += 1
    assert checked >= 3


def test_kdelta_vanishes_on_coplanar_pairs(kd3):  # test_kernels.cpp:242-254
    a, kd = kd3
    V, T, N, Cc = a["vertices"], a["triangles"], a["normals"], a["centroids"]
    vt = _vertex_triangles(T, len(V))
    for t in range(len(T)):
        node = T[t][0]
        if all(np.linalg.norm(N[u] - N[t]) < 1e-14 and abs((Cc[u] - Cc[t]) @ N[t]) < 1e-14
               for u in vt[node]):
            assert abs(kd.entry(0, t, node)) < 1e-14
            return
    pytest.fail("no coplanar witness found")


def test_kdelta_canonical_matches_literal_and_hmatrix(kd3):
    a, kd = kd3
    rng = np.random.default_rng(1)
    D = kd.dense(0)
    scale = np.abs(D).max()
    for _ in range(40):
        i = int(rng.integers(0, D.shape[0]))
        j = int(rng.integers(0, D.shape[1]))
        assert abs(kd.entry(0, i, j) - kd.entry_literal(0, i, j)) <= 1e-13 * scale
    eps = 1e-6
    kd.assemble(eps=eps, beta=0.8)
    x = orc.random_vector(D.shape[1], 4)
    y = kd.matvec(x)
    assert np.linalg.norm(y - D @ x) <= 10 * eps * np.linalg.norm(D @ x)
