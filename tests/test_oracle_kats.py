"""Pins the CPU oracle against the reference's own known-answer tests and
property tests.  The reference ships no stored golden
vectors; these are its doctest cases restated (file:line cited per test)."""
import math

import numpy as np
import pytest

from oracle import oracle as orc
from tests.helpers import separated_kernel_matrix

RV = orc.random_vector


# ---- test_kernels.cpp ------------------------------------------------------
def test_lame_constants_kat():  # test_kernels.cpp:7-21
    lam, mu = orc.lame_constants(1.0, 0.3)
    assert lam == pytest.approx(0.576923076923, rel=1e-9)
    assert mu == pytest.approx(0.384615384615, rel=1e-9)
    lam, mu = orc.lame_constants(2.0, 0.25)
    assert lam == pytest.approx(0.8) and mu == pytest.approx(0.8)
    for E, nu in [(1.0, 0.0), (1.0, 0.5), (-1.0, 0.3)]:
        with pytest.raises(orc.OracleError):
            orc.lame_constants(E, nu)


def test_kelvin_closed_form_kat():  # test_kernels.cpp:23-40
    nu, r = 0.3, 2.5
    s = orc.kelvin_tensor([r, 0, 0], 1.0, nu)
    c = (1.0 + nu) / (8.0 * math.pi * (1.0 - nu))
    assert s[0, 0] == pytest.approx(c * ((3 - 4 * nu) + 1.0) / r)
    assert s[1, 1] == pytest.approx(c * (3 - 4 * nu) / r)
    assert s[2, 2] == pytest.approx(c * (3 - 4 * nu) / r)
    assert abs(s[0, 1]) < 1e-15 and abs(s[1, 2]) < 1e-15
    x = RV(3, 5)
    p = np.array([x[0] + 2.0, x[1], x[2]])
    a = orc.kelvin_tensor(p)
    assert np.linalg.norm(a - orc.kelvin_tensor(-p)) < 1e-15
    assert np.linalg.norm(a - a.T) < 1e-15
    with pytest.raises(orc.OracleError):
        orc.kelvin_tensor([0, 0, 0])


def test_canonical_entry_matches_literal():
    """The canonical evaluation order of colloc_single (shared bit for bit
    with the device) agrees with the literal kelvin_tensor form of
    kernels.cpp:176-187 to rounding."""
    v, t = orc.voxel_surface(4, -1.0, 1.0)
    prob = orc.Problem.kelvin(v, t, b_min=8, eta=1.0)
    rng = np.random.default_rng(1)
    for _ in range(300):
        i, j = rng.integers(0, len(t), 2)
        if i == j:
            continue
        for comp in range(6):
            a = prob.entry(comp, i, j)
            b = prob.entry_literal(comp, i, j)
            scale = abs(prob.entry(0, i, j))
            assert abs(a - b) <= 1e-14 * scale, (i, j, comp)


# ---- test_quadrature.cpp ---------------------------------------------------
def _monomial(a, b):
    return math.factorial(a) * math.factorial(b) / math.factorial(a + b + 2)


@pytest.mark.parametrize("order", range(1, 7))
def test_gauss_rule_exact(order):  # test_quadrature.cpp:29-43
    pa, pb, w = orc.gauss_rule(order)
    assert (w > 0).all()
    assert w.sum() == pytest.approx(0.5, rel=1e-14)
    for a in range(order + 1):
        for b in range(order + 1 - a):
            got = float(np.sum(w * pa ** a * pb ** b))
            assert abs(got - _monomial(a, b)) < 1e-13, (order, a, b)


def test_gauss_rule_small_orders():  # test_quadrature.cpp:45-69
    pa, pb, w = orc.gauss_rule(1)
    assert len(w) == 1 and pa[0] == pytest.approx(1 / 3) and pb[0] == pytest.approx(1 / 3)
    assert w[0] == pytest.approx(0.5)
    pa, pb, w = orc.gauss_rule(2)
    assert len(w) == 3 and w.sum() == pytest.approx(0.5)
    assert float(np.sum(w * pa) + np.sum(w * pb)) == pytest.approx(1 / 3, rel=1e-14)
    assert [len(orc.gauss_rule(o)[2]) for o in range(1, 7)] == [1, 3, 6, 6, 7, 12]
    for bad in (0, 7, -2):
        with pytest.raises(orc.OracleError):
            orc.gauss_rule(bad)


def test_gauss_legendre_01():  # test_quadrature.cpp:71-81
    for n in range(1, 11):
        x, w = orc.gauss_legendre_01(n)
        for p in range(2 * n):
            assert abs(float(np.sum(w * x ** p)) - 1.0 / (p + 1)) < 1e-13


# ---- test_mesh.cpp (cube KATs through the voxel generator) -----------------
def test_cube9_mesh_kat():  # test_mesh.cpp:22-39
    v, t = orc.voxel_surface(9, -1.0, 1.0)
    assert len(v) == 488 and len(t) == 972
    g = orc.mesh_geometry(v, t)
    assert g["areas"].sum() == pytest.approx(24.0, rel=1e-12)
    assert (np.einsum("ij,ij->i", g["normals"], g["centroids"]) > 0).all()


# ---- builder-defined self term vs the analytic flat-triangle potential -----
def _analytic_potential(p, tri):
    """analytic_triangle_potential (proj/tests/oracles.cpp:209-232), numpy."""
    nrm = np.cross(tri[1] - tri[0], tri[2] - tri[0])
    nrm /= np.linalg.norm(nrm)
    d = nrm @ (p - tri[0])
    proj = p - d * nrm
    acc = 0.0
    for e in range(3):
        a, b = tri[e], tri[(e + 1) % 3]
        s_hat = (b - a) / np.linalg.norm(b - a)
        m_hat = np.cross(s_hat, nrm)
        t = (a - proj) @ m_hat
        s1, s2 = (a - proj) @ s_hat, (b - proj) @ s_hat
        r1, r2 = np.linalg.norm(p - a), np.linalg.norm(p - b)
        r0sq = t * t + d * d
        if r1 + s1 > 0 and r2 + s2 > 0:
            acc += t * math.log((r2 + s2) / (r1 + s1))
        ad = abs(d)
        acc -= ad * (math.atan2(t * s2, r0sq + ad * r2) - math.atan2(t * s1, r0sq + ad * r1))
    return acc


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5])
def test_self_term_matches_analytic_potential(seed):
    tri = RV(9, seed).reshape(3, 3) * np.array([1.0, 0.7, 0.3])
    p = tri.mean(axis=0)
    got = orc.self_term_i1(tri, p)
    want = _analytic_potential(p, tri)
    assert got == pytest.approx(want, rel=1e-13)


def test_self_term_matches_fine_quadrature():
    """Every component of the closed-form self term against brute-force
    subdivision quadrature (the reference's test strategy for singular
    integrals, oracles.cpp:141-207) on a right triangle."""
    v = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    p = v.mean(axis=0)
    # polar integration about p with many Gauss-Legendre points per edge
    xg, wg = np.polynomial.legendre.leggauss(400)
    irr = np.zeros((3, 3))
    for e in range(3):
        a, b = v[e], v[(e + 1) % 3]
        for s, w in zip(0.5 * (xg + 1), 0.5 * wg):
            q = a + s * (b - a)
            # sub-triangle (p, a, b): area element via the edge parameter
            r = q - p
            L = np.linalg.norm(r)
            h = np.linalg.norm(np.cross(b - a, r)) / np.linalg.norm(b - a)
            dtheta = np.linalg.norm(b - a) * h / (L * L)
            e_hat = r / L
            irr += w * dtheta * L * np.outer(e_hat, e_hat)
    prob = orc.Problem.kelvin(np.vstack([v, [[0, 0, -1.0]]]),
                              np.array([[0, 1, 2], [0, 3, 1], [1, 3, 2], [0, 2, 3]], np.int32),
                              E=1.0, nu=0.3, b_min=1, eta=1.0)
    c = 1.3 / (8 * math.pi * 0.7)
    i1 = np.trace(irr)
    for k, (r, cc) in enumerate([(0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2)]):
        want = c * ((1.8 * i1 if r == cc else 0.0) + irr[r, cc])
        assert prob.entry(k, 0, 0) == pytest.approx(want, rel=1e-9, abs=1e-12)


# ---- test_cluster.cpp ------------------------------------------------------
def _point_problem(pts, b_min, eta=0.8):
    return orc.Problem.newton(np.asarray(pts, dtype=float), b_min=b_min, eta=eta)


def test_single_point_tree():  # test_cluster.cpp:59-64
    nodes, _, _, depth = _point_problem([[1, 2, 3]], 4).tree()
    assert len(nodes) == 1 and depth == 0 and nodes[0, 2] < 0


def test_collinear_points_split_evenly():  # test_cluster.cpp:66-81
    pts = [[i, 0, 0] for i in range(16)]
    nodes, _, perm, depth = _point_problem(pts, 4).tree()
    leaves = nodes[nodes[:, 2] < 0]
    assert len(leaves) == 4 and (leaves[:, 1] - leaves[:, 0] == 4).all()
    assert depth == 2 and (perm == np.arange(16)).all()


def test_admissibility_kat():  # test_cluster.cpp:83-103
    a = [0, 0, 0, 1, 1, 1]
    assert not orc.admissible(a, a, 0.8)
    assert orc.admissible(a, [11, 0, 0, 12, 1, 1], 0.8)
    assert not orc.admissible(a, [3, 0, 0, 4, 1, 1], 0.8)
    with pytest.raises(orc.OracleError):
        orc.admissible(a, [3, 0, 0, 4, 1, 1], 0.0)


def test_small_partitions_kat():  # test_cluster.cpp:105-125, 161-169
    p = _point_problem([[0, 0, 0], [1, 0, 0]], 4)
    assert p.partition_info()[0] == 1 and p.blocks()[0, 2] == 0 and p.partition_info()[2] == 1
    pts = [[0, 0, 0], [0.001, 0, 0], [10, 0, 0], [10.001, 0, 0]]
    assert _point_problem(pts, 2, 1.0).partition_info()[2] == 2


def test_cube_partition_tiles_index_square():  # test_cluster.cpp:127-152
    v, t = orc.voxel_surface(9, -1.0, 1.0)
    prob = orc.Problem.kelvin(v, t, b_min=15, eta=0.8)
    nodes, _, perm, _ = prob.tree()
    blocks = prob.blocks()
    seen = np.zeros((972, 972), np.int8)
    for rn, cn, adm, _ in blocks:
        if not adm:
            assert nodes[rn, 2] < 0 or nodes[cn, 2] < 0
        r = perm[nodes[rn, 0]:nodes[rn, 1]]
        c = perm[nodes[cn, 0]:nodes[cn, 1]]
        seen[np.ix_(r, c)] += 1
    assert (seen == 1).all()
    nb, na, _ = prob.partition_info()
    assert 0 < na < nb
    # tree invariants (test_cluster.cpp:25-48)
    for nd in nodes:
        if nd[2] < 0:
            assert nd[1] - nd[0] <= 15
        else:
            l, r = nodes[nd[2]], nodes[nd[3]]
            assert l[0] == nd[0] and l[1] == r[0] and r[1] == nd[1]


def test_increasing_eta_keeps_admissible_leaves():  # test_cluster.cpp:154-159
    v, t = orc.voxel_surface(6, -1.0, 1.0)
    n1 = orc.Problem.kelvin(v, t, b_min=10, eta=0.8).partition_info()[1]
    n2 = orc.Problem.kelvin(v, t, b_min=10, eta=1.6).partition_info()[1]
    assert n2 >= n1


def test_partition_json_is_valid():  # test_cluster.cpp:171-177
    import json
    v, t = orc.voxel_surface(3, -1.0, 1.0)
    prob = orc.Problem.kelvin(v, t, b_min=8, eta=0.8)
    j = json.loads(prob.partition_json())
    assert len(j["blocks"]) == prob.partition_info()[0]
    assert j["c_sp"] == prob.partition_info()[2]


# ---- test_aca.cpp ------------------------------------------------------------
def test_rank1_block_in_one_cross():  # test_aca.cpp:35-47
    m = np.outer(RV(20, 11), RV(15, 12))
    s = orc.AcaDense(m).run(1e-8, 0.8, 100).state()
    assert s["rank"] == 1 and s["last_stop"] == 2 and s["num_consumed"] == 20
    assert np.linalg.norm(m - s["U"] @ s["V"].T) < 1e-12 * np.linalg.norm(m)


def test_zero_block_exhausts_at_rank0():  # test_aca.cpp:49-56
    s = orc.AcaDense(np.zeros((8, 6))).run(1e-6, 0.8, 100).state()
    assert s["rank"] == 0 and s["num_consumed"] == 8


def test_kernel_block_accuracy():  # test_aca.cpp:58-65
    a, _, _ = separated_kernel_matrix(30, 30, 5, RV)
    s = orc.AcaDense(a).run(1e-6, 0.8, 30).state()
    assert np.linalg.norm(a - s["U"] @ s["V"].T) <= 1e-6 * np.linalg.norm(a)
    assert s["rank"] <= 20


def test_pivots_interpolate():  # test_aca.cpp:67-81
    a, _, _ = separated_kernel_matrix(25, 20, 7, RV)
    s = orc.AcaDense(a).run(1e-4, 0.8, 25).state()
    S = s["U"] @ s["V"].T
    for l, (i, j) in enumerate(s["pivots"]):
        np.testing.assert_allclose(S[i, :], a[i, :], rtol=1e-9)
        np.testing.assert_allclose(S[:, j], a[:, j], rtol=1e-9)
        assert s["V"][j, l] == pytest.approx(1.0)


def test_frobenius_bookkeeping():  # test_aca.cpp:83-90
    a, _, _ = separated_kernel_matrix(22, 28, 3, RV)
    s = orc.AcaDense(a).run(1e-8, 0.8, 22).state()
    assert s["frob_sq"] == pytest.approx(np.sum((s["U"] @ s["V"].T) ** 2), rel=1e-10)


def test_extension_replays_bitwise():  # test_aca.cpp:92-110
    a, _, _ = separated_kernel_matrix(30, 30, 9, RV)
    once = orc.AcaDense(a).extend(6, 30).state()
    twice = orc.AcaDense(a).extend(3, 30).extend(3, 30).state()
    assert once["rank"] == twice["rank"] == 6
    assert (once["pivots"] == twice["pivots"]).all()
    assert (once["U"] == twice["U"]).all() and (once["V"] == twice["V"]).all()


def test_exhausted_extension_is_noop():  # test_aca.cpp:112-135
    m = np.outer(RV(10, 21), RV(10, 22))
    h = orc.AcaDense(m).run(1e-10, 0.8, 10)
    k = h.state()["rank"]
    s = h.extend(3, 10).state()
    assert s["rank"] == k and s["last_stop"] == 2
    s2 = orc.AcaDense(np.outer(RV(12, 31), RV(9, 32))).extend(2, 12).state()
    assert s2["rank"] == 1 and s2["num_consumed"] == 12


def test_stop_rule_sound():  # test_aca.cpp:169-180
    for seed in (101, 202, 303, 404):
        a, _, _ = separated_kernel_matrix(32, 26, seed, RV)
        s = orc.AcaDense(a).run(1e-5, 0.8, 26).state()
        if s["last_stop"] == 1:
            assert np.linalg.norm(a - s["U"] @ s["V"].T) <= 3e-5 * np.linalg.norm(a)
