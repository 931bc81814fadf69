"""Host-side product logic without a GPU: meshes, quadrature tables, cluster
tree and block partition bit-exact against the oracle, error behaviour,
and the C ABI exports (every symbol include/*.h declares)."""
import ctypes
import json
import os
import re

import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from paper_2205_04752_b200 import _lib
from oracle import oracle as orc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b((?:hmgpu|hmb)_[a-z_0-9]+)\s*\(", txt)))


@pytest.mark.parametrize("header,lib", [("hmgpu.h", _lib.HMGPU_PATH),
                                        ("hmbem.h", _lib.HMBEM_PATH)])
def test_c_abi_exports_every_declared_symbol(header, lib):
    names = _declared(header)
    assert len(names) > 10
    so = ctypes.CDLL(lib)
    missing = [n for n in names if not hasattr(so, n)]
    assert not missing, missing


def test_no_device_is_reported_cleanly():
    if hm.device_count() > 0:
        pytest.skip("GPU present")
    h = hm.HMatrix.kelvin(hm.Mesh.icosphere(1), b_min=8, device=-1)
    with pytest.raises(hm.DeviceError):
        h.assemble(eps=1e-4)
    with pytest.raises(hm.DeviceError):
        hm.HMatrix.kelvin(hm.Mesh.icosphere(1), b_min=8, device=0)


# ---- meshes -----------------------------------------------------------------
def test_voxel_cube_matches_oracle_bitwise():
    for n, lo, hi in [(9, -1.0, 1.0), (4, 0.0, 1.0), (16, 0.0, 1.0)]:
        m = hm.Mesh.voxel_cube(n, lo, hi).arrays()
        v, t = orc.voxel_surface(n, lo, hi)
        assert (m["vertices"] == v).all() and (m["triangles"] == t).all()
        g = orc.mesh_geometry(v, t)
        for k in ("centroids", "areas", "normals", "diam"):
            assert (m[k] == g[k]).all(), k


def test_cube9_counts_and_area():  # test_mesh.cpp:22-39
    m = hm.Mesh.voxel_cube(9, -1.0, 1.0)
    a = m.arrays()
    assert m.sizes == (488, 972)
    assert a["areas"].sum() == pytest.approx(24.0, rel=1e-12)
    m.validate()


@pytest.mark.parametrize("level", [0, 1, 3, 5])
def test_icosphere(level):
    m = hm.Mesh.icosphere(level)
    a = m.arrays()
    nt = 20 * 4 ** level
    assert m.num_triangles == nt and m.num_vertices == nt // 2 + 2
    m.validate()  # closed, consistently oriented
    assert (np.einsum("ij,ij->i", a["normals"], a["centroids"]) > 0).all()
    assert np.allclose(np.linalg.norm(a["vertices"], axis=1), 1.0, atol=1e-15)
    g = orc.mesh_geometry(a["vertices"], a["triangles"])
    for k in ("centroids", "areas", "normals", "diam"):
        assert (a[k] == g[k]).all(), k
    if level >= 3:
        assert a["areas"].sum() == pytest.approx(4 * np.pi, rel=2e-2)


def test_ellipsoid_and_labels(tmp_path):
    m = hm.Mesh.ellipsoid(2, 2.0, 1.0, 0.5)
    v = m.arrays()["vertices"]
    assert np.allclose((v[:, 0] / 2) ** 2 + v[:, 1] ** 2 + (v[:, 2] / 0.5) ** 2, 1.0)
    c = hm.Mesh.voxel_cube(4, 0.0, 1.0)
    c.label_dirichlet("x3<=0")
    a = c.arrays()
    assert (a["dirichlet"] == (a["centroids"][:, 2] <= 0)).all() and a["dirichlet"].sum() == 32
    with pytest.raises(hm.MeshError):
        c.label_dirichlet("y3<=0")
    p = str(tmp_path / "c.off")
    c.save_off(p)
    back = hm.Mesh.load_off(p).arrays()
    assert (back["vertices"] == a["vertices"]).all() and (back["triangles"] == a["triangles"]).all()


def test_off_rejects_open_surface(tmp_path):
    p = tmp_path / "open.off"
    p.write_text("OFF\n4 2 0\n0 0 0\n1 0 0\n0 1 0\n0 0 1\n3 0 1 2\n3 0 1 3\n")
    with pytest.raises(hm.MeshError):
        hm.Mesh.load_off(str(p))


# ---- quadrature tables --------------------------------------------------------
def test_rules_match_oracle_bitwise():
    """The tables the host uploads to the device (tiers 2/4/5) are the
    reference's gauss_rule; compared through the oracle restatement."""
    for order in range(1, 7):
        ref = orc.gauss_rule(order)
        got = hm.gauss_rule(order)
        for x, y in zip(got, ref):
            assert (x == y).all()
        assert len(got[2]) == [1, 3, 6, 6, 7, 12][order - 1]
    with pytest.raises(hm.Error):
        hm.gauss_rule(7)


# ---- tree / partition: bit-exact against the oracle ----------------------------
def _compare_partition(mesh, b_min, eta):
    a = mesh.arrays()
    h = hm.HMatrix.kelvin(mesh, b_min=b_min, eta=eta, device=-1)
    ref = orc.Problem.kelvin(a["vertices"], a["triangles"], b_min=b_min, eta=eta)
    t = h.tree()
    nodes, boxes, perm, depth = ref.tree()
    assert (t.nodes == nodes).all() and (t.perm == perm).all() and t.depth == depth
    assert (t.boxes == boxes).all()
    assert (h.partition_blocks() == ref.blocks()).all()
    assert h.partition_info() == ref.partition_info()
    assert h.partition_json() == ref.partition_json()
    return h


@pytest.mark.parametrize("level,b_min", [(3, 32), (4, 32), (5, 32)])
def test_partition_bit_exact_icosphere(level, b_min):
    h = _compare_partition(hm.Mesh.icosphere(level), b_min, 1.0)
    j = json.loads(h.partition_json())
    assert j["beta"] == 1.0 and j["rows"] == 20 * 4 ** level


def test_partition_bit_exact_cube_and_ellipsoid():
    _compare_partition(hm.Mesh.voxel_cube(9, -1.0, 1.0), 15, 0.8)
    _compare_partition(hm.Mesh.voxel_cube(32, 0.0, 1.0), 64, 1.0)
    _compare_partition(hm.Mesh.ellipsoid(4, 2.0, 1.0, 0.5), 32, 1.0)


def test_newton_partition_bit_exact():
    pts = orc.random_vector(3 * 300, 9).reshape(300, 3)
    h = hm.HMatrix.newton(pts, b_min=12, eta=1.2, device=-1)
    ref = orc.Problem.newton(pts, b_min=12, eta=1.2)
    assert h.partition_json() == ref.partition_json()
    assert (h.tree().perm == ref.tree()[2]).all()


def test_config_tree_shapes():
    """exact tree shapes of the BASELINE configs."""
    for mesh, b_min, depth, leaves, leaf in [
        (hm.Mesh.icosphere(3), 32, 6, 64, 20),
        (hm.Mesh.icosphere(5), 32, 10, 1024, 20),
        (hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 12, 4096, 48),
    ]:
        t = hm.HMatrix.kelvin(mesh, b_min=b_min, device=-1).tree()
        lv = t.nodes[t.leaves()]
        assert t.depth == depth and len(lv) == leaves
        assert (lv[:, 1] - lv[:, 0] == leaf).all()


def test_admissible_matches_oracle():
    rng = np.random.default_rng(0)
    for _ in range(200):
        lo1, lo2 = rng.normal(size=3), rng.normal(size=3) * 3
        b1 = np.concatenate([lo1, lo1 + rng.random(3)])
        b2 = np.concatenate([lo2, lo2 + rng.random(3)])
        eta = rng.random() * 2 + 0.1
        assert hm.admissible(b1, b2, eta) == orc.admissible(b1, b2, eta)
    with pytest.raises(hm.Error):
        hm.admissible([0] * 6, [1] * 6, 0.0)


def test_bad_arguments_raise_reference_errors():
    m = hm.Mesh.icosphere(2)
    with pytest.raises(hm.Error):
        hm.HMatrix.kelvin(m, b_min=0, device=-1)
    with pytest.raises(hm.Error):
        hm.HMatrix.kelvin(m, eta=-1.0, device=-1)
    with pytest.raises(hm.Error):
        hm.HMatrix.kelvin(m, nu=0.5, device=-1)
    with pytest.raises(hm.MeshError):
        hm.Mesh.from_arrays(np.zeros((3, 3)), np.array([[0, 1, 2]]))


def test_shards_cover_rows_disjointly():
    m = hm.Mesh.icosphere(4)
    for count in (1, 2, 4, 8):
        ranges = [hm.HMatrix.kelvin(m, b_min=32, device=-1, shard=(r, count)).row_range
                  for r in range(count)]
        assert ranges[0][0] == 0 and ranges[-1][1] == m.num_triangles
        for a, b in zip(ranges, ranges[1:]):
            assert a[1] == b[0] and a[0] < a[1]


# ---- Galerkin / operator-algebra host pieces vs the oracle -------
@pytest.mark.parametrize("case,order", [(1, 7), (2, 7), (3, 9), (2, 5)])
def test_pair_rules_match_oracle_bitwise(case, order):
    got, ref = hm.pair_rule(case, order), orc.pair_rule(case, order)
    for x, y in zip(got, ref):
        assert (x == y).all()


def test_sparse_ops_match_oracle_bitwise():
    mesh = hm.Mesh.voxel_cube(3, -1.0, 1.0)
    a = mesh.arrays()
    for which in range(4):
        cols, vals = hm.sparse_op(mesh, which)
        dense = np.zeros((mesh.num_triangles, mesh.num_vertices))
        for t in range(mesh.num_triangles):
            for s in range(3):
                dense[t, cols[t, s]] += vals[t, s]
        assert (dense == orc.sparse_op(a["vertices"], a["triangles"], which)).all()


def test_galerkin_and_kdelta_partitions_bit_exact():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    for which in (0, 1):
        h = hm.HMatrix.galerkin(mesh, which, b_min=32, eta=1.0, device=-1)
        o = orc.Problem.galerkin(a["vertices"], a["triangles"], which, b_min=32, eta=1.0)
        assert h.partition_json() == o.partition_json()
    h = hm.HMatrix.kdelta(mesh, b_min=32, eta=1.0, device=-1)
    o = orc.Problem.kdelta(a["vertices"], a["triangles"], b_min=32, eta=1.0)
    assert h.partition_json() == o.partition_json()
    assert (h.rows, h.cols) == (mesh.num_triangles, mesh.num_vertices)


def test_dof_layout_of_the_experiment_cube():
    """classify_dofs (mesh.cpp:278-293) on make_cube_mesh's labelling."""
    mesh = hm.Mesh.voxel_cube(4, -1.0, 1.0)
    mesh.label_dirichlet("x1>=1|x2<=-1|x3>=1")
    L = hm.DofLayout(mesh)
    a = mesh.arrays()
    d = a["dirichlet"].astype(bool)
    assert (L.dirichlet_triangle_ids == np.nonzero(d)[0]).all()
    T = a["triangles"]
    for v in L.neumann_interior_nodes:
        assert not d[(T == v).any(axis=1)].any()
    assert len(L.t_dofs) == 3 * d.sum() and len(L.u_dofs) == 3 * len(L.neumann_interior_nodes)


# ---- inputs shared with the reference arm (no product import there) -------
def test_oracle_mesh_generators_match_product_bitwise():
    for level in (0, 2, 5):
        v, t = orc.icosphere(level)
        a = hm.Mesh.icosphere(level).arrays()
        assert (v == a["vertices"]).all() and (t == a["triangles"]).all()
    v, t = orc.ellipsoid(4, 2.0, 1.0, 0.5)
    a = hm.Mesh.ellipsoid(4, 2.0, 1.0, 0.5).arrays()
    assert (v == a["vertices"]).all() and (t == a["triangles"]).all()


def test_random_vector_streams_match_oracle():
    """hm.random_vector: mt19937_64 + uniform_real_distribution(-1,1) (the
    reference's random_vector, proj/tests/oracles.cpp:415-421) and
    std::normal_distribution, identical to the oracle's streams."""
    for seed in (0, 1, 3):
        assert (hm.random_vector(5000, seed, "uniform") == orc.random_vector(5000, seed)).all()
    for seed in (2, 4):
        assert (hm.random_vector(5000, seed, "normal") == orc.normal_vector(5000, seed)).all()


def test_random_vector_stream_matches_oracle_and_golden():
    """hm.random_vector (hmb_random_vector) is the reference test suite's
    random_vector (proj/tests/oracles.cpp:414-420: std::mt19937_64 seeded
    with `seed`, uniform_real_distribution(-1, 1)) -- equal to the oracle's
    restatement bit for bit, and to committed values of the stream (seed 0);
    the normal variant (std::normal_distribution) likewise."""
    import paper_2205_04752_b200 as hm
    from oracle import oracle as orc
    for seed in (0, 1, 2, 3, 4, 12345):
        for n in (1, 7, 1000):
            assert (hm.random_vector(n, seed) == orc.random_vector(n, seed)).all()
            assert (hm.random_vector(n, seed, "normal") == orc.normal_vector(n, seed)).all()
    golden = [-0.6804132732590783, 0.9842904192596575, -0.9208619483102687,
              0.19498932538934355]
    assert hm.random_vector(4, 0).tolist() == golden
    assert hm.random_vector(3, 4, "normal").tolist() == [
        -0.2361666787221914, 1.460615509829741, -0.6497372926308559]
    # the stream is a prefix stream: longer vectors extend shorter ones
    assert (hm.random_vector(100, 7)[:10] == hm.random_vector(10, 7)).all()
