"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on
the same seeded inputs.  Bars (BASELINE.json north_star):
partition bit-exact, ACA ranks within +-2 per (component, block), matvec
relative l2 error <= 10 eps_ACA against the oracle H-matvec, near-field
entries within 1e-13 of the component scale, and the reference's own
property tests re-run on the device path."""
import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc
from tests.helpers import centroid_points_and_boxes, cube_mesh, separated_kernel_matrix

pytestmark = pytest.mark.gpu
RV = orc.random_vector


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


# ---------------------------------------------------------------------------
# config 1: icosphere L3, 1280 triangles, b_min 32, eta 1, eps 1e-4, x seed 0
@pytest.fixture(scope="module")
def c1():
    mesh = hm.Mesh.icosphere(3)
    a = mesh.arrays()
    eps = 1e-4
    g = hm.HMatrix.kelvin(mesh, E=1.0, nu=0.3, b_min=32, eta=1.0, device=0)
    g.assemble(eps=eps, beta=0.8, lookahead=2)
    o = orc.Problem.kelvin(a["vertices"], a["triangles"], 1.0, 0.3, b_min=32, eta=1.0)
    o.assemble(eps=eps, beta=0.8, lookahead=2)
    return dict(g=g, o=o, eps=eps, x=RV(3 * 1280, 0), mesh=mesh)


def test_c1_partition_identical(c1):
    assert c1["g"].partition_json() == c1["o"].partition_json()


def test_c1_ranks_within_two(c1):
    gk, gl, gc, _ = c1["g"].ranks()
    ok, ol, oc, _ = c1["o"].ranks()
    adm = ok >= 0
    assert (gk[adm] >= 0).all() and (gk[~adm] == -1).all()
    assert np.abs(gk[adm] - ok[adm]).max() <= 2
    assert np.abs(gl[adm] - ol[adm]).max() <= 2
    # canonical arithmetic: the device ACA is bit-reproducible by the oracle
    assert (gk == ok).all() and (gl == ol).all() and (gc == oc).all()


def test_c1_nearfield_entries(c1):
    g, o = c1["g"], c1["o"]
    nodes = g.tree().nodes
    blocks = g.partition_blocks()
    worst = 0.0
    for comp in range(6):
        scale = 0.0
        diffs = []
        for b, (rn, cn, adm, _) in enumerate(blocks):
            if adm:
                continue
            m = nodes[rn, 1] - nodes[rn, 0]
            n = nodes[cn, 1] - nodes[cn, 0]
            want = o.dense_block(comp, b, m, n)
            got = g.dense_block(comp, b)
            scale = max(scale, np.abs(want).max())
            diffs.append(np.abs(got - want).max())
            if rn != cn:  # off the diagonal the entries are bit-identical
                assert (got == want).all()
        worst = max(worst, max(diffs) / scale)
    assert worst <= 1e-13, worst  # self terms (closed form with log) to rounding


def test_c1_matvec_vs_oracle_and_dense(c1):
    g, o, x, eps = c1["g"], c1["o"], c1["x"], c1["eps"]
    y = g.matvec(x)
    assert rel(y, o.matvec(x)) <= 10 * eps
    A = o.dense_grid()
    assert rel(y, A @ x) <= 10 * eps
    yl = g.matvec(x, hm.Mode.Lookahead)
    assert rel(yl, o.matvec(x, 1)) <= 10 * eps
    assert rel(yl, A @ x) <= rel(y, A @ x) * 1.5


def test_c1_matvec_deterministic_and_multi_rhs(c1):
    g = c1["g"]
    X = np.stack([RV(3 * 1280, s) for s in range(4)], axis=1)
    Y = g.matvec(X)
    for q in range(4):
        y = g.matvec(X[:, q])
        assert (y == g.matvec(X[:, q])).all()  # bitwise repeatable
        # same products, different reduction segmentation per nrhs
        assert np.allclose(Y[:, q], y, rtol=1e-12, atol=1e-14 * np.abs(y).max())
    # linearity
    y01 = g.matvec(2.0 * X[:, 0] - 0.5 * X[:, 1])
    assert rel(y01, 2.0 * Y[:, 0] - 0.5 * Y[:, 1]) < 1e-13


@pytest.mark.parametrize("nrhs", [2, 16, 17, 35])
def test_c1_multi_rhs_dmma_sweep(c1, nrhs):
    """nrhs > 1 runs the fp64 tensor-core sweep (16 RHS per pass, zero-padded
    remainder); every column must equal the single-RHS product."""
    g, o = c1["g"], c1["o"]
    X = np.asfortranarray(np.stack([RV(3 * 1280, 100 + s) for s in range(nrhs)], axis=1))
    for mode, om in ((hm.Mode.Current, 0), (hm.Mode.Lookahead, 1)):
        Y = g.matvec(X, mode)
        assert Y.shape == X.shape
        assert (Y == g.matvec(X, mode)).all()  # deterministic
        for q in (0, nrhs // 2, nrhs - 1):
            y = g.matvec(np.ascontiguousarray(X[:, q]), mode)
            assert rel(Y[:, q], y) < 1e-13
            assert rel(Y[:, q], o.matvec(np.ascontiguousarray(X[:, q]), om)) < 1e-12


def test_c1_direct_matvec_policy(c1):
    """One-shot matvecs after a rank change sweep the blocks in place (no
    stream plan); same product within rounding of the summation order."""
    g, o = c1["g"], c1["o"]
    x = RV(3 * 1280, 11)
    y_plan = g.matvec(x)
    g.set_matvec_policy(True)
    try:
        y_direct = g.matvec(x)
        assert (y_direct == g.matvec(x)).all()
    finally:
        g.set_matvec_policy(False)
    assert rel(y_direct, y_plan) < 1e-13
    assert rel(y_direct, o.matvec(x)) < 1e-12


def test_c1_factors_match_oracle(c1):
    g, o = c1["g"], c1["o"]
    blocks = g.partition_blocks()
    adm = np.nonzero(blocks[:, 2])[0]
    for b in adm[:: max(1, len(adm) // 40)]:
        for comp in (0, 1, 4):
            fg, fo = g.factor(comp, b), o.factor(comp, b)
            assert (fg["pivots"] == fo["pivots"]).all()
            assert (fg["U"] == fo["U"]).all() and (fg["V"] == fo["V"]).all()
            assert fg["frob_sq"] == fo["frob_sq"]


def test_device_pointer_matvec(c1):
    torch = pytest.importorskip("torch")
    g, x = c1["g"], c1["x"]
    xd = torch.tensor(x, dtype=torch.float64, device="cuda")
    yd = torch.zeros(g.rows, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    g.matvec_ptr(xd.data_ptr(), yd.data_ptr(), 1)
    torch.cuda.synchronize()  # device-wide: covers the ctx's own stream
    assert (yd.cpu().numpy() == g.matvec(x)).all()


# ---------------------------------------------------------------------------
# small cube (config-3 family) and ellipsoid (config-4 family)
@pytest.mark.parametrize("kind", ["cube", "ellipsoid"])
def test_other_geometries(kind):
    if kind == "cube":
        mesh, b_min, eps = hm.Mesh.voxel_cube(16, 0.0, 1.0), 64, 1e-5
    else:
        mesh, b_min, eps = hm.Mesh.ellipsoid(3, 2.0, 1.0, 0.5), 32, 1e-4
    a = mesh.arrays()
    g = hm.HMatrix.kelvin(mesh, b_min=b_min, eta=1.0, device=0)
    g.assemble(eps=eps)
    o = orc.Problem.kelvin(a["vertices"], a["triangles"], b_min=b_min, eta=1.0)
    o.assemble(eps=eps)
    assert g.partition_json() == o.partition_json()
    gk, gl, _, _ = g.ranks()
    ok, ol, _, _ = o.ranks()
    assert (gk == ok).all() and (gl == ol).all()
    x = orc.normal_vector(g.cols, 2)
    assert rel(g.matvec(x), o.matvec(x)) <= 10 * eps


# ---------------------------------------------------------------------------
# the reference's H-matrix fixture (Newton kernel, cube(4), b_min 10, beta 0.8)
@pytest.fixture(scope="module")
def newton_pts():
    return centroid_points_and_boxes(cube_mesh(4))


def _newton(pts_boxes, **cfg):
    pts, boxes = pts_boxes
    g = hm.HMatrix.newton(pts, boxes, diag=2.0, b_min=10, eta=0.8, device=0)
    g.assemble(**cfg)
    o = orc.Problem.newton(pts, boxes, diag=2.0, b_min=10, eta=0.8)
    o.assemble(**cfg)
    return g, o


def test_newton_full_mode(newton_pts):  # test_hmatrix.cpp:76-90
    g, o = _newton(newton_pts, eps=1e-6)
    A = o.dense(0)
    x = RV(192, 17)
    assert rel(g.matvec(x), A @ x) <= 1e-5
    gk, gl, _, _ = g.ranks()
    ok, ol, _, _ = o.ranks()
    assert (gk == ok).all() and (gl == ol).all()  # entries are bit-exact here
    assert rel(g.matvec(x), o.matvec(x)) < 1e-13


def test_newton_coarse_mode_and_lookahead(newton_pts):  # test_hmatrix.cpp:92-140
    g, o = _newton(newton_pts, initial_rank=3, lookahead=2)
    A = o.dense(0)
    t = g.tree()
    kc, kl, co, _ = g.ranks()
    blocks = g.partition_blocks()
    for b, (rn, cn, adm, _) in enumerate(blocks):
        if not adm:
            continue
        assert kc[0, b] <= 3 and kl[0, b] <= 5
        r = t.perm[t.nodes[rn, 0]:t.nodes[rn, 1]]
        c = t.perm[t.nodes[cn, 0]:t.nodes[cn, 1]]
        ab = A[np.ix_(r, c)]
        f = g.factor(0, b)
        e_lo = np.linalg.norm(ab - f["U"][:, :kc[0, b]] @ f["V"][:, :kc[0, b]].T)
        e_hi = np.linalg.norm(ab - f["U"] @ f["V"].T)
        assert e_hi <= e_lo * (1 + 1e-12)


# ---------------------------------------------------------------------------
# single admissible block of an explicit matrix: test_aca.cpp on the device
def _aca_block(a, **cfg):
    m, n = a.shape
    rp = RV(3 * m, 1).reshape(m, 3)
    cp = RV(3 * n, 2).reshape(n, 3) + np.array([8.0, 0, 0])
    g = hm.HMatrix.dense(a, rp, cp, b_min=max(m, n), eta=0.8, device=0)
    assert g.partition_blocks().tolist() == [[0, 0, 1, 0]]
    g.assemble(**cfg)
    return g


def test_gpu_aca_rank1_and_zero():  # test_aca.cpp:35-56
    m = np.outer(RV(20, 11), RV(15, 12))
    g = _aca_block(m, eps=1e-8, beta=0.8, lookahead=0, max_rank=100)
    kc, kl, co, ls = g.ranks()
    assert kc[0, 0] == 1 and co[0, 0] == 20 and ls[0, 0] == hm.AcaStop.Exhausted
    f = g.factor(0, 0)
    assert np.linalg.norm(m - f["U"] @ f["V"].T) < 1e-12 * np.linalg.norm(m)
    z = _aca_block(np.zeros((8, 6)), eps=1e-6, lookahead=0)
    kc, _, co, _ = z.ranks()
    assert kc[0, 0] == 0 and co[0, 0] == 8


def test_gpu_aca_accuracy_interpolation_frob():  # test_aca.cpp:58-90
    a, _, _ = separated_kernel_matrix(30, 30, 5, RV)
    g = _aca_block(a, eps=1e-6, lookahead=0, max_rank=30)
    f = g.factor(0, 0)
    assert np.linalg.norm(a - f["U"] @ f["V"].T) <= 1e-6 * np.linalg.norm(a)
    assert f["U"].shape[1] <= 20
    a, _, _ = separated_kernel_matrix(25, 20, 7, RV)
    g = _aca_block(a, eps=1e-4, lookahead=0, max_rank=25)
    f = g.factor(0, 0)
    S = f["U"] @ f["V"].T
    for l, (i, j) in enumerate(f["pivots"]):
        np.testing.assert_allclose(S[i, :], a[i, :], rtol=1e-9)
        np.testing.assert_allclose(S[:, j], a[:, j], rtol=1e-9)
        assert f["V"][j, l] == pytest.approx(1.0)
    a, _, _ = separated_kernel_matrix(22, 28, 3, RV)
    g = _aca_block(a, eps=1e-8, lookahead=0, max_rank=22)
    f = g.factor(0, 0)
    assert f["frob_sq"] == pytest.approx(np.sum((f["U"] @ f["V"].T) ** 2), rel=1e-10)
    # same pivots as the oracle's aca_run on the same matrix
    s = orc.AcaDense(a).run(1e-8, 0.8, 22).state()
    assert (f["pivots"] == s["pivots"]).all()


def test_gpu_aca_extension_replay():  # test_aca.cpp:92-124
    a, _, _ = separated_kernel_matrix(30, 30, 9, RV)
    once = _aca_block(a, initial_rank=6, lookahead=0, max_rank=30)
    twice = _aca_block(a, initial_rank=3, lookahead=0, max_rank=30)
    twice.extend_lookahead([(0, 0)], 3)
    f1, f2 = once.factor(0, 0), twice.factor(0, 0)
    assert f1["U"].shape[1] == f2["U"].shape[1] == 6
    assert (f1["pivots"] == f2["pivots"]).all()
    assert (f1["U"] == f2["U"]).all() and (f1["V"] == f2["V"]).all()
    ref = orc.AcaDense(a).extend(6, 30).state()
    assert (f1["pivots"] == ref["pivots"]).all()
    # exhausted: extension is a no-op
    r1 = _aca_block(np.outer(RV(10, 21), RV(10, 22)), eps=1e-10, lookahead=0, max_rank=10)
    k = r1.ranks()[1][0, 0]
    r1.extend_lookahead([(0, 0)], 3)
    assert r1.ranks()[1][0, 0] == k


# ---------------------------------------------------------------------------
# adaptive matvec: estimator, marking and Algorithm 2 against the oracle
def test_gpu_gamma_and_marking_match_oracle(newton_pts):
    g, o = _newton(newton_pts, initial_rank=2, lookahead=2)
    x = RV(192, 3)
    gg = g.gamma_contributions(x)
    og, odiff, oterms = o.gamma(x)
    assert gg.gamma == og and (gg.difference == odiff).all()
    assert len(gg.terms) == len(oterms)
    for tg, to in zip(gg.terms, oterms):
        assert (tg.comp, tg.block) == (to["comp"], to["block"])
        assert (tg.idx == to["idx"]).all() and (tg.val == to["val"]).all()
    c_sp = g.sparsity_constant
    for theta in (0.3, 0.7, 0.9):
        mg, gpk = g.mark_blocks(theta, c_sp, 192, 192)
        mo, opk = o.mark(theta, c_sp, 192, 192, len(oterms))
        assert (mg == mo).all() and gpk == opk


def test_gpu_amvm_matches_oracle_newton(newton_pts):  # test_amvm.cpp:162-193
    g, o = _newton(newton_pts, initial_rank=2, lookahead=2)
    x = RV(192, 11)
    b_true = o.dense(0) @ x
    eps = 1e-7 * np.linalg.norm(b_true)
    bg, rep = g.amvm_multiply(x, theta=0.7, eps_amvm=eps, max_iterations=100)
    bo, it, conv = o.amvm(x, theta=0.7, eps_amvm=eps, max_iterations=100)
    assert rep.converged and conv and len(rep.iterations) == len(it)
    for r, ref in zip(rep.iterations, it):
        assert r.marked == int(ref[3])
        assert r.gamma == pytest.approx(ref[1], rel=1e-8, abs=1e-14)
    assert np.linalg.norm(bg - b_true) <= 50 * eps
    assert rel(bg, bo) < 1e-12


def test_gpu_amvm_kelvin_ellipsoid_matches_oracle():
    """config-4 family at desk scale: full-mode eps 1e-2, 5 sweeps."""
    mesh = hm.Mesh.ellipsoid(3, 2.0, 1.0, 0.5)
    a = mesh.arrays()
    g = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
    g.assemble(eps=1e-2, beta=0.8, lookahead=2)
    o = orc.Problem.kelvin(a["vertices"], a["triangles"], b_min=32, eta=1.0)
    o.assemble(eps=1e-2, beta=0.8, lookahead=2)
    c = a["centroids"]
    bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.05 ** 2))
    x = np.tile(bump, 3) + 1e-3 * RV(3 * len(c), 3)
    bg, rep = g.amvm_multiply(x, theta=0.7, eps_amvm=1e-6, max_iterations=5)
    bo, it, conv = o.amvm(x, theta=0.7, eps_amvm=1e-6, max_iterations=5)
    assert len(rep.iterations) == len(it)
    for r, ref in zip(rep.iterations, it):
        assert r.gamma == ref[1]  # bit-identical estimator
        assert r.marked == int(ref[3])
        assert r.cumulative_pivots == int(ref[4])
    assert rel(bg, bo) < 1e-13
    gk, gl, _, _ = g.ranks()
    ok, ol, _, _ = o.ranks()
    assert (gk == ok).all() and (gl == ol).all()


@pytest.mark.parametrize("world", [2, 4])
def test_block_row_shards_on_one_device(c1, world):
    """The multi-GPU decomposition run shard by shard on one
    device: every shard assembles the blocks of its row range and its matvec
    fills only its rows, so the sum of the shard products (the all-reduce of
    bench.py) equals the whole operator's product, and every owned block has
    the whole operator's ranks."""
    g = c1["g"]
    mesh = hm.Mesh.icosphere(3)
    x = RV(3 * 1280, 5)
    X = np.asfortranarray(np.stack([RV(3 * 1280, 40 + s) for s in range(3)], axis=1))
    y_full = g.matvec(x)
    Y_full = g.matvec(X)
    k_full, kl_full, _, _ = g.ranks()
    y = np.zeros_like(y_full)
    Y = np.zeros_like(Y_full)
    owned = np.zeros(k_full.shape[1], dtype=int)
    for r in range(world):
        s = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0, shard=(r, world))
        s.assemble(eps=1e-4, beta=0.8, lookahead=2)
        ys = s.matvec(x)
        rb, re = s.row_range
        t = s.tree()
        rows = t.perm[rb:re]
        mask = np.zeros(1280, dtype=bool)
        mask[rows] = True
        full_mask = np.tile(mask, 3)
        assert (ys[~full_mask] == 0.0).all()  # only the shard's rows
        y += ys
        Y += s.matvec(X)  # the tensor-core multi-RHS sweep on a shard
        k, kl, _, _ = s.ranks()
        mine = k[0] >= 0
        owned += mine
        assert (k[:, mine] == k_full[:, mine]).all() and (kl[:, mine] == kl_full[:, mine]).all()
    adm = k_full[0] >= 0
    assert (owned[adm] == 1).all()
    assert rel(y, y_full) < 1e-15
    assert rel(Y, Y_full) < 1e-15


@pytest.mark.parametrize("layout", ["1", "2"])
def test_stream_layouts_agree(c1, layout):
    """Both job layouts of the streamed matvec (contiguous runs per warp,
    round-robin chain units; HMGPU_MV_LAYOUT) give the product of this
    process within rounding of the summation order, and each is
    deterministic."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    y = c1["g"].matvec(c1["x"])
    code = ("import sys, numpy as np; sys.path.insert(0, %r);"
            "import paper_2205_04752_b200 as hm; from oracle import oracle as orc;"
            "g = hm.HMatrix.kelvin(hm.Mesh.icosphere(3), E=1.0, nu=0.3, b_min=32, eta=1.0,"
            " device=0); g.assemble(eps=1e-4, beta=0.8, lookahead=2);"
            "x = orc.random_vector(3 * 1280, 0); a = g.matvec(x); b = g.matvec(x);"
            "sys.stdout.write(a.tobytes().hex() + ' ' + b.tobytes().hex())" % root)
    env = dict(os.environ, HMGPU_MV_LAYOUT=layout)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True,
                         text=True, timeout=600, check=True).stdout.split()
    a = np.frombuffer(bytes.fromhex(out[0]))
    b = np.frombuffer(bytes.fromhex(out[1]))
    assert (a == b).all()
    assert rel(a, y) < 1e-13
    assert rel(a, c1["o"].matvec(c1["x"])) < 10 * c1["eps"]


def test_multi_rhs_plans_share_the_spare_arena_and_follow_rank_changes():
    """The 16-RHS plan packs its factors into the same idle arena as the
    1-RHS stream plan: alternating the two keeps every product right, and a
    refinement (promote + extend) invalidates both plans."""
    mesh = hm.Mesh.icosphere(3)
    g = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
    g.assemble(eps=1e-3, beta=0.8, lookahead=2)
    n = g.cols
    X = np.asfortranarray(np.stack([RV(n, 200 + s) for s in range(16)], axis=1))

    def cols():
        return np.stack([g.matvec(np.ascontiguousarray(X[:, q])) for q in range(16)], axis=1)

    Y1 = g.matvec(X)
    C1 = cols()
    Y2 = g.matvec(X)
    assert (Y1 == Y2).all() and rel(Y1, C1) < 1e-13
    kc, kl, _, _ = g.ranks()
    pairs = [(q, b) for q in range(6) for b in range(kc.shape[1])
             if kc[q, b] >= 0 and kl[q, b] > kc[q, b]][::3]
    assert pairs
    g.promote(pairs)
    g.extend_lookahead(pairs, 2)
    Y3 = g.matvec(X)
    C3 = cols()
    assert rel(Y3, C3) < 1e-13 and rel(Y3, Y1) > 1e-12  # the new ranks are used


def test_auto_matvec_policy_runs_the_first_product_in_place(c1):
    """Policy "auto": the first 1-RHS product after a rank change sweeps the
    blocks in place (no plan), the second builds the plan; a rank change
    re-arms it.  Both agree with the planned product to rounding."""
    mesh = hm.Mesh.icosphere(3)
    g = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
    g.assemble(eps=1e-4, beta=0.8, lookahead=2)
    x = RV(g.cols, 21)
    g.set_profiling(True)

    def launches():
        return {k: g.kernel_times(k, reset=True)[1] for k in ("hmv_blocks", "hmv_stream")}

    launches()
    g.set_matvec_policy("auto")
    try:
        y1 = g.matvec(x)
        n1 = launches()
        y2 = g.matvec(x)
        n2 = launches()
        y3 = g.matvec(x)
        assert n1["hmv_blocks"] == 1 and n1["hmv_stream"] == 0  # in place
        assert n2["hmv_blocks"] == 0 and n2["hmv_stream"] == 1  # the plan
        assert (y2 == y3).all() and rel(y1, y2) < 1e-13
        launches()
        kc, kl, _, _ = g.ranks()
        pairs = [(q, b) for q in range(6) for b in range(kc.shape[1])
                 if kc[q, b] >= 0 and kl[q, b] > kc[q, b]][:5]
        g.promote(pairs)
        g.matvec(x)
        n4 = launches()
        assert n4["hmv_blocks"] == 1 and n4["hmv_stream"] == 0  # re-armed by the rank change
    finally:
        g.set_matvec_policy(False)
        g.set_profiling(False)
    assert hm.api._lib.gpu.hmgpu_set_matvec_policy(g.gpu_ctx, 3) != 0  # 0, 1, 2 only


@pytest.mark.parametrize("mesh_name,rows,parts", [
    ("ico3", 40, 0),     # 40-row leaves: 5 consumer warps, a row tile each
    ("cube16", 48, 0),   # 48-row leaves: 6 consumer warps (config 3's shape)
    ("cube12", 54, 0),   # 54-row leaves: 8 consumer warps, 7 row tiles
    ("cube16", 48, 3),   # every leaf cut into 3 parts: partial slices + ordered reduce
    ("ico3", 40, 8),
])
def test_multi_rhs_consumer_warp_configurations(mesh_name, rows, parts, monkeypatch):
    """The 16-RHS sweep picks its consumer warps from the leaves' row tiles and
    may cut leaves into parts; every configuration gives the 1-RHS product."""
    mesh = {"ico3": lambda: hm.Mesh.icosphere(3), "cube16": lambda: hm.Mesh.voxel_cube(16, 0.0, 1.0),
            "cube12": lambda: hm.Mesh.voxel_cube(12, 0.0, 1.0)}[mesh_name]()
    if parts:
        monkeypatch.setenv("HMGPU_M16_PARTS", str(parts))
    g = hm.HMatrix.kelvin(mesh, b_min=64, eta=1.0, device=0)
    g.assemble(eps=1e-4, beta=0.8, lookahead=2)
    t = g.tree()
    leaves = t.nodes[t.nodes[:, 2] < 0]
    sizes = leaves[:, 1] - leaves[:, 0]
    assert sizes.max() == rows and sizes.max() <= 64
    for nrhs in (16, 19):
        X = np.asfortranarray(np.stack([RV(g.cols, 400 + s) for s in range(nrhs)], axis=1))
        for mode in (hm.Mode.Current, hm.Mode.Lookahead):
            Y = g.matvec(X, mode)
            assert (Y == g.matvec(X, mode)).all()  # deterministic (dynamic hand-out included)
            for q in (0, 9, nrhs - 1):
                y = g.matvec(np.ascontiguousarray(X[:, q]), mode)
                assert rel(Y[:, q], y) < 1e-13


def test_multi_rhs_large_leaves_fall_back_to_the_block_sweep():
    """Leaves above 64 rows are outside the TMA-fed sweep's tiling: the
    product runs on the block-sweep kernel and stays the same product."""
    mesh = hm.Mesh.icosphere(3)
    g = hm.HMatrix.kelvin(mesh, b_min=96, eta=1.0, device=0)
    g.assemble(eps=1e-4, beta=0.8, lookahead=2)
    t = g.tree()
    leaves = t.nodes[t.nodes[:, 2] < 0]
    assert (leaves[:, 1] - leaves[:, 0]).max() > 64
    X = np.asfortranarray(np.stack([RV(g.cols, 300 + s) for s in range(16)], axis=1))
    Y = g.matvec(X)
    for q in (0, 7, 15):
        assert rel(Y[:, q], g.matvec(np.ascontiguousarray(X[:, q]))) < 1e-13
