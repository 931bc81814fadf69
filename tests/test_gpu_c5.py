"""Parity at config 5's size (1,310,720 triangles, 16 RHS): one 1/8
block-row shard -- the per-GPU share at 8 GPUs (~60 GB on the device) --
checked for its partition, sampled ACA blocks (re-run by the oracle, bit-
identical state), rows of A x from oracle entries (within 10 eps_ACA of the
exact row sums), and each of the 16 columns of the tensor-core multi-RHS
sweep against the single-RHS sweep."""
import gc
import os

import numpy as np
import pytest

import paper_2205_04752_b200 as hm
from oracle import oracle as orc

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_config5_shard():
    """Config 5's per-GPU share at 8 GPUs: block-row shard 0 of 8 of the
    1,310,720-triangle icosphere (163,840 rows, ~60 GB on the device)."""
    gc.collect()
    eps = 1e-5
    mesh = hm.Mesh.icosphere(8)
    a = mesh.arrays()
    g = hm.HMatrix.kelvin(mesh, b_min=64, eta=1.0, device=0, shard=(0, 8))
    g.assemble(eps=eps, beta=0.8, lookahead=2)
    o = orc.Problem.kelvin(a["vertices"], a["triangles"], b_min=64, eta=1.0)
    assert (g.partition_blocks() == o.blocks()).all()
    t = g.tree()
    assert (t.perm == o.tree()[2]).all()
    rb, re = g.row_range
    blocks = g.partition_blocks()
    owned = (t.nodes[blocks[:, 0], 0] >= rb) & (t.nodes[blocks[:, 0], 1] <= re)
    adm = np.nonzero(owned & (blocks[:, 2] == 1))[0]
    gk, gl, _, _ = g.ranks()
    assert (gk[:, owned & (blocks[:, 2] == 1)] >= 0).all()
    assert (gk[:, ~owned] == -1).all()
    # sampled ACA blocks re-run by the oracle: bit-identical state
    sizes = t.nodes[blocks[adm, 0], 1] - t.nodes[blocks[adm, 0], 0]
    rng = np.random.default_rng(5)
    pick = list(adm[np.argsort(-sizes)[:4]]) + list(rng.choice(adm, 24, replace=False))
    for b in pick:
        comp = int(rng.integers(0, 6))
        kc, K, fs, _ = o.aca_block(comp, int(b), eps=eps, beta=0.8, lookahead=2)
        assert (gk[comp, b], gl[comp, b]) == (kc, K), (b, comp)
        assert g.factor(comp, int(b))["frob_sq"] == fs
    # 16 RHS (fp64 tensor-core sweep) against 16 single-RHS sweeps
    n = g.cols
    X = np.asfortranarray(hm.random_vector(n * 16, 4, "normal").reshape(16, n).T)
    Y = g.matvec(X)
    for q in range(16):
        yq = g.matvec(np.ascontiguousarray(X[:, q]))
        assert rel(Y[:, q], yq) < 1e-13, q
    # rows of A x from oracle entries: the H-approximation within 10 eps
    N = mesh.num_triangles
    orc.set_threads(os.cpu_count() or 1)
    own_rows = t.perm[rb:re]
    dofs = np.concatenate([c * N + rng.choice(own_rows, 8, replace=False) for c in range(3)])
    exact, mag = o.rows_dot(dofs, X[:, 0])
    got = Y[dofs, 0]
    assert np.all(np.abs(got - exact) <= 10 * eps * mag)
    assert np.linalg.norm(got - exact) <= 10 * eps * np.linalg.norm(exact)
