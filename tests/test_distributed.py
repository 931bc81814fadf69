"""Block-row sharding over ranks on CPU with gloo, world 2.

Each rank builds the host-side operator for its shard (device = -1), takes
the blocks whose row cluster lies in its row range, computes their partial
product from the oracle's dense Kelvin matrix, and the ranks combine with
the protocol bench.py runs over NCCL: x broadcast from rank 0, y summed with
all-reduce (rows are disjoint, so the sum is a gather).  The result must be
the full product, and the owned block sets must partition the partition."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import paper_2205_04752_b200 as hm
    from oracle import oracle as orc

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    mesh = hm.Mesh.icosphere(2)
    a = mesh.arrays()
    N = mesh.num_triangles
    op = hm.HMatrix.kelvin(mesh, b_min=8, eta=1.0, device=-1, shard=(rank, world))
    rb, re = op.row_range
    t = op.tree()
    blocks = op.partition_blocks()
    owned = [b for b, (rn, cn, adm, lvl) in enumerate(blocks)
             if t.nodes[rn, 0] >= rb and t.nodes[rn, 1] <= re]
    ref = orc.Problem.kelvin(a["vertices"], a["triangles"], b_min=8, eta=1.0)
    A = ref.dense_grid()
    x = torch.zeros(3 * N, dtype=torch.float64)
    if rank == 0:
        x = torch.tensor(orc.random_vector(3 * N, 7))
    dist.broadcast(x, src=0)
    xn = x.numpy()
    y = np.zeros(3 * N)
    for b in owned:
        rn, cn = blocks[b, 0], blocks[b, 1]
        rows = t.perm[t.nodes[rn, 0]:t.nodes[rn, 1]]
        cols = t.perm[t.nodes[cn, 0]:t.nodes[cn, 1]]
        for r in range(3):
            for c in range(3):
                y[r * N + rows] += A[np.ix_(r * N + rows, c * N + cols)] @ xn[c * N + cols]
    yt = torch.tensor(y)
    dist.all_reduce(yt)
    owned_t = torch.zeros(len(blocks), dtype=torch.int64)
    owned_t[owned] = 1
    dist.all_reduce(owned_t)
    if rank == 0:
        full = A @ xn
        np.save(os.path.join(outdir, "err.npy"),
                np.array([np.linalg.norm(yt.numpy() - full) / np.linalg.norm(full),
                          float(owned_t.min()), float(owned_t.max())]))
    dist.destroy_process_group()


def test_block_row_shards_gloo(tmp_path):
    world = 2
    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    err, lo, hi = np.load(tmp_path / "err.npy")
    assert lo == 1 and hi == 1  # every block owned by exactly one rank
    assert err < 1e-14


def test_shard_ranges_align_with_blocks():
    import paper_2205_04752_b200 as hm
    mesh = hm.Mesh.icosphere(4)
    for world in (2, 4, 8):
        rows_owned = np.zeros(mesh.num_triangles, dtype=int)
        for r in range(world):
            op = hm.HMatrix.kelvin(mesh, b_min=32, device=-1, shard=(r, world))
            rb, re = op.row_range
            rows_owned[rb:re] += 1
        assert (rows_owned == 1).all()
    with pytest.raises(hm.ConfigError):
        hm.HMatrix.kelvin(hm.Mesh.icosphere(1), b_min=32, device=-1, shard=(0, 8))


def _mark_worker(rank, world, port, outdir, theta):
    """One rank of the sharded marking walk (hmb_mark_sharded): the oracle's
    estimator terms of the blocks on this rank's rows, the whole difference
    vector, the events exchanged over gloo."""
    import paper_2205_04752_b200 as hm
    from paper_2205_04752_b200.dist import torch_transport
    from oracle import oracle as orc

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    mesh = hm.Mesh.ellipsoid(3, 2.0, 1.0, 0.5)
    a = mesh.arrays()
    N = mesh.num_triangles
    o = orc.Problem.kelvin(a["vertices"], a["triangles"], b_min=16, eta=1.0)
    o.assemble(eps=1e-2, beta=0.8, lookahead=2)
    c = a["centroids"]
    bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.1 ** 2))
    x = np.tile(bump, 3) + 1e-3 * orc.random_vector(3 * N, 3)
    gamma, diff, terms = o.gamma(x)
    op = hm.HMatrix.kelvin(mesh, b_min=16, eta=1.0, device=-1, shard=(rank, world))
    rb, re = op.row_range
    t = op.tree()
    blocks = op.partition_blocks()
    own = np.zeros(3 * N, dtype=bool)
    for r in range(3):
        own[r * N + t.perm[rb:re]] = True
    mine = [i for i, term in enumerate(terms)
            if t.nodes[blocks[term["block"], 0], 0] >= rb and
            t.nodes[blocks[term["block"], 0], 1] <= re]
    local = [hm.BlockTerm(terms[i]["comp"], terms[i]["block"], terms[i]["idx"],
                          terms[i]["val"], terms[i]["norm_sq"]) for i in mine]
    _, allgather = torch_transport()
    marked, total, gpk = hm.mark_blocks_sharded(local, diff, own, theta,
                                                op.sparsity_constant, 3 * N, 3 * N, world,
                                                rank, allgather)
    np.save(os.path.join(outdir, f"m{rank}.npy"),
            np.array([[mine[i] for i in marked], total, gpk, len(mine)], dtype=object),
            allow_pickle=True)
    dist.destroy_process_group()


@pytest.mark.parametrize("world,theta", [(2, 0.7), (3, 0.5), (4, 0.9)])
def test_sharded_marking_matches_unsharded_walk(tmp_path, world, theta):
    """hmb_mark_sharded (the marking step of the sharded adaptive matvec) on
    CPU ranks over gloo: the union of the ranks' marked terms, the marked
    count and gamma(P_k) equal the oracle's unsharded mark_blocks bit for bit,
    and every term belongs to exactly one rank."""
    import paper_2205_04752_b200 as hm
    from oracle import oracle as orc

    port = _free_port()
    mp.spawn(_mark_worker, args=(world, port, str(tmp_path), theta), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"m{r}.npy", allow_pickle=True) for r in range(world)]
    mesh = hm.Mesh.ellipsoid(3, 2.0, 1.0, 0.5)
    a = mesh.arrays()
    N = mesh.num_triangles
    o = orc.Problem.kelvin(a["vertices"], a["triangles"], b_min=16, eta=1.0)
    o.assemble(eps=1e-2, beta=0.8, lookahead=2)
    c = a["centroids"]
    bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.1 ** 2))
    x = np.tile(bump, 3) + 1e-3 * orc.random_vector(3 * N, 3)
    _, _, terms = o.gamma(x)
    op = hm.HMatrix.kelvin(mesh, b_min=16, eta=1.0, device=-1)
    ref_marked, ref_gpk = o.mark(theta, op.sparsity_constant, 3 * N, 3 * N, len(terms))
    assert len(ref_marked) > 0
    union = sorted(i for r in range(world) for i in outs[r][0])
    assert union == sorted(ref_marked.tolist())
    assert sum(outs[r][3] for r in range(world)) == len(terms)
    for r in range(world):
        assert outs[r][1] == len(ref_marked)
        assert outs[r][2] == ref_gpk


def test_mark_sharded_argument_errors():
    """hmb_mark_sharded validates its sizes and reports a failing all-gather
    as the library's error (no crash)."""
    import paper_2205_04752_b200 as hm
    term = hm.BlockTerm(0, 0, np.array([0, 2], np.int64), np.array([1.0, -2.0]), 5.0)
    diff = np.array([1.0, 0.0, -2.0])
    with pytest.raises(hm.DimensionError):
        hm.mark_blocks_sharded([term], diff[:2], np.ones(3, bool), 0.7, 1, 3, 3, 1, 0,
                               lambda s, r: None)
    with pytest.raises(hm.DimensionError):
        hm.mark_blocks_sharded([term], diff, np.ones(2, bool), 0.7, 1, 3, 3, 1, 0,
                               lambda s, r: None)

    def broken(s, r):
        raise RuntimeError("transport down")

    with pytest.raises(hm.Error):
        hm.mark_blocks_sharded([term], diff, np.ones(3, bool), 0.7, 1, 3, 3, 2, 0, broken)
    # one rank, a trivial all-gather: the unsharded walk (every term marked
    # once the target needs it)
    marked, total, gpk = hm.mark_blocks_sharded(
        [term], diff, np.ones(3, bool), 0.7, 1, 3, 3, 1, 0,
        lambda s, r: r.__setitem__(slice(None), s))
    assert list(marked) == [0] and total == 1 and gpk == 0.0
    # rank index out of range
    with pytest.raises(hm.Error):
        hm.mark_blocks_sharded([term], diff, np.ones(3, bool), 0.7, 1, 3, 3, 2, 2,
                               lambda s, r: None)


def test_amvm_occurrences_config_errors():
    import paper_2205_04752_b200 as hm
    with pytest.raises(hm.ConfigError):
        hm.amvm_multiply_occurrences([], lambda v: v, np.zeros(3), 3, 3,
                                     hm.AmvmConfig(theta=1.0))
    with pytest.raises(hm.ConfigError):
        hm.amvm_multiply_occurrences([], lambda v: v, np.zeros(3), 3, 3,
                                     hm.AmvmConfig(eps_amvm=0.0))
    with pytest.raises(hm.DimensionError):
        hm.amvm_multiply_occurrences([], lambda v: v, np.zeros(2), 3, 3, hm.AmvmConfig())
    # no H-leaf at all: gamma = 0, the product itself
    b, rep = hm.amvm_multiply_occurrences([], lambda v: 2.0 * v, np.ones(3), 3, 3,
                                          hm.AmvmConfig())
    assert (b == 2.0).all() and rep.converged and rep.iterations[0].gamma == 0.0
