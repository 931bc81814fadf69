"""The library's distributed matvec (hmgpu_matvec_dist) with
world 2 and 4 on the one visible GPU: each rank is a process with its own
context holding its block-row shard (hmgpu_set_partition row range), the
transport is the host-callback one over torch.distributed gloo (the
collectives run on the host, so no rank's kernel waits on another rank's
kernel).  Every rank must return the whole product; each rank's own rows
must equal its local shard sweep bit for bit (the gather is a copy), all
ranks must hold identical y, and y must match the unsharded operator."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, outdir):
    import torch.distributed as dist
    import paper_2205_04752_b200 as hm
    from paper_2205_04752_b200.dist import torch_transport
    from oracle import oracle as orc

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    mesh = hm.Mesh.icosphere(3)
    n = 3 * mesh.num_triangles
    h = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0, shard=(rank, world))
    h.assemble(eps=1e-4, beta=0.8, lookahead=2)
    h.attach_comm(world, rank, *torch_transport())
    info = h.comm_info()
    out = {"tiles": bool(info["row_begin"][0] == 0 and
                         (info["row_begin"][1:] == info["row_end"][:-1]).all() and
                         info["row_end"][-1] == mesh.num_triangles),
           "kind": info["kind"]}
    rb, re = h.row_range
    t = h.tree()
    own = np.zeros(mesh.num_triangles, dtype=bool)
    own[t.perm[rb:re]] = True
    own = np.tile(own, 3)
    res = []
    for nrhs, mode in ((1, hm.Mode.Current), (1, hm.Mode.Lookahead), (3, hm.Mode.Current),
                       (16, hm.Mode.Current)):
        X = np.stack([orc.random_vector(n, 5 + s) for s in range(nrhs)], axis=1)
        X = X[:, 0] if nrhs == 1 else np.asfortranarray(X)
        y = h.matvec_dist(X if rank == 0 else None, mode, nrhs)
        y_loc = h.matvec(X, mode)  # this shard's sweep, external order
        own_ok = bool((y[own] == y_loc[own]).all())
        res.append((nrhs, int(mode), y, own_ok))
    np.save(os.path.join(outdir, f"r{rank}.npy"),
            np.array([out, [(a, b, yy, ok) for a, b, yy, ok in res]], dtype=object),
            allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_matvec_dist_world_on_one_gpu(tmp_path, world):
    import torch.multiprocessing as mp
    import paper_2205_04752_b200 as hm
    from oracle import oracle as orc

    port = _free_port()
    mp.spawn(_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"r{r}.npy", allow_pickle=True) for r in range(world)]
    mesh = hm.Mesh.icosphere(3)
    n = 3 * mesh.num_triangles
    full = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
    full.assemble(eps=1e-4, beta=0.8, lookahead=2)
    for r in range(world):
        assert outs[r][0]["tiles"] and outs[r][0]["kind"] == "host"
    for case in range(4):
        nrhs, mode = outs[0][1][case][0], outs[0][1][case][1]
        y0 = outs[0][1][case][2]
        for r in range(world):
            assert outs[r][1][case][3], (r, nrhs, mode)           # own rows bitwise
            assert (outs[r][1][case][2] == y0).all(), (r, nrhs)     # identical on all ranks
        X = np.stack([orc.random_vector(n, 5 + s) for s in range(nrhs)], axis=1)
        X = X[:, 0] if nrhs == 1 else np.asfortranarray(X)
        yf = full.matvec(X, hm.Mode(mode))
        assert np.linalg.norm(y0 - yf) <= 1e-14 * np.linalg.norm(yf), (nrhs, mode)


def test_matvec_dist_requires_a_communicator():
    import paper_2205_04752_b200 as hm
    h = hm.HMatrix.kelvin(hm.Mesh.icosphere(2), b_min=16, device=0)
    h.assemble(eps=1e-4)
    with pytest.raises(hm.DeviceError):
        h.matvec_dist(np.zeros(h.cols))


def test_matvec_dist_single_rank_nccl():
    """world 1 through the library's own NCCL communicator (the transport
    the multi-GPU bench uses): the product equals the plain matvec bitwise."""
    import paper_2205_04752_b200 as hm
    from oracle import oracle as orc
    ok, ver = hm.nccl_available()
    if not ok:
        pytest.skip("libnccl not loadable")
    h = hm.HMatrix.kelvin(hm.Mesh.icosphere(3), b_min=32, device=0)
    h.assemble(eps=1e-4)
    h.attach_nccl(1, 0, hm.nccl_unique_id())
    assert h.comm_info()["kind"] == "nccl"
    x = orc.random_vector(h.cols, 3)
    assert (h.matvec_dist(x) == h.matvec(x)).all()


def _amvm_worker(rank, world, port, outdir):
    import torch.distributed as dist
    import paper_2205_04752_b200 as hm
    from paper_2205_04752_b200.dist import torch_transport

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    mesh, x = _amvm_case()
    h = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0, shard=(rank, world))
    h.assemble(eps=1e-2, beta=0.8, lookahead=2)
    h.attach_comm(world, rank, *torch_transport())
    b, rep = h.amvm_multiply(x, theta=0.7, eps_amvm=1e-6, max_iterations=5)
    gk, gl, _, _ = h.ranks()
    np.save(os.path.join(outdir, f"a{rank}.npy"),
            np.array([b, [(r.gamma, r.gamma_pk, r.marked, r.cumulative_pivots, r.storage_mb,
                           r.e_hat) for r in rep.iterations], gk, gl], dtype=object),
            allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def _amvm_case():
    import paper_2205_04752_b200 as hm
    mesh = hm.Mesh.ellipsoid(4, 2.0, 1.0, 0.5)
    c = mesh.arrays()["centroids"]
    bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.05 ** 2))
    x = np.tile(bump, 3) + 1e-3 * hm.random_vector(3 * len(c), 3)
    return mesh, x


@pytest.mark.parametrize("world", [2, 3])
def test_amvm_sharded_world_on_one_gpu(tmp_path, world):
    """The adaptive matvec on block-row shards: the ranks
    exchange the estimator's difference vector and the marking events; the
    record (gamma, marked count, cumulative pivots of every sweep) must be
    the unsharded operator's, bit for bit, every block's ranks after the
    loop the unsharded ones, and b the same product."""
    import torch.multiprocessing as mp
    import paper_2205_04752_b200 as hm

    port = _free_port()
    mp.spawn(_amvm_worker, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    outs = [np.load(tmp_path / f"a{r}.npy", allow_pickle=True) for r in range(world)]
    mesh, x = _amvm_case()
    full = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
    full.assemble(eps=1e-2, beta=0.8, lookahead=2)
    bf, rep = full.amvm_multiply(x, theta=0.7, eps_amvm=1e-6, max_iterations=5)
    fk, fl, _, _ = full.ranks()
    its = [(r.gamma, r.gamma_pk, r.marked, r.cumulative_pivots, r.storage_mb)
           for r in rep.iterations]
    assert sum(r.marked for r in rep.iterations) > 0
    for r in range(world):
        b, rit, gk, gl = outs[r]
        assert len(rit) == len(its)
        for a, e in zip(rit, its):
            assert a[0] == e[0] and a[2] == e[2] and a[3] == e[3], (r, a, e)
            assert a[1] == pytest.approx(e[1], rel=1e-12)
            assert a[4] == pytest.approx(e[4], rel=1e-12)
        assert np.linalg.norm(b - bf) <= 1e-13 * np.linalg.norm(bf)
        own = gk >= 0
        assert (gk[own] == fk[own]).all() and (gl[own] == fl[own]).all()
    # every low-rank (comp, block) is owned by exactly one rank
    owned = sum((outs[r][2] >= 0).astype(int) for r in range(world))
    assert (owned[fk >= 0] == 1).all()
