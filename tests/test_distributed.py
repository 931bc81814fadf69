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
