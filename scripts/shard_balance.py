"""Per-shard matvec bytes (block-row shards) for a config: load balance of
the multi-GPU split, measured shard by shard on one device (development
helper; argv: config c2|c3, world sizes...)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
worlds = [int(w) for w in sys.argv[2:]] or [2, 4, 8]
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
for w in worlds:
    by, rows = [], []
    for r in range(w):
        h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0, shard=(r, w))
        h.assemble(eps=eps, beta=0.8)
        by.append(h.storage()["matvec_bytes"])
        rows.append(h.shard_rows() if hasattr(h, "shard_rows") else 0)
        del h
    by = np.array(by, dtype=float)
    print(f"{cfg} world {w}: bytes/shard GB {np.round(by / 1e9, 3).tolist()} "
          f"max/mean {by.max() / by.mean():.3f}", flush=True)
