"""Config 5 block-row shard r of G on one GPU (development helper): the
per-GPU share of the 1,310,720-triangle icosphere at G-way sharding."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
r, G = int(sys.argv[1]), int(sys.argv[2])
nrhs = int(sys.argv[3]) if len(sys.argv) > 3 else 16
t = time.perf_counter()
mesh = hm.Mesh.icosphere(8)
print("mesh", mesh.num_triangles, round(time.perf_counter() - t, 1), "s", flush=True)
t = time.perf_counter()
h = hm.HMatrix.kelvin(mesh, b_min=64, eta=1.0, device=0, shard=(r, G))
print("tree+partition", round(time.perf_counter() - t, 1), "s rows", h.row_range, flush=True)
t = time.perf_counter()
st = h.assemble(eps=1e-5, beta=0.8)
print("assemble", round(time.perf_counter() - t, 1), "s", st, flush=True)
s = h.storage()
print("storage MB", round(s["mb_current"]), "matvec GB", s["matvec_bytes"] / 1e9, flush=True)
X = np.asfortranarray(hm.random_vector(h.cols * nrhs, 4, "normal").reshape(nrhs, -1).T)
h.set_profiling(True)
for it in range(3):
    t = time.perf_counter()
    Y = h.matvec(X)
    print("matvec", nrhs, "rhs", round((time.perf_counter() - t) * 1e3, 1), "ms", flush=True)
for k in ("gather", "hmv16_z", "hmv16_leaf", "pack16"):
    ms, n = h.kernel_times(k, reset=True)
    print(f"  {k:12s} {ms / max(n, 1):.3f} ms/launch")
x = np.ascontiguousarray(X[:, 0])
for it in range(3):
    t = time.perf_counter()
    y = h.matvec(x)
    print("matvec 1 rhs", round((time.perf_counter() - t) * 1e3, 1), "ms", flush=True)
