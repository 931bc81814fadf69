"""Multi-RHS sweep for ncu / kernel timing (development helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 16
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0)
h.assemble(eps=eps, beta=0.8)
X = np.asfortranarray(hm.random_vector(h.cols * nrhs, 2, "normal").reshape(nrhs, -1).T)
h.set_profiling(True)
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3  # many: the power-limited steady state
import torch
Xd = torch.tensor(np.ascontiguousarray(X.T), device="cuda")  # column-major (dofs x nrhs)
Yd = torch.empty_like(Xd)
for it in range(iters):
    if iters > 3:
        h.matvec_ptr(Xd.data_ptr(), Yd.data_ptr(), nrhs)
    else:
        Y = h.matvec(X)
torch.cuda.synchronize()
if iters > 3:
    Y = Yd.cpu().numpy().T
names = ["gather", "hmv16_z", "hmv16_leaf", "pack16"]
for k in names:
    ms, n = h.kernel_times(k, reset=True)
    print(f"{k:12s} {ms / max(n, 1) * 1:.3f} ms/launch  ({n} launches)")
y0 = h.matvec(np.ascontiguousarray(X[:, 0]))
err = np.linalg.norm(Y[:, 0] - y0) / np.linalg.norm(y0)
print(f"col 0 vs 1-RHS sweep: rel {err:.2e}")
assert err < 1e-12
print("ok")
