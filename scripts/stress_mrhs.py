"""Repeat the 16-RHS product and require bit-identical results every time
(the dynamic hand-out of work units must not change what is summed in which
order); development helper.  argv: config (c2 | c3), repetitions."""
import os, sys, hashlib
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_04752_b200 as hm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 100
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0)
h.assemble(eps=eps, beta=0.8)
nrhs = 16
X = hm.random_vector(h.cols * nrhs, 2, "normal").reshape(nrhs, -1)
Xd = torch.tensor(X, device="cuda")
Yd = torch.empty((nrhs, h.rows), dtype=torch.float64, device="cuda")
ref = None
for r in range(reps):
    Yd.zero_()
    h.matvec_ptr(Xd.data_ptr(), Yd.data_ptr(), nrhs)
    torch.cuda.synchronize()
    if ref is None:
        ref = Yd.clone()
        y0 = h.matvec(np.ascontiguousarray(X[0]))
        err = np.linalg.norm(ref[0].cpu().numpy() - y0) / np.linalg.norm(y0)
        assert err < 1e-12, err
    else:
        assert torch.equal(Yd, ref), f"run {r} differs from run 0"
print(f"{cfg}: {reps} 16-RHS products bit-identical, digest "
      f"{hashlib.sha1(ref.cpu().numpy().tobytes()).hexdigest()[:16]}")
