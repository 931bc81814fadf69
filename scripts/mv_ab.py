"""A/B of the 1-RHS matvec (device time per matvec, CUDA events on the
library stream) and a digest of y (development helper; argv: config, reps)."""
import hashlib, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2205_04752_b200 as hm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0)
h.assemble(eps=eps, beta=0.8)
x = torch.tensor(hm.random_vector(h.cols, 1, "uniform"), device="cuda")
y = torch.zeros(h.rows, dtype=torch.float64, device="cuda")
st = torch.cuda.ExternalStream(h.stream())
for _ in range(5):
    h.matvec_ptr(x.data_ptr(), y.data_ptr(), 1)
torch.cuda.synchronize()
best = []
for r in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        e0.record(st)
        for _ in range(reps):
            h.matvec_ptr(x.data_ptr(), y.data_ptr(), 1)
        e1.record(st)
    torch.cuda.synchronize()
    best.append(e0.elapsed_time(e1) / reps)
print(f"{cfg} matvec ms min {min(best):.4f} all {[round(b, 4) for b in best]} "
      f"digest {hashlib.sha1(y.cpu().numpy().tobytes()).hexdigest()[:16]}", flush=True)
