import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
from oracle import oracle as orc
mesh = hm.Mesh.voxel_cube(128, 0.0, 1.0)
h = hm.HMatrix.kelvin(mesh, b_min=64, eta=1.0, device=0)
h.set_profiling(True)
t0 = time.time()
st = h.assemble(eps=1e-5, beta=0.8)
print("C3 assemble wall s", time.time() - t0, st, flush=True)
for k in ("nearfield", "aca", "compact", "relocate"):
    print(k, h.kernel_times(k, reset=True))
print("storage", h.storage(), flush=True)
x = orc.normal_vector(h.cols, 2)
for it in range(3):
    y = h.matvec(x)
for k in ("gather", "hmv_stream", "hmv_ypart", "hmv_blocks", "hmv_reduce", "pack"):
    ms, n = h.kernel_times(k, reset=True)
    print(k, ms / max(n, 1), "ms/launch", n)
