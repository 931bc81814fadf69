"""Quick GPU probe: smoke + config-2 timings (development helper)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import __graft_entry__ as g
import paper_2205_04752_b200 as hm
from oracle import oracle as orc

g.smoke()
level = int(sys.argv[1]) if len(sys.argv) > 1 else 5
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
mesh = hm.Mesh.icosphere(level)
h = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
h.set_profiling(True)
t0 = time.time()
st = h.assemble(eps=eps, beta=0.8)
print("assemble wall s", time.time() - t0, st)
for k in ("nearfield", "aca", "compact", "relocate"):
    print(k, h.kernel_times(k, reset=True))
print("storage", h.storage())
x = orc.random_vector(h.cols, 1)
for it in range(5):
    y = h.matvec(x)
for k in ("gather", "hmv_stream", "hmv_ypart", "hmv_blocks", "hmv_reduce", "pack"):
    ms, n = h.kernel_times(k, reset=True)
    print(k, ms / max(n, 1), "ms/launch", n)
kc, kl, co, ls = h.ranks()
print("rank max", kl.max(), "mean", kc[kc >= 0].mean())
