"""Assembly + first matvec (config 2's 'assembly plus one matvec'), the
plan build and the direct (plan-free) sweep (development helper)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0)
x = hm.random_vector(h.cols, 1)
for rep in range(3):
    t0 = time.perf_counter()
    st = h.assemble(eps=eps, beta=0.8, lookahead=2)
    t1 = time.perf_counter()
    y = h.matvec(x)
    t2 = time.perf_counter()
    y2 = h.matvec(x)
    t3 = time.perf_counter()
    print(f"{cfg} rep {rep}: assemble {1e3*(t1-t0):.1f} ms (stats {st.ms_total:.1f}), first matvec "
          f"{1e3*(t2-t1):.1f} ms, second {1e3*(t3-t2):.2f} ms", flush=True)
h.set_matvec_policy(True)
for rep in range(3):
    t0 = time.perf_counter()
    yd = h.matvec(x)
    t1 = time.perf_counter()
    print(f"{cfg} direct matvec {1e3*(t1-t0):.2f} ms  rel diff {np.linalg.norm(yd-y)/np.linalg.norm(y):.2e}", flush=True)
