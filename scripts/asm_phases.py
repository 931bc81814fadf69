"""Warm assembly phase timings (HMGPU_VERBOSE=1) for a config (development helper)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04752_b200 as hm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0)
for r in range(3):
    t = time.perf_counter()
    st = h.assemble(eps=eps, beta=0.8)
    print(f"run {r}: wall {1e3*(time.perf_counter()-t):.1f} ms", st, flush=True)
