"""A/B helper: warm assembly of a config with the library in HMGPU_LIB_DIR;
prints device times and a digest of the ranks and one matvec (the digest must
not change between variants: the ACA is bit-exact).  Development helper."""
import hashlib, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
elif cfg == "c1":
    mesh, bmin, eps = hm.Mesh.icosphere(3), 32, 1e-4
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0)
ts, ka = [], []
h.set_profiling(True)
for r in range(reps):
    t = time.perf_counter()
    h.kernel_times("aca", reset=True)
    st = h.assemble(eps=eps, beta=0.8)
    ka.append(h.kernel_times("aca", reset=True)[0])
    ts.append(st.ms_total)
    print(f"{cfg} run {r}: wall {1e3*(time.perf_counter()-t):.1f} ms  ms={st.ms_total:.2f} "
          f"near={st.ms_nearfield:.3f} entries={st.aca_entries}", flush=True)
w = sorted(ts[1:] or ts)
k = sorted(ka[1:] or ka)
print(f"{cfg} summary: min {w[0]:.2f} median {w[len(w)//2]:.2f} ms (warm runs); "
      f"aca kernel min {k[0]:.2f} median {k[len(k)//2]:.2f} ms", flush=True)
x = np.random.default_rng(1).uniform(-1, 1, h.cols)
y = h.matvec(x)
print(cfg, "digest", hashlib.sha1(np.ascontiguousarray(y).tobytes()).hexdigest()[:16],
      "pivots", st.pivots, flush=True)
