"""Galerkin V_kl / V_Delta / K_Delta assembly times on an icosphere
(development helper; argv: level, reps)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04752_b200 as hm
lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 5
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
mesh = hm.Mesh.icosphere(lvl)
for name, mk in (("vkl", lambda: hm.HMatrix.galerkin(mesh, 0, 32, 1.0, 0)),
                 ("vdelta", lambda: hm.HMatrix.galerkin(mesh, 1, 32, 1.0, 0)),
                 ("kdelta", lambda: hm.HMatrix.kdelta(mesh, 32, 1.0, 0))):
    h = mk()
    h.set_profiling(True)
    for r in range(reps):
        for k in ("aca", "nearfield", "compact"):
            h.kernel_times(k, reset=True)
        st = h.assemble(eps=1e-6, beta=0.8)
        kt = {k: round(h.kernel_times(k, reset=True)[0], 2) for k in ("aca", "nearfield", "compact")}
        print(f"{name} L{lvl} run {r}: ms={st.ms_total:.1f} {kt} entries={st.aca_entries}+{st.dense_entries} pivots={st.pivots}", flush=True)
