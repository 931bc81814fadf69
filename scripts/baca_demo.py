"""Reduced-mode BACA (V_h t = f, all-Dirichlet) on an icosphere: iteration
record (development helper; argv: level, eps_aca, eps_baca)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
lvl = int(sys.argv[1]) if len(sys.argv) > 1 else 4
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-2
eb = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-6
mesh = hm.Mesh.icosphere(lvl)
t = time.perf_counter()
ops = hm.OperatorSet(mesh, 1.0, 0.3, b_min=32, eta=1.0, device=0)
st = ops.assemble(eps=eps, beta=0.8, lookahead=2)
print(f"L{lvl}: {mesh.num_triangles} triangles, assembly {1e3*(time.perf_counter()-t):.0f} ms "
      f"(device {sum(s.ms_total for s in st):.0f} ms)", flush=True)
f = hm.random_vector(3 * mesh.num_triangles, 7)
t = time.perf_counter()
x, rep = hm.baca_solve(ops, f, hm.BacaConfig(eps_baca=eb))
print(f"baca: {rep.termination} after {len(rep.iterations)} sweeps, {time.perf_counter()-t:.2f} s")
for it in rep.iterations:
    print(f"  k={it.k} E_k={it.ek:.3e} tail={it.tail_norm:.3e} res={it.residual:.3e} "
          f"inner={it.inner_iterations} marked={it.marked_v} MB={it.storage_mb:.1f} t={it.wall_time_s:.2f}s")
print("residual vs current V_h:", np.linalg.norm(ops.vh(x) - f) / np.linalg.norm(f))
