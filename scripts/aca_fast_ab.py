"""Price of the bit-exact entry contract (development helper): warm assembly
of a config with the library in HMGPU_LIB_DIR (the canonical build or the
HMGPU_FAST_ENTRY / --fmad=true variant of scripts/build_variant.sh); dumps
ACA kernel time, ranks and one matvec to an npz; `compare a.npz b.npz`
prints the time ratio, max rank difference and matvec difference.
usage: aca_fast_ab.py dump <c2|c3> <out.npz> | compare <a.npz> <b.npz>"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

if sys.argv[1] == "compare":
    a, b = np.load(sys.argv[2]), np.load(sys.argv[3])
    adm = a["kc"] >= 0
    dk = np.abs(a["kc"][adm] - b["kc"][adm])
    dl = np.abs(a["kl"][adm] - b["kl"][adm])
    rel = np.linalg.norm(a["y"] - b["y"]) / np.linalg.norm(a["y"])
    print(f"aca kernel {a['aca_ms']:.2f} -> {b['aca_ms']:.2f} ms "
          f"(x{a['aca_ms'] / b['aca_ms']:.3f}), assembly {a['asm_ms']:.2f} -> "
          f"{b['asm_ms']:.2f} ms; ranks: max |dk| {dk.max()} (|dk|>0 on {np.mean(dk > 0):.2%}),"
          f" max |dK| {dl.max()}; pivots {a['pivots']} -> {b['pivots']}; "
          f"matvec rel diff {rel:.3e}")
    sys.exit(0)
import paper_2205_04752_b200 as hm
cfg, out = sys.argv[2], sys.argv[3]
if cfg == "c2":
    mesh, bmin, eps = hm.Mesh.icosphere(5), 32, 1e-6
else:
    mesh, bmin, eps = hm.Mesh.voxel_cube(128, 0.0, 1.0), 64, 1e-5
h = hm.HMatrix.kelvin(mesh, b_min=bmin, eta=1.0, device=0)
h.set_profiling(True)
ka, ta = [], []
for r in range(3):
    h.kernel_times("aca", reset=True)
    st = h.assemble(eps=eps, beta=0.8, lookahead=2)
    ka.append(h.kernel_times("aca", reset=True)[0])
    ta.append(st.ms_total)
kc, kl, _, _ = h.ranks()
x = hm.random_vector(h.cols, 1)
np.savez(out, aca_ms=min(ka[1:]), asm_ms=min(ta[1:]), kc=kc, kl=kl, y=h.matvec(x),
         pivots=st.pivots)
print(cfg, "aca", min(ka[1:]), "assembly", min(ta[1:]))
