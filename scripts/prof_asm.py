"""Assembly for ncu (development helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04752_b200 as hm
mesh = hm.Mesh.icosphere(int(sys.argv[1]) if len(sys.argv) > 1 else 5)
h = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
st = h.assemble(eps=1e-6, beta=0.8)
print("ok", st)
