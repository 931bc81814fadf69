"""C3 matvec loop for ncu (development helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_04752_b200 as hm
mesh = hm.Mesh.voxel_cube(int(sys.argv[1]) if len(sys.argv) > 1 else 128, 0.0, 1.0)
h = hm.HMatrix.kelvin(mesh, b_min=64, eta=1.0, device=0)
h.assemble(eps=1e-5, beta=0.8)
x = hm.random_vector(h.cols, 2, "normal")
for it in range(3):
    y = h.matvec(x)
print("ok")
