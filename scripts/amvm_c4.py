"""Config 4 adaptive matvec timing (development helper)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm
mesh = hm.Mesh.ellipsoid(6, 2.0, 1.0, 0.5)
a = mesh.arrays()
g = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
t = time.perf_counter()
st = g.assemble(eps=1e-2, beta=0.8, lookahead=2)
print("assemble", time.perf_counter() - t, st)
c = a["centroids"]
bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.05 ** 2))
x = np.tile(bump, 3) + 1e-3 * hm.random_vector(3 * len(c), 3)
for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    g.assemble(eps=1e-2, beta=0.8, lookahead=2)
    t = time.perf_counter()
    b, r = g.amvm_multiply(x, theta=0.7, eps_amvm=1e-6, max_iterations=5)
    print("amvm", time.perf_counter() - t, r.termination, len(r.iterations))
    for it in r.iterations:
        print("  ", it)
