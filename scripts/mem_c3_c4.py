"""Diagnostics: device memory left by a resident config-3 H-matrix, then the
config-4 adaptive matvec (HMGPU_VERBOSE=1 logs the arena growth)."""
import os
import sys
import ctypes

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2205_04752_b200 as hm

cudart = ctypes.CDLL("libcudart.so") if False else None


def meminfo(tag):
    import torch
    f, t = torch.cuda.mem_get_info(0)
    print(f"[mem] {tag}: free {f / 1e9:.1f} GB of {t / 1e9:.1f} GB", flush=True)


meminfo("start")
keep = None
if "--no-c3" not in sys.argv:
    mesh3 = hm.Mesh.voxel_cube(128, 0.0, 1.0)
    keep = hm.HMatrix.kelvin(mesh3, b_min=64, eta=1.0, device=0)
    keep.assemble(eps=1e-5, beta=0.8, lookahead=2)
    meminfo("c3 assembled")
    keep.matvec(hm.random_vector(keep.cols, 1))
    meminfo("c3 after matvec")
mesh = hm.Mesh.ellipsoid(6, 2.0, 1.0, 0.5)
a = mesh.arrays()
g = hm.HMatrix.kelvin(mesh, b_min=32, eta=1.0, device=0)
g.assemble(eps=1e-2, beta=0.8, lookahead=2)
meminfo("c4 assembled")
c = a["centroids"]
bump = np.exp(-np.sum((c - np.array([2.0, 0, 0])) ** 2, axis=1) / (2 * 0.05 ** 2))
x = np.tile(bump, 3) + 1e-3 * hm.random_vector(3 * len(c), 3)
bg, rep = g.amvm_multiply(x, theta=0.7, eps_amvm=1e-6, max_iterations=5)
meminfo("c4 amvm done")
print([(r.gamma, r.marked) for r in rep.iterations])
