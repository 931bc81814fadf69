"""Shared fixtures for the parity tests (meshes, the reference's test
fixtures restated: make_cube_mesh, CentroidKernelOracle points)."""
import numpy as np

import paper_2205_04752_b200 as hm


def cube_mesh(n: int) -> hm.Mesh:
    """test::make_cube_mesh(n): voxel cube on [-1,1]^3 (oracles.cpp:113-119)."""
    return hm.Mesh.voxel_cube(n, -1.0, 1.0)


def centroid_points_and_boxes(mesh: hm.Mesh):
    """Centroids with triangle-corner support boxes (test_hmatrix.cpp:36-43)."""
    a = mesh.arrays()
    v, t = a["vertices"], a["triangles"]
    corners = v[t]  # nt x 3 x 3
    boxes = np.concatenate([corners.min(axis=1), corners.max(axis=1)], axis=1)
    return a["centroids"], boxes


def separated_kernel_matrix(m, n, seed, rv):
    """two separated clouds, Newton kernel (test_aca.cpp:16-27)."""
    rx = rv(3 * m, seed)
    ry = rv(3 * n, seed + 1)
    x = rx.reshape(m, 3)
    y = ry.reshape(n, 3) + np.array([8.0, 0.0, 0.0])
    a = np.zeros((m, n))
    for i in range(m):
        for j in range(n):
            d = x[i] - y[j]
            a[i, j] = 1.0 / np.sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2])
    return a, x, y


def doctest_approx(got: float, want: float, eps: float) -> bool:
    """doctest::Approx(want).epsilon(eps) == got: |got - want| <
    eps * (scale + max(|got|, |want|)) with the default scale 1 (the
    comparison the reference's test suite uses)."""
    return abs(got - want) < eps * (1.0 + max(abs(got), abs(want)))
