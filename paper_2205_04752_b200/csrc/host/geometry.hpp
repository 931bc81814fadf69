// Surface meshes for the collocation BEM: geometry caches, synthetic mesh
// generators for the BASELINE configs, OFF input.
//
// Mirrors the reference's SurfaceMesh (proj/include/hmbem/mesh.hpp:15-40):
// centroids/areas/normals as computed by load_mesh (proj/src/mesh.cpp:229-247)
// and the longest-edge diameter (mesh.cpp:105-109).  The generators are new
// (the reference ships no icosphere/ellipsoid); the voxel
// cube follows meshgen's voxel_surface (proj/tools/meshgen.cpp:27-83).
#pragma once

#include <array>
#include <string>
#include <vector>

namespace hmb {

using Real = double;
using V3 = std::array<Real, 3>;

struct Mesh {
  std::vector<V3> vertices;
  std::vector<std::array<int, 3>> triangles;
  std::vector<char> dirichlet;  // per-triangle D/N flag (may be empty)
  // geometry caches (filled by finish())
  std::vector<V3> centroids, normals;
  std::vector<Real> areas, diam;

  int nv() const { return static_cast<int>(vertices.size()); }
  int nt() const { return static_cast<int>(triangles.size()); }
  const V3& corner(int t, int k) const { return vertices[triangles[t][k]]; }

  // computes the caches; throws on degenerate triangles (mesh.cpp:233-244)
  void finish();
  // closed + consistently oriented + no duplicated faces (mesh.cpp:68-101)
  void validate_admissible() const;
  // centroid predicate "x3<=0|x1>=1" (mesh.cpp:29-66, 171-178)
  void label_dirichlet(const std::string& predicate);
};

// unit-sphere icosphere: icosahedron refined `level` times by edge midpoints
// projected to the sphere, outward winding (20 * 4^level triangles)
Mesh make_icosphere(int level);
// icosphere scaled by the semi-axes
Mesh make_ellipsoid(int level, Real ax, Real ay, Real az);
// voxel cube surface on [lo,hi]^3 with n cells per edge (meshgen.cpp:27-83)
Mesh make_voxel_cube(int n, Real lo, Real hi);

Mesh load_off(const std::string& path);
void save_off(const Mesh& m, const std::string& path);

}  // namespace hmb
