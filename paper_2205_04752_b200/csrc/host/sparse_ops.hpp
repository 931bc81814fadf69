// The fixed sparse transforms of the Galerkin BEM operators
// (build_sparse_ops, proj/src/operators.cpp:7-95): T(k,l) = n_l d_k - n_k d_l
// applied to the nodal hat functions (constant per triangle) and the
// triangle x node mass pairing, in ELL form -- every triangle row holds its
// three vertices (slot a = local vertex a), value 0 where the reference
// drops the entry.  Composed into K_h and D_h by the package
// (compose_Kh / compose_Dh, operators.cpp:107-158).
#pragma once

#include <vector>

#include "geometry.hpp"

namespace hmb {

struct Ell3 {
  int rows = 0, cols = 0;
  std::vector<int> col;     // rows x 3
  std::vector<double> val;  // rows x 3
};

// T(k, l), 0-based component indices k < l (build_t_matrix, operators.cpp:16-33)
Ell3 build_t_matrix(const Mesh& mesh, int k, int l);
// mass: area / 3 per (triangle, vertex) (operators.cpp:82-88)
Ell3 build_mass_matrix(const Mesh& mesh);

}  // namespace hmb
