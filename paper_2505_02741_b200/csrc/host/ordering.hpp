// ordering.hpp -- fill-reducing ordering for the exact Laplacian solves of
// the spectral stack (spectral.cu GroundedChol): nested dissection by
// breadth-first level-set separators (George's nested dissection with a
// pseudo-peripheral root per piece). No reference counterpart: the
// reference factorises with Eigen's SimplicialLDLT / AMD (laplacian.cpp:
// 57-85); any symmetric permutation gives the same factorisation up to
// rounding, so this only decides fill and time.
#pragma once

#include <vector>

namespace dyg {

// Symmetric CSR pattern of an m x m matrix (diagonal entries may be
// present; they are ignored). Returns p with p[new] = old (B = A(p, p)).
std::vector<int> nested_dissection_order(int m, const int* row_ptr, const int* cols);

}  // namespace dyg
