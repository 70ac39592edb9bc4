// TEST INFRASTRUCTURE ONLY.  Link stubs for the two H-matrix entry points
// assembly.cpp references from bem_h / radiation_h (assembly.cpp:322-351).
// The H-matrix engine (hmatrix.cpp) is outside the pinned path and needs
// LU/QR/SVD that the Eigen-API shim does not provide; nothing in oracle/_ref
// calls these.
#include <stdexcept>

#include "galerk/hmatrix.hpp"

namespace galerk {

std::shared_ptr<const ClusterTree> ClusterTree::build(const MatX3&, int) {
  throw std::logic_error("oracle/_ref: the H-matrix engine is not built (out of the pinned path)");
}

HMatrix HMatrix::assemble(const BlockEvaluator&, std::shared_ptr<const ClusterTree>,
                          std::shared_ptr<const ClusterTree>, const HParams&) {
  throw std::logic_error("oracle/_ref: the H-matrix engine is not built (out of the pinned path)");
}

}  // namespace galerk
