// TEST INFRASTRUCTURE ONLY (oracle/_ref build shim).
//
// Stand-in for /root/reference/proj/include/diffsim/svd3.hpp, whose only
// dependency is Eigen 3 (absent from this image).  The reference reaches it
// through the quoted include at tape.hpp:453; putting this directory first
// on the include path lets every other reference header compile unchanged.
// The two entry points keep the reference signatures (tape.hpp:55-57) and
// forward to the self-written restatement in oracle/svd3x3.hpp.
#pragma once

#include "oracle/svd3x3.hpp"

namespace diffsim::detail {

inline void svd3x3_values(const double f[9], double u[9], double s[3], double vt[9]) {
  oracle::svd3x3_values(f, u, s, vt);
}

inline void svd3x3_adjoint(const double u[9], const double s[3], const double vt[9],
                           const double out_adj[21], double f_adj[9]) {
  oracle::svd3x3_adjoint(u, s, vt, out_adj, f_adj);
}

}  // namespace diffsim::detail
