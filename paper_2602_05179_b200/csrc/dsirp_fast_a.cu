// dsirp_fast_a.cu -- K3 fast-form instantiations for H = 1..4 (own
// translation unit so the fully unrolled kernels compile in parallel).
#include "common.cuh"
#include "internal.hpp"
#include "dsirp_kernels.cuh"

namespace scendp_dsirp {
bool launch_fast_a(scendp_ctx* c, const DsirpArgs& a, size_t s, bool i, bool f) {
  switch (a.H) {
    case 1: return launch_fast_h<1>(c, a, s, i, f), true;
    case 2: return launch_fast_h<2>(c, a, s, i, f), true;
    case 3: return launch_fast_h<3>(c, a, s, i, f), true;
    case 4: return launch_fast_h<4>(c, a, s, i, f), true;
    default: return false;
  }
}
}  // namespace scendp_dsirp
