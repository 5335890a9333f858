// dsirp_fast_b.cu -- K3 fast-form instantiations for H = 5..8 (own
// translation unit so the fully unrolled kernels compile in parallel).
#include "common.cuh"
#include "internal.hpp"
#include "dsirp_kernels.cuh"

namespace scendp_dsirp {
bool launch_fast_a(scendp_ctx*, const DsirpArgs&, size_t, bool, bool);  // dsirp_fast_a.cu

bool launch_fast(scendp_ctx* c, const DsirpArgs& a, size_t s, bool i, bool f) {
  switch (a.H) {
    case 5: return launch_fast_h<5>(c, a, s, i, f), true;
    case 6: return launch_fast_h<6>(c, a, s, i, f), true;
    case 7: return launch_fast_h<7>(c, a, s, i, f), true;
    case 8: return launch_fast_h<8>(c, a, s, i, f), true;
    default: return launch_fast_a(c, a, s, i, f);
  }
}
}  // namespace scendp_dsirp
