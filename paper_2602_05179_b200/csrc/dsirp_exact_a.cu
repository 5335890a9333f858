// dsirp_exact_a.cu -- K3 instantiations with HMAX == H for H = 1..4 (own
// translation unit so the fully unrolled kernels compile in parallel).
#include "common.cuh"
#include "internal.hpp"
#include "dsirp_kernels.cuh"

namespace scendp_dsirp {
bool launch_exact_a(scendp_ctx* c, const DsirpArgs& a, size_t s, bool i, bool f) {
  const int H = a.H;
  if (H == 1) return launch_h<1>(c, a, s, i, f), true;
  if (H == 2) return launch_h<2>(c, a, s, i, f), true;
  if (H == 3) return launch_h<3>(c, a, s, i, f), true;
  if (H == 4) return launch_h<4>(c, a, s, i, f), true;
  return false;
}
}  // namespace scendp_dsirp
