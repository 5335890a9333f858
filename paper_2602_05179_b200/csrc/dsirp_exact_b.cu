// dsirp_exact_b.cu -- K3 instantiations with HMAX == H for H = 5..8 (own
// translation unit so the fully unrolled kernels compile in parallel).
#include "common.cuh"
#include "internal.hpp"
#include "dsirp_kernels.cuh"

namespace scendp_dsirp {
bool launch_exact_b(scendp_ctx* c, const DsirpArgs& a, size_t s, bool i, bool f) {
  const int H = a.H;
  if (H == 5) return launch_h<5>(c, a, s, i, f), true;
  if (H == 6) return launch_h<6>(c, a, s, i, f), true;
  if (H == 7) return launch_h<7>(c, a, s, i, f), true;
  if (H == 8) return launch_h<8>(c, a, s, i, f), true;
  return false;
}
}  // namespace scendp_dsirp
