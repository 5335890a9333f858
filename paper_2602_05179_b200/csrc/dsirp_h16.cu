// dsirp_h16.cu -- K3 instantiations for horizons <= 16 (own translation
// unit so the unrolled kernels compile in parallel).
#include "common.cuh"
#include "internal.hpp"
#include "dsirp_kernels.cuh"

namespace scendp_dsirp {
void launch_h16(scendp_ctx* c, const DsirpArgs& a, size_t s, bool i, bool f) {
  launch_h<16>(c, a, s, i, f);
}
}  // namespace scendp_dsirp
