// dsirp_exact.cu -- dispatch of horizons 1..8 to the HMAX == H kernels.
#include "common.cuh"
#include "internal.hpp"
#include "dsirp_kernels.cuh"

namespace scendp_dsirp {
bool launch_exact_a(scendp_ctx*, const DsirpArgs&, size_t, bool, bool);  // H 1..4
bool launch_exact_b(scendp_ctx*, const DsirpArgs&, size_t, bool, bool);  // H 5..8

void launch_exact(scendp_ctx* c, const DsirpArgs& a, size_t s, bool i, bool f) {
  if (launch_exact_a(c, a, s, i, f) || launch_exact_b(c, a, s, i, f)) return;
  scendp_host::fail(SCENDP_ERR_UNSUPPORTED, "dsirp: horizon outside 1..8 in launch_exact");
}
}  // namespace scendp_dsirp
