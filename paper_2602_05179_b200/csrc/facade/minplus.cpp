// minplus.cpp -- the (min,+) algebra of the drop-in facade (reference:
// proj/src/minplus.cpp).  Shapes are validated on the host with the
// reference's messages; every apply / sweep runs on the GPU through
// scendp_minplus_sweep (K5).
#include "scendp/minplus.hpp"

#include <algorithm>
#include <stdexcept>
#include <string>

#include "runtime.hpp"

namespace scendp {

static_assert(sizeof(ExtendedCost) == sizeof(double), "ExtendedCost is one double");

MaskedTransition::MaskedTransition(std::size_t rows, std::size_t cols, std::size_t option_depth)
    : rows_(rows), cols_(cols), depth_(option_depth) {
  if (rows == 0 || cols == 0 || option_depth == 0)
    throw std::invalid_argument("transition matrix dimensions must be positive");
  entries_.assign(rows * cols * option_depth, ExtendedCost::infinity());
}

MaskedTransition MaskedTransition::collapse_options() const {
  MaskedTransition out(rows_, cols_, 1);
  for (std::size_t r = 0; r < depth_; ++r)
    for (std::size_t i = 0; i < rows_; ++i)
      for (std::size_t j = 0; j < cols_; ++j) out.at(i, j) = extended_min(out.at(i, j), at(i, j, r));
  return out;
}

namespace {

// The chain on the default device: `batch` frontiers of `width` values in
// `init` (item-major); returns [batch][all ? width + sum cols : last cols].
std::vector<double> sweep(std::span<const MaskedTransition> stages, const double* init,
                          std::size_t width, std::size_t batch, bool all) {
  std::vector<scendp_minplus_stage> cs(stages.size());
  std::size_t total = width, last = width;
  for (std::size_t s = 0; s < stages.size(); ++s) {
    const MaskedTransition& a = stages[s];
    if (a.rows() != last)
      throw std::invalid_argument("min-plus apply: matrix has " + std::to_string(a.rows()) +
                                  " rows but frontier has " + std::to_string(last) + " entries");
    cs[s] = {a.rows(), a.cols(), a.option_depth(), reinterpret_cast<const double*>(a.data())};
    last = a.cols();
    total += a.cols();
  }
  std::vector<double> out(batch * (all ? total : last));
  if (batch == 0 || stages.empty()) {  // nothing to apply: the frontiers as given
    std::copy(init, init + out.size(), out.begin());
    return out;
  }
  detail::DeviceSlot& slot = detail::device_slot(-1);
  std::lock_guard<std::mutex> g(slot.mu);
  detail::check(scendp_minplus_sweep(slot.ctx, cs.data(), static_cast<std::uint32_t>(cs.size()),
                                     init, width, batch, SCENDP_MEM_HOST,
                                     all ? SCENDP_MINPLUS_ALL_STAGES : 0u, out.data()));
  return out;
}

ValueFrontier to_frontier(int stage, const double* v, std::size_t n) {
  ValueFrontier f;
  f.stage = stage;
  f.values.resize(n);
  for (std::size_t k = 0; k < n; ++k) f.values[k] = ExtendedCost{v[k]};
  return f;
}

}  // namespace

ValueFrontier minplus_apply(const MaskedTransition& a, const ValueFrontier& j) {
  if (a.option_depth() != 1)
    throw std::invalid_argument("min-plus apply: option depth > 1, use minplus_apply_options");
  return minplus_apply_options(a, j);
}

ValueFrontier minplus_apply_options(const MaskedTransition& a, const ValueFrontier& j) {
  const std::vector<double> out =
      sweep({&a, 1}, reinterpret_cast<const double*>(j.values.data()), j.size(), 1, false);
  return to_frontier(j.stage + 1, out.data(), a.cols());
}

std::vector<ValueFrontier> forward_sweep(std::span<const MaskedTransition> stages,
                                         const ValueFrontier& initial) {
  const std::vector<double> all = sweep(
      stages, reinterpret_cast<const double*>(initial.values.data()), initial.size(), 1, true);
  std::vector<ValueFrontier> out;
  out.reserve(stages.size() + 1);
  out.push_back(initial);
  std::size_t off = initial.size();
  for (std::size_t s = 0; s < stages.size(); ++s) {
    out.push_back(to_frontier(initial.stage + static_cast<int>(s) + 1, all.data() + off,
                              stages[s].cols()));
    off += stages[s].cols();
  }
  return out;
}

std::vector<ValueFrontier> forward_sweep_batch(std::span<const MaskedTransition> stages,
                                               std::span<const ValueFrontier> initials) {
  if (initials.empty()) return {};
  const std::size_t width = initials[0].size();
  std::vector<double> init(initials.size() * width);
  for (std::size_t b = 0; b < initials.size(); ++b) {
    if (initials[b].size() != width)
      throw std::invalid_argument("forward_sweep_batch: frontiers differ in size");
    for (std::size_t k = 0; k < width; ++k) init[b * width + k] = initials[b].values[k].value;
  }
  const std::vector<double> out = sweep(stages, init.data(), width, initials.size(), false);
  const std::size_t last = stages.empty() ? width : stages.back().cols();
  std::vector<ValueFrontier> res;
  res.reserve(initials.size());
  for (std::size_t b = 0; b < initials.size(); ++b)
    res.push_back(to_frontier(initials[b].stage + static_cast<int>(stages.size()),
                              out.data() + b * last, last));
  return res;
}

}  // namespace scendp
