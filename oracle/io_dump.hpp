// io_dump.hpp -- TEST INFRASTRUCTURE ONLY.  Canonical text dumps of the io.hpp
// types, compiled twice: into oracle/_ref (against the reference's headers,
// via ref_shim.cpp) and into tests/cpp/facade_main (against the drop-in
// facade's headers).  Both headers declare the same names and fields, so the
// two dumps of equal values are byte-identical and the tests compare text.
#pragma once

#include <cstdio>
#include <exception>
#include <fstream>
#include <sstream>
#include <string>
#include <variant>
#include <vector>

namespace io_dump {

inline std::string num(double v) {
  char b[40];
  std::snprintf(b, sizeof(b), "%.17g", v);
  return b;
}

template <typename V>
std::string list(const char* tag, const V& v) {
  std::string s = std::string(tag) + " " + std::to_string(v.size());
  for (const auto& x : v) s += " " + num(static_cast<double>(x));
  return s + "\n";
}

// parse_instance_text result (or the exception text) as lines.
template <typename Parsed, typename RoutingT, typename DsirpT>
std::string instance(const Parsed& p) {
  std::string s;
  if (const RoutingT* r = std::get_if<RoutingT>(&p)) {
    s += "routing n " + std::to_string(r->n) + " Q " + std::to_string(r->capacity) + " hard " +
         std::to_string(r->hard ? 1 : 0) + " beta " + num(r->penalty_beta) + "\n";
    s += list("costs", r->costs);
    return s;
  }
  const DsirpT& d = std::get<DsirpT>(p);
  s += "dsirp U " + std::to_string(d.spec.capacity) + " I0 " +
       std::to_string(d.spec.initial_inventory) + " H " + std::to_string(d.spec.horizon) +
       " h " + num(d.spec.holding) + " rho " + num(d.spec.stockout_multiplier) + "\n";
  s += "delivery H " + std::to_string(d.delivery.horizon) + " R " +
       std::to_string(d.delivery.options) + " tabular " +
       std::to_string(d.delivery.tabular ? 1 : 0) + " q " +
       std::to_string(d.delivery.table_quantities) + "\n";
  s += list("fixed", d.delivery.fixed) + list("unit", d.delivery.unit) +
       list("table", d.delivery.table);
  s += "holding tabular " + std::to_string(d.holding.tabular ? 1 : 0) + "\n";
  s += list("htable", d.holding.table);
  return s;
}

}  // namespace io_dump
