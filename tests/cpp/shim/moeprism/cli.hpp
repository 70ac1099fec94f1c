// Stand-in for the reference's <moeprism/cli.hpp> (CLI11 is not in this
// image): lets proj/tests/acceptance.cpp compile for its criterion 1; the CLI
// criterion itself is not run by tests/cpp/ref_acceptance_c1.cpp.
#pragma once

#include <ostream>
#include <string>
#include <vector>

namespace moeprism::cli {
inline int run_cli(const std::vector<std::string>&, std::ostream&) { return 2; }
}  // namespace moeprism::cli
