// Drop-in shadow of the reference's <moeprism/expert.hpp> (proj/include/
// moeprism/expert.hpp).  Put include/moeprism/dropin FIRST on the include
// path, the reference's proj/include after it: code written against the
// reference -- its own test suites included -- then gets the reference's
// header unchanged except that moeprism::partitioned_forward
// (inc/expert.hpp:101-135) is the GPU implementation of moe_layer.hpp
// (same signature, same ValidationError verdicts, 1e-5 relative).  The CPU
// definition stays available as moeprism::partitioned_forward_reference_cpu.
#pragma once

#define partitioned_forward partitioned_forward_reference_cpu
#include_next <moeprism/expert.hpp>
#undef partitioned_forward

#include "moeprism/moe_layer.hpp"

namespace moeprism {
using b200::partitioned_forward;
}  // namespace moeprism
