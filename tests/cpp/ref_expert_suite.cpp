// The reference's own expert test suite (proj/tests/test_expert.cpp),
// compiled in place from /root/reference (never copied) against the GPU
// drop-in: include/moeprism/dropin/moeprism/expert.hpp shadows the reference's
// expert.hpp so every partitioned_forward call in the suite runs on the B200
// (include/moeprism/moe_layer.hpp), while toy_ffn_forward and
// collect_activation_matrix stay the reference's CPU definitions -- the suite's
// decomposition KATs (all-active == full forward, single sub-expert hand sum,
// additivity, empty set, validation verdicts) compare the two.  doctest is
// not in the image: tests/cpp/shim/doctest.h provides its macros.
// Built by oracle/Makefile into oracle/_ref/ref_expert_suite (the reference
// sources exist only in the build container); run by tests/test_cpp_api.py.
#include "doctest.h"

#include "test_expert.cpp"  // NOLINT: proj/tests/test_expert.cpp, from the include path

int run_acceptance_c1();  // ref_acceptance_c1.cpp

int main() {
    std::printf("== proj/tests/test_expert.cpp against the GPU partitioned_forward\n");
    const int failed = doctest_shim::run_all();
    std::printf("== proj/tests/acceptance.cpp criterion 1 against the GPU partitioned_forward\n");
    const int c1 = run_acceptance_c1();
    if (failed == 0 && c1 == 0) std::printf("ALL PASSED\n");
    return failed == 0 && c1 == 0 ? 0 : 1;
}
