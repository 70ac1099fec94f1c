// Acceptance criterion 1 of the reference (proj/tests/acceptance.cpp:69-100,
// "decomposition exactness": 100 random experts / partitions, every
// sub-expert active == toy_ffn_forward within 1e-5 relative, 10 s budget),
// compiled in place from /root/reference with partitioned_forward resolved to
// the GPU drop-in (see ref_expert_suite.cpp).  The reference's main() is
// renamed away; only criterion 1 exercises the drop-in.
#include <cstdio>

#define main reference_acceptance_main
#include "acceptance.cpp"  // NOLINT: proj/tests/acceptance.cpp, from the include path
#undef main

int run_acceptance_c1() {
    Outcome out;
    try {  // as the reference's main() does (acceptance.cpp:481-486)
        out = criterion_decomposition();
    } catch (const std::exception& e) {
        out.fail(std::string("unhandled exception: ") + e.what());
    }
    std::printf("%s criterion 1: decomposition exactness (%s)\n", out.pass ? "PASS" : "FAIL", out.detail.c_str());
    return out.pass ? 0 : 1;
}
