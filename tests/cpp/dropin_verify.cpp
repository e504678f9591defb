// The reference's own verification harness (verify.cpp run_verify) driven
// through the drop-in build: its packed / bypass / sharded suites run on the
// B200 (compat_impl.inc inside namespace moesim), and its --perturb self-test
// (a +0.5 nudge of one combine weight before dispatch, verify.cpp:34) must
// make the harness report a mismatch.  TEST INFRASTRUCTURE.  Exit 0 = both hold.
#include <cstdio>

#include "moesim/verify.hpp"

int main() {
    moesim::VerifyOptions ok_opt;
    ok_opt.trials = 50;
    const auto ok = moesim::run_verify(ok_opt);
    std::printf("verify: ok=%d trials=%d suite=%s max_rel=%.3g\n", ok.ok, ok.trials_run, ok.suite.c_str(), ok.max_rel);
    moesim::VerifyOptions bad_opt = ok_opt;
    bad_opt.perturb = true;
    const auto bad = moesim::run_verify(bad_opt);
    std::printf("perturbed: ok=%d suite=%s seed=%llu max_rel=%.3g\n", bad.ok, bad.suite.c_str(),
                static_cast<unsigned long long>(bad.failing_seed), bad.max_rel);
    const bool pass = ok.ok && !bad.ok && bad.suite == "padded-vs-packed";
    std::printf("%s\n", pass ? "verify self-test holds" : "verify self-test FAILED");
    return pass ? 0 : 1;
}
