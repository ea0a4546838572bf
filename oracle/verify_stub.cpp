// verify_stub.cpp -- link-time stand-ins for the reference's verify.cpp, which
// cannot be compiled here (it needs Eigen 3.3+, absent from this image;
// /root/reference/proj/src/verify.cpp:3).  execute_plan only calls these when
// verification is enabled (engine.cpp:422-425); every oracle/_ref entry point
// runs with verification off, so reaching one of these is a bug and throws.
// TEST INFRASTRUCTURE ONLY.
#include "bandmatch/verify.hpp"

namespace bandmatch {

SaoOutcome sao_filter(const PairMatches&, const std::vector<Keypoint>&,
                      const std::vector<Keypoint>&, const SaoParams&) {
  fail("Unsupported", "verify.cpp needs Eigen, which is absent: verification is unavailable");
}

InlierSet ransac_fundamental(const PairMatches&, const std::vector<Keypoint>&,
                             const std::vector<Keypoint>&, const RansacParams&, std::uint64_t) {
  fail("Unsupported", "verify.cpp needs Eigen, which is absent: verification is unavailable");
}

}  // namespace bandmatch
