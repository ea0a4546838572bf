// verify_stub.cpp -- link-time stand-in for the part of the reference's
// verify.cpp that cannot be compiled here: ransac_fundamental needs Eigen
// 3.3+, absent from this image (/root/reference/proj/src/verify.cpp:3, 345+).
// The Eigen-free SAO part (verify.cpp:1-341) is compiled from the reference
// source (oracle/Makefile: _ref/verify_sao.cpp).  execute_plan only calls
// RANSAC when verification is enabled (engine.cpp:422-425); every oracle/_ref
// entry point runs with verification off, so reaching it is a bug and throws.
// TEST INFRASTRUCTURE ONLY.
#include "bandmatch/verify.hpp"

namespace bandmatch {

InlierSet ransac_fundamental(const PairMatches&, const std::vector<Keypoint>&,
                             const std::vector<Keypoint>&, const RansacParams&, std::uint64_t) {
  fail("Unsupported", "verify.cpp needs Eigen, which is absent: verification is unavailable");
}

}  // namespace bandmatch
