// Drop-in build: the reference's hot-path operators
// (gating.cpp, pft.cpp, pf_pipeline.cpp, rbd.cpp, ssmb.cpp) are NOT compiled;
// their moesim:: symbols come from xmoe's reference-shaped adapter
// (paper_2508_13337_b200/csrc/compat_impl.inc) included here inside
// namespace moesim against the reference's own headers, so every call runs
// on the B200 through libxmoe.so.  The reference's non-hot-path sources
// (collectives/ledger, padded pipeline, planner, placement, verify, CPU
// kernels) and its acceptance suite are compiled unmodified from
// /root/reference and linked against it (tests/cpp/Makefile, target dropin).
// TEST INFRASTRUCTURE.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "moesim/collectives.hpp"
#include "moesim/error.hpp"
#include "moesim/gating.hpp"
#include "moesim/pf_pipeline.hpp"
#include "moesim/pft.hpp"
#include "moesim/rbd.hpp"
#include "moesim/ssmb.hpp"
#include "xmoe/xmoe.h"

namespace moesim {
#include "compat_impl.inc"
}  // namespace moesim
