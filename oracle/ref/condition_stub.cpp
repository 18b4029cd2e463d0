// Oracle build stub (test infrastructure only, NOT product code).
// calibrate_budget (/root/reference/proj/src/sparsifier.cpp:561-577) calls
// condition_number (spectral.cpp:252-276), which needs Eigen. The oracle
// never calibrates (configs use a fixed K), so the symbol throws.
#include "spectral.hpp"

namespace dysparse {
ConditionEstimate condition_number(const DynamicGraph&, const DynamicGraph&,
                                   const ConditionOptions&) {
  throw_numeric("condition_number is unavailable in the oracle build (no Eigen)");
}
}  // namespace dysparse
