// stream_gen.cuh -- generate_update_stream with its insertion sampling on
// the device (stream_gen.cu).
#pragma once

#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dyg.h"

namespace dyg {

struct GenError {
  int code;  // ErrorKind (error.hpp:9)
  std::string message;
};

struct GenStats {
  uint64_t rounds = 0;      // speculative rounds of insertion attempts
  uint64_t rejections = 0;  // rejected attempts (self-loop, edge, repeat)
  uint64_t rehashes = 0;    // pair-set rebuilds
};

// stream.cpp:114-200 for locality 0, bit-identical; throws GenError with the
// reference's messages. Uses the current device.
void generate_stream_device(const dyg_csr& g, double insert_fraction, double delete_fraction,
                            uint32_t batches, uint64_t seed, std::vector<dyg_event>& events,
                            uint32_t& batch_count, GenStats* stats);

}  // namespace dyg
