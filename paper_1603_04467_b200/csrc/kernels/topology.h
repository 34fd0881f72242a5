// SM -> die map of the device, measured once per device by L2 hit latencies (topology.cu).
#pragma once
#include <vector>

namespace dflow {
// true when the map is clean (every SM decisively on one of two populated dies); *die_of_sm
// gets die 0 / 1 per SM id (even when not clean, for inspection); *agreement = the weakest
// SM's agreement with its die's near/far pattern (1.0 = perfect; first call only).
bool measure_die_map(int device, std::vector<int>* die_of_sm, double* agreement);
}  // namespace dflow
