// The simulated N-rank world (comm.h): N sessions on one GPU, one host thread per rank,
// one shared stream.  Test harness of the N-GPU path; not a transport for real training.
#pragma once
#include <cuda_runtime.h>

#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <vector>

#include "../../include/dflow.h"
#include "kernels/gemm.h"

struct dflow_sim_world {
  int world = 0, device = 0;
  cudaStream_t stream = nullptr;
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  uint64_t gen = 0;
  bool broken = false;                    // a rendezvous failed: every later one fails fast
  std::vector<const void*> slot;          // per-rank pointer published for the current collective
  struct Box {                            // point-to-point mailbox [src][dst]
    const void* ptr = nullptr;
    size_t bytes = 0;
    int state = 0;                        // 0 empty, 1 posted by the sender, 2 consumed
  };
  Box box[dflow::kMaxRanks][dflow::kMaxRanks];
  int drop_rank = -1;                     // fault injection: this rank sends no gradient contributions
  int64_t timeout_ms = 120000;            // host rendezvous timeout
};

namespace dflow {
// Runs fn(rank) for every rank of the world on its own host thread (device set), joins, and
// synchronises the world's stream.  Returns the first failing rank's status; its message
// becomes this thread's dflow_last_error.
dflow_status sim_run(dflow_sim_world* w, const std::function<dflow_status(int)>& fn);
}  // namespace dflow
