// Fused NVLink gradient exchange: the TRUNC16 schedule of
// a6-a9 with peer-memory stores instead of NCCL calls.
//
//   wgrad GEMM (EPI_TRUNC16_P2P) : each rank stores bits(dW)>>16 straight into the
//                                  owner's receive slot  recv[owner][rank*shard + i]
//   colsum_final_p2p             : db the same way, then raises phase-0 flags on every
//                                  owner: "rank r's layer-l contribution is complete"
//   owner_reduce_p2p             : waits for all N phase-0 flags, folds its shard in rank
//                                  order (x 1/N, truncate), stores q_bar into every
//                                  rank's gath[rank*shard + i], raises phase-1 flags
//   apply (+ wait)               : waits for all N phase-1 flags, applies expand(q_bar)
//
// Flags are monotonically increasing step epochs (no resets); ordering uses
// system-scope fences and release/acquire flag accesses.  Every wait is bounded (timeout_ns):
// a dead or desynchronised peer ends in a poisoned session, not a hung GPU.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "gemm.h"
#include "round16.h"

namespace dflow {

struct P2PLayer {
  uint16_t* recv[kMaxRanks];   // rank j's receive area of this layer  [world * shard]
  uint16_t* gath[kMaxRanks];   // rank j's gathered bucket             [world * shard]
  uint32_t* flags[kMaxRanks];  // rank j's flags of this layer         [2][kMaxRanks]
  int* done;                   // local grid-completion counters       [2]
  int64_t shard;
  int rank, world;
  // owner-apply (SURVEY §8(e), bf16 path): the owner applies the update to its fp32 shard and
  // pushes the new bf16 operand values (and fp32 biases) into every rank's copies
  int owner_apply;
  float* w32[kMaxRanks];       // rank j's fp32 master W [in*out] (dense, bucket order)
  float* b32[kMaxRanks];       // rank j's fp32 bias [out]
  uint16_t* wop[kMaxRanks];    // rank j's bf16 operand copy of W [in, ldwb] (unicast pushes)
  uint16_t* mc_wop;            // multicast address of every rank's copy (NVLink SHARP), or NULL:
                               // one multimem.st replaces the N unicast stores of the gather leg
  int64_t in, out, ldwb;
  float lr_w, lr_b;
  // bounded waits (failures abort the step): a flag wait that has not seen
  // its epoch after timeout_ns writes 1 to *abort (host-mapped) and its kernel returns without
  // signalling anyone, so every peer's wait times out as well; the host poisons the session
  uint32_t* abort;
  uint64_t timeout_ns;
};

// The cost C = mean_r C_r of a synchronous step over the same peer memory (no NCCL call in the
// step): every rank pushes its C_r into slot [epoch & 1][rank] of every rank and raises its
// flag; a rank that wants the value sums the N slots in rank order once all flags reach epoch.
struct LossPeers {
  float* slots[kMaxRanks];     // rank j's [2][kMaxRanks] loss slots
  uint32_t* flags[kMaxRanks];  // rank j's [kMaxRanks] loss flags
};
cudaError_t launch_loss_push(const float* loss, const LossPeers& p, int rank, int world, uint32_t epoch,
                             cudaStream_t s);
// out[0] = slots[par][0] + ... + slots[par][world-1] (fp32, rank order) once flags >= epoch
cudaError_t launch_loss_gather(const float* slots, const uint32_t* flags, int world, uint32_t epoch, float* out,
                               uint32_t* abort, uint64_t timeout_ns, cudaStream_t s);

// db_l (sum of the per-32-row partials), coded (truncate / SR16) and stored at bucket index
// base_idx + c in its owner's receive slot; then phase-0 flags.
cudaError_t launch_colsum_final_p2p(const float* ws, int chunks, int64_t cols, int64_t base_idx, const P2PLayer& p,
                                    uint32_t epoch, cudaStream_t s, Round16 r = {0, 0});
// Owner step over peer memory (see above); the mean is coded with r (truncate or SR16).
// With p.owner_apply the owner instead applies W <- fl(W - fl(lr * expand(q_bar))) to its own
// shard and pushes bf16(W) / fp32 b to every rank (phase-1 flags then mean "parameters in").
cudaError_t launch_owner_reduce_p2p(const P2PLayer& p, uint32_t epoch, cudaStream_t s, Round16 r = {0, 0});
// owner-apply: this rank's fp32 W <- every owner's shard (NVLink loads), for reads of W
cudaError_t launch_gather_w32(const P2PLayer& p, cudaStream_t s);
// Block until all `world` phase-1 flags of this rank reach `epoch` (one CTA, acquire.sys), or
// give up after timeout_ns (writing *abort).
cudaError_t launch_wait_flags(const uint32_t* flags, int world, uint32_t epoch, uint32_t* abort, uint64_t timeout_ns,
                              cudaStream_t s);

}  // namespace dflow
