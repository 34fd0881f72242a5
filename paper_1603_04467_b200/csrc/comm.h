// Cross-replica transport of the replicated step (§3.2.2 :404-420 Send/Recv,
// §7 :934-941 the gradient combine): the collectives and point-to-point calls the session
// issues, over either
//
//   * NCCL (one process or thread per GPU; the production transport), or
//   * a simulated world: N sessions ("ranks") of one process on ONE GPU, each driven by its
//     own host thread, all enqueueing on one shared stream.  Every collective is a host
//     rendezvous (all ranks have enqueued their producing work) followed by device copies
//     from the peers' buffers; the fused NVLink exchange's "peer pointers" are the other
//     sessions' buffers on the same device.  The simulated world runs exactly the kernels
//     of the N-GPU step — the dW epilogue storing into owner slots (EPI_TRUNC16_P2P /
//     EPI_ASYNC_PUSH), the owner fold with and without owner-apply, the u16 expand-apply,
//     the flags — so their parity against the oracle can be checked on one GPU at any N <=
//     kMaxRanks.  Because every wait is rendezvoused on the host and the stream serialises
//     all ranks, no device-side flag wait can block a producer (no deadlock by construction).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <vector>

#include "../../include/dflow.h"

struct dflow_sim_world;

namespace dflow {

// NCCL init (world > 1, not simulated) or attach to the simulated world.
dflow_status comm_init(dflow_session* s, const uint8_t* nccl_id);
void comm_destroy(dflow_session* s);
bool comm_simulated(const dflow_session* s);

// Host rendezvous of all ranks in a simulated world (every rank has enqueued its work up to
// here on the shared stream); a no-op with NCCL, where the device flags order the ranks.
dflow_status comm_rendezvous(dflow_session* s);

// recv[i*bytes .. (i+1)*bytes) <- rank i's send[rank*bytes ..)   (ncclAlltoAll semantics)
dflow_status comm_alltoall(dflow_session* s, const void* send, void* recv, size_t bytes, cudaStream_t st);
// recv[i*bytes ..) <- rank i's send[0 .. bytes)                     (ncclAllGather)
dflow_status comm_allgather(dflow_session* s, const void* send, void* recv, size_t bytes, cudaStream_t st);
// recv[k] <- sum over ranks of send[k] (fp32; in place allowed)     (ncclAllReduce sum)
dflow_status comm_allreduce_f32(dflow_session* s, const float* send, float* recv, size_t n, cudaStream_t st);
// buf <- root's buf                                                 (ncclBroadcast)
dflow_status comm_broadcast_f32(dflow_session* s, float* buf, size_t n, int root, cudaStream_t st);
// point-to-point (f4 model parallelism channels)
dflow_status comm_send(dflow_session* s, const void* buf, size_t bytes, int peer, cudaStream_t st);
dflow_status comm_recv(dflow_session* s, void* buf, size_t bytes, int peer, cudaStream_t st);

// Symmetric-memory setup: every rank contributes `count` device allocations; *all receives
// world*count pointers valid on this rank (rank j's k-th at j*count + k): CUDA IPC mappings
// of the peers' allocations (recorded in *opened, closed at destroy), or — simulated — the
// peers' own pointers.
dflow_status comm_share_ptrs(dflow_session* s, void* const* mine, int count, std::vector<void*>* all,
                             std::vector<void*>* opened);

// NVLink SHARP multicast (f1, "data ... only transmitted once"): `bytes`
// of symmetric memory on every rank (ncclMemAlloc + a symmetric NCCL window; collective) and,
// when the switch can multicast, its multicast address: one `multimem.st` to *mc lands in every
// rank's copy.  *mc = nullptr when multicast is unavailable (the caller keeps unicast).
struct SymRegion;
dflow_status comm_symmetric_alloc(dflow_session* s, size_t bytes, void** local, void** mc, SymRegion** out);
void comm_symmetric_free(dflow_session* s, SymRegion* r);

// Fault injection of the simulated world (tests of the bounded flag waits): the dropped
// rank never sends its gradient contributions, as if it had died mid-step.
bool comm_dropped(const dflow_session* s);

}  // namespace dflow
