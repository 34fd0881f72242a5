// Asynchronous data parallelism (Fig.7 bottom;
// readings A29-A31).  The shared fp32 parameters live once, sharded over the N ranks by
// bucket position (the synchronous exchange's sharding); every rank maps every shard
// through CUDA IPC.  A replica's step:
//
//   pull  (k_async_pull)    : read all shards (NVLink loads) -> local W32, b32 and the bf16
//                             operand copy the GEMMs read
//   forward / backward      : on the local copies
//   push  (GEMM EPI_ASYNC_PUSH for dW, k_colsum_push for db): for every element the
//                             delta -fl(lr * g_hat) is added to its owner's shard with a
//                             system-scope fp32 reduction over NVLink (g_hat = the 16-bit
//                             coded gradient when the owner is another rank, reading A30)
//
// No mean over replicas, no barrier: each replica's update lands whenever it is pushed.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "gemm.h"
#include "round16.h"

namespace dflow {

struct AsyncLayer {
  float* master[kMaxRanks];  // rank j's shard of this layer's bucket [dW ; db]  [shard]
  int64_t shard;             // P_pad / N
  int64_t in, out;           // bucket = in*out weights (row-major) then out biases
  int rank, world;
};

// local W32 [in*out] (may be NULL: not refreshed), b32 [out] and the bf16 operand copy
// wop [in, ldwb] <- the shared shards (16-byte NVLink loads when out % 4 == 0)
cudaError_t launch_async_pull(const AsyncLayer& a, float* W32, float* b32, __nv_bfloat16* wop, int64_t ldwb,
                              cudaStream_t s);
// db_l (sum of the per-32-row partials, fixed order) pushed into the owners' shards:
// master[owner][idx - owner*shard] += -fl(lr * g_hat), idx = in*out + c
cudaError_t launch_colsum_push(const float* ws, int chunks, const AsyncLayer& a, float lr, int coded, Round16 r,
                               cudaStream_t s);
// this rank's shard of the bucket <- W32 / b32 (assignment of the initial values)
cudaError_t launch_async_publish(const AsyncLayer& a, const float* W32, const float* b32, cudaStream_t s);

// System-scope fp32 reductions into (possibly peer) memory.  Note the hardware's fp32
// reduction flushes subnormal operands and results to zero (reading A31).
__device__ __forceinline__ void red_add_sys(float* p, float v) {
  asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(p), "f"(v) : "memory");
}
__device__ __forceinline__ void red_add_sys_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.relaxed.sys.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

}  // namespace dflow
