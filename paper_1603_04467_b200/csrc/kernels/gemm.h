// Host-side GEMM launcher interface (NK1-NK6).  See gemm.cuh for the kernel.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "round16.h"

namespace dflow {

// "operand" outputs are written as bf16 (RNE) in the bf16 path, or as the tf32
// pair (big -> out, small -> out2, fp32 each) in the 3xTF32 path.
enum GemmEpilogue : int {
  EPI_F32 = 0,             // out_f32[m,n] = acc                                           (a4 fetch, dx)
  EPI_TRUNC16 = 1,         // out_u16[m,n] = bits(acc) >> 16                               (a4 + a6)
  EPI_BIAS_RELU = 2,       // a = relu(acc + bias[n]) -> operand out and/or fp32 out_f32   (a1)
  EPI_RELUGRAD = 3,        // dz = acc * 1[mask[m,n] > 0] -> operand out [+ db partials]    (a3 + a5)
  EPI_BIAS_RELU_LOSS = 4,  // a = relu(acc + bias) [-> out_f32]; loss seed dz -> operand out
                           // [+ db partials, + loss partials]                            (a1 + a2 + a5)
  EPI_SGD_APPLY = 5,       // out_f32 (fp32 master W) -= lr * acc; operand copy refreshed  (a4 + a9, N = 1)
  EPI_TRUNC16_P2P = 6,     // bits(acc) >> 16 stored straight into the OWNER rank's receive slot over
                           // NVLink (peer pointers): a4 + a6 + the all-to-all leg of a7 in one kernel
  EPI_ASYNC_PUSH = 7,      // f3: owner's shard[m*N + n] += -fl(lr * g_hat) by a system-scope fp32
                           // reduction over NVLink (g_hat coded when the owner is another rank)
};

constexpr int kMaxRanks = 8;

// Kernel arguments (by value, __grid_constant__-style).
struct GemmArgs {
  int M, N, K;
  int tiles_m, tiles_n;   // tiles of (128*CG) x BN
  void* out;              // operand output (bf16 / tf32 big) or u16 (TRUNC16)
  void* out2;             // 3xTF32: operand output small part
  int64_t ldo;
  float* out_f32;         // fp32 output (F32, SGD master, optional for BIAS_RELU[_LOSS])
  int64_t ldo32;
  const float* bias;      // [N]
  const void* mask;       // RELUGRAD: the forward activation A_{l-1} (bf16, or tf32 big part)
  int64_t ldm;
  int vec_out;            // 1: 16-byte vector stores are aligned for out (and out2)
  int vec_out32;          // 1: 16-byte vector stores are aligned for out_f32
  int vec_mask;           // 1: 16-byte vector loads are aligned for mask
  // EPI_BIAS_RELU_LOSS
  const float* y;         // target [M, ldy] (MSE)
  int64_t ldy;
  int loss_kind;          // 0 MSE, 1 SUM
  float loss_denom;       // rows * cols (MSE seed divisor, IEEE division)
  float inv_denom;        // 1 / loss_denom, exact when denom_pow2
  int denom_pow2;         // 1: loss_denom is a power of two, so d * inv_denom == d / loss_denom
  int vec_y;              // 1: 16-byte vector loads are aligned for y
  int vec_bias;           // 1: 16-byte vector loads are aligned for bias
  int group_m;            // tile raster: M-tiles per group (L2 reuse of the B panels)
  int prefetch;           // k-blocks the producer's L2 prefetch runs ahead of its loads (0: off)
  int evict;              // 1: epilogue loads / stores of once-touched data use the streaming
                          // (evict-first) L2 policy (ld/st.global.cs)
  int debug;              // profiling only (DFLOW_GEMM_DEBUG): 1 no TMA loads, 2 no epilogue work,
                          // 4 hint-free barrier waits in the producer / MMA loop,
                          // 8 EPI_BIAS_RELU_LOSS targets not loaded (y = 0)
  int* sched;             // [4]: tile counters of die 0 / die 1, done counter, pad (zero at launch; the
                          // kernel resets them)
  const int* die_map;     // [#SMs] die of each SM id (die-aware schedule), or NULL
  int die_split;          // die_mode 1: raster tiles [0, die_split) to die 0, the rest to die 1;
                          // die_mode 2: N-tiles [0, die_split) of every M-group to die 0
  int die_mode;
  float seed_const;       // 1 / rows (SUM seed)
  float sgd_lr;           // EPI_SGD_APPLY learning rate
  double* loss_partials;  // [tiles * CG * 4] per-(tile, CTA, epilogue warp) partial sums
  // EPI_RELUGRAD / EPI_BIAS_RELU_LOSS: column sums of the stored dz per 32-row block
  float* colsum_ws;       // [ceil(M / 32), N] or nullptr
  // EPI_TRUNC16_P2P: element (m, n) is bucket index m*N + n, owned by rank idx / p2p_shard;
  // it lands at p2p_recv[owner][p2p_rank * p2p_shard + idx - owner * p2p_shard]
  uint16_t* p2p_recv[kMaxRanks];
  int64_t p2p_shard;
  int p2p_rank;
  int p2p_world;
  int p2p_bulk;           // 1: each staged row goes out as bulk (TMA engine) copies, not st.global
  // EPI_TRUNC16 / EPI_TRUNC16_P2P: the 16-bit code of element (m, n) is
  // round16(bits, m*N + n, r16) — truncation, or SR16 (reading A26)
  Round16 r16;
  // EPI_ASYNC_PUSH: every rank's shard of the layer bucket (shard/rank/world in p2p_*, lr in
  // sgd_lr); async_coded = 0 for the FP32 channel
  float* async_master[kMaxRanks];
  int async_coded;
  // EPI_BIAS_RELU: 1 = store the operand as the channel's 16-bit truncation code instead of
  // the RNE bf16 value (f4: the activation that crosses to the next device, reading A33)
  int trunc_out;
};

struct GemmDesc {
  int64_t M, N, K;
  bool tf32;                                // false: bf16 operands; true: 3xTF32 (fp32 big/small pairs)
  const void* A;  const void* A2; int64_t lda; bool a_mn;  // a_mn=0: A(m,k)=A[m*lda+k]; 1: A[k*lda+m]
  const void* B;  const void* B2; int64_t ldb; bool b_mn;  // b_mn=0: B(k,n)=B[n*ldb+k]; 1: B[k*ldb+n]
  int epilogue;                             // GemmEpilogue
  void* out;  void* out2; int64_t ldo;
  float* out_f32; int64_t ldo32;
  const float* bias;
  const void* mask; int64_t ldm;
  const float* y; int64_t ldy;              // EPI_BIAS_RELU_LOSS
  int loss_kind;
  double* loss_partials;
  float* colsum_ws;                         // fused db partials (RELUGRAD, BIAS_RELU_LOSS)
  float sgd_lr;                             // EPI_SGD_APPLY
  uint16_t* const* p2p_recv;                // EPI_TRUNC16_P2P: [world] peer receive bases
  float* const* async_master;               // EPI_ASYNC_PUSH: [world] shard bases
  int async_coded;
  int trunc_out;                            // EPI_BIAS_RELU: truncation code instead of RNE
  int64_t p2p_shard;
  int p2p_rank, p2p_world;
  int p2p_bulk;    // EPI_TRUNC16_P2P: ship staged rows with bulk copies (TMA engine)
  int group;       // tile-raster group (M tiles); 0 = default
  int tile;        // 0 = auto, 1 = 128x128 (1 CTA), 2 = 256x256 (CTA pair)
  int max_ctas;    // 0 = all SMs; else cap (SM reservation for concurrent NCCL kernels)
  int* sched;      // tile-scheduler counters [4] (zeroed); NULL = those of the device's legacy
                   // stream.  GEMMs that may run concurrently must not share counters
};

// Prepared launch: tensor maps + args, reusable across calls while buffers stay put.
struct GemmPlan {
  CUtensorMap tmA, tmB, tmA2, tmB2;
  GemmDesc d;
  GemmArgs args;
  int tile;
  int grid;
  int tiles_m, tiles_n;
  void* kernel;
  int smem;
  int cluster;
};

// Returns cudaSuccess or an error (cudaErrorInvalidValue for unsupported layouts).
cudaError_t gemm_prepare(const GemmDesc& d, int num_sms, GemmPlan* plan);
cudaError_t gemm_launch(const GemmPlan& plan, cudaStream_t stream);
// Tile-scheduler counters owned by (current device, stream), for GEMMs outside a session.
int* gemm_stream_sched(cudaStream_t stream);
const char* gemm_last_error();

}  // namespace dflow
