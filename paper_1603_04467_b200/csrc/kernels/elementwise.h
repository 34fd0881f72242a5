// HBM-bound kernels of the step (NK7-NK13): codec, loss seed, bias-gradient
// column sum, owner reduce, SGD apply, casts, relu masks.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cstdint>

#include "gemm.h"
#include "round16.h"

namespace dflow {

// NK9 / NK10: dst[i] = bits(src[i]) >> 16  /  dst[i] = float(bits = src[i] << 16)
cudaError_t launch_truncate16(const float* src, uint16_t* dst, size_t n, cudaStream_t s);
// a6 with either codec (round16.h): dst[i] = round16(bits(src[i]), idx_base + i, r)
cudaError_t launch_round16(const float* src, uint16_t* dst, size_t n, Round16 r, int64_t idx_base, cudaStream_t s);
cudaError_t launch_expand16(const uint16_t* src, float* dst, size_t n, cudaStream_t s);

// NK13: dst bf16 [rows, ldd] = RNE(src f32 [rows, lds]) for cols columns.
cudaError_t launch_cast_bf16(const float* src, int64_t lds, __nv_bfloat16* dst, int64_t ldd, int64_t rows,
                             int64_t cols, cudaStream_t s);
// NK13 (3xTF32): hi = tf32_rna(x), lo = fl32(x - hi) for fp32 x [rows, lds] -> hi, lo [rows, ldd]
// (reading A14).  hi + lo == x exactly.
cudaError_t launch_split_tf32(const float* src, int64_t lds, float* hi, float* lo, int64_t ldd, int64_t rows,
                              int64_t cols, cudaStream_t s);
// dense fp32 [rows, cols] = hi + lo (exact reconstruction of a 3xTF32 operand pair)
cudaError_t launch_join_tf32(const float* hi, const float* lo, int64_t ld, int64_t rows, int64_t cols, float* out,
                             cudaStream_t s);
// bf16 [rows, lds] -> bf16 [rows, ldd] (bf16 feeds with a foreign leading dim).
cudaError_t launch_copy_bf16(const __nv_bfloat16* src, int64_t lds, __nv_bfloat16* dst, int64_t ldd, int64_t rows,
                             int64_t cols, cudaStream_t s);

// NK7 final pass: the last forward GEMM's epilogue (EPI_BIAS_RELU_LOSS) leaves
// n per-(CTA, warp) partial sums; C = sum / (2 rows cols) (MSE) or sum / rows
// (SUM), summed in a fixed order (deterministic) into *loss (fp32).
cudaError_t launch_loss_final(int kind, const double* partials, int n, int64_t rows, int64_t cols, float* loss,
                              cudaStream_t s);

// NK8 final pass: db[c] = sum_k ws[k, c] over the `chunks` per-32-row partial
// column sums the dz-producing epilogue wrote (fixed order).  fp32 and/or u16 out.
// The u16 output is round16(bits(db[c]), idx_base + c, r) (the db tail of the layer bucket).
// bias != NULL (N = 1 train step): also bias[c] <- fl(bias[c] - fl(lr * db[c])).
cudaError_t launch_colsum_final(const float* ws, int chunks, int64_t cols, float* out_f32, uint16_t* out_u16,
                                cudaStream_t s, Round16 r = {0, 0}, int64_t idx_base = 0, float* bias = nullptr,
                                float lr = 0.f);

// NK11: owner fold of N received shards (rank order), x (1/N), 16-bit code (truncate or
// SR16 at bucket positions idx_base + i).
cudaError_t launch_owner_reduce_t16(const uint16_t* recv, int64_t shard, int nranks, uint16_t* out,
                                    cudaStream_t s, Round16 r = {0, 0}, int64_t idx_base = 0);
cudaError_t launch_owner_reduce_f32(const float* recv, int64_t shard, int nranks, float* out, cudaStream_t s);
// Simulated transport (comm.h): dst[k] = p[0][k] + p[1][k] + ... + p[n-1][k] (fp32, rank
// order) over the ranks' buffers on this device (the sum of an all-reduce).
struct RankPtrs {
  const float* p[kMaxRanks];
};
cudaError_t launch_sum_ranks_f32(RankPtrs src, int nranks, float* dst, size_t count, cudaStream_t s);
// x (1/N) in place (FP32_NCCL after an allreduce-sum).
cudaError_t launch_scale_f32(float* x, int64_t n, float scale, cudaStream_t s);

// NK12: W <- fl(W - fl(lr * g)); g from fp32 (g32) or expanded u16 (g16).
// W dense [n = rows*cols]; optional bf16 working copy wbf [rows, ldwb].
cudaError_t launch_apply_sgd(float* W, const float* g32, const uint16_t* g16, int64_t rows, int64_t cols,
                             __nv_bfloat16* wbf, int64_t ldwb, float lr, cudaStream_t s);
// Same update, refreshing the 3xTF32 operand pair (whi, wlo) [rows, ldw] instead.
cudaError_t launch_apply_sgd_tf32(float* W, const float* g32, const uint16_t* g16, int64_t rows, int64_t cols,
                                  float* whi, float* wlo, int64_t ldw, float lr, cudaStream_t s);

// f4 (model parallelism), the receiving end of the backward channel: dz = expand(code) where
// this rank's activation a > 0, else 0 (ReluGrad on the received dA, reading A33), stored
// bf16 [rows, ldz]; also the per-32-row column partial sums of dz ([ceil(rows/32), cols]).
cudaError_t launch_relugrad_recv(const uint16_t* code, int64_t ldc, const __nv_bfloat16* a, int64_t lda, int64_t rows,
                                 int64_t cols, __nv_bfloat16* dz, int64_t ldz, float* colsum_ws, cudaStream_t s);

// Bit-pack 1[a > 0] of a bf16 [rows, ld] activation (cols columns) row-major.
cudaError_t launch_relu_mask_bits(const __nv_bfloat16* a, int64_t ld, int64_t rows, int64_t cols, uint32_t* bits,
                                  cudaStream_t s);
cudaError_t launch_relu_mask_bits_f32(const float* a, int64_t ld, int64_t rows, int64_t cols, uint32_t* bits,
                                      cudaStream_t s);
// bf16 [rows, ld] -> dense fp32 [rows, cols]
cudaError_t launch_bf16_to_f32(const __nv_bfloat16* a, int64_t ld, int64_t rows, int64_t cols, float* out,
                               cudaStream_t s);
// fp32 [rows, lds] -> dense fp32 [rows, cols]
cudaError_t launch_copy_f32(const float* a, int64_t lds, int64_t rows, int64_t cols, float* out, int64_t ldd,
                            cudaStream_t s);

}  // namespace dflow
