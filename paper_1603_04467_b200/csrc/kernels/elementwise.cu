// HBM-bound kernels of the replicated MLP step (NK7-NK13).  Vectorised 16-byte
// loads/stores, grid-stride loops sized to a few waves of 148 SMs, explicit
// round-to-nearest intrinsics (no FMA contraction, no flush-to-zero) wherever the
// oracle fixes the bits (codec, owner fold, SGD update).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdint>

#include "elementwise.h"
#include "colsum.cuh"

namespace dflow {

namespace {

constexpr int kThreads = 256;
constexpr int kMaxBlocks = 148 * 8;

inline int blocks_for(int64_t work_items) {
  int64_t b = (work_items + kThreads - 1) / kThreads;
  if (b < 1) b = 1;
  return static_cast<int>(std::min<int64_t>(b, kMaxBlocks));
}

inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

__device__ __forceinline__ uint32_t pack2_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

// ------------------------------------------------------------------ codec
__global__ void k_truncate16(const float* __restrict__ src, uint16_t* __restrict__ dst, int64_t n, int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nv = n / 8;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int64_t i = tid; i < nv; i += stride) {
      const uint4 a = s4[2 * i], b = s4[2 * i + 1];
      uint4 o;
      o.x = (a.x >> 16) | (a.y & 0xFFFF0000u);
      o.y = (a.z >> 16) | (a.w & 0xFFFF0000u);
      o.z = (b.x >> 16) | (b.y & 0xFFFF0000u);
      o.w = (b.z >> 16) | (b.w & 0xFFFF0000u);
      d4[i] = o;
    }
    done = nv * 8;
  }
  const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
  for (int64_t i = done + tid; i < n; i += stride) dst[i] = static_cast<uint16_t>(s[i] >> 16);
}

// a6 with the SR16 codec: element i is bucket position idx_base + i
__global__ void k_round16(const float* __restrict__ src, uint16_t* __restrict__ dst, int64_t n, Round16 r,
                          int64_t idx_base) {
  const uint32_t* s = reinterpret_cast<const uint32_t*>(src);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
    dst[i] = static_cast<uint16_t>(round16(s[i], idx_base + i, r));
}

__global__ void k_expand16(const uint16_t* __restrict__ src, float* __restrict__ dst, int64_t n, int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t done = 0;
  if (vec) {
    const int64_t nv = n / 8;
    const uint4* s4 = reinterpret_cast<const uint4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int64_t i = tid; i < nv; i += stride) {
      const uint4 q = s4[i];
      d4[2 * i] = make_uint4(q.x << 16, q.x & 0xFFFF0000u, q.y << 16, q.y & 0xFFFF0000u);
      d4[2 * i + 1] = make_uint4(q.z << 16, q.z & 0xFFFF0000u, q.w << 16, q.w & 0xFFFF0000u);
    }
    done = nv * 8;
  }
  uint32_t* d = reinterpret_cast<uint32_t*>(dst);
  for (int64_t i = done + tid; i < n; i += stride) d[i] = static_cast<uint32_t>(src[i]) << 16;
}

// ------------------------------------------------------------------ casts
__global__ void k_cast_bf16(const float* __restrict__ src, int64_t lds, __nv_bfloat16* __restrict__ dst,
                            int64_t ldd, int64_t rows, int64_t cols, int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {  // cols % 8 == 0, aligned rows
    const int64_t per_row = cols / 8, total = rows * per_row;
    for (int64_t i = tid; i < total; i += stride) {
      const int64_t r = i / per_row, c = (i - r * per_row) * 8;
      const float4 a = *reinterpret_cast<const float4*>(src + r * lds + c);
      const float4 b = *reinterpret_cast<const float4*>(src + r * lds + c + 4);
      *reinterpret_cast<uint4*>(dst + r * ldd + c) =
          make_uint4(pack2_bf16(a.x, a.y), pack2_bf16(a.z, a.w), pack2_bf16(b.x, b.y), pack2_bf16(b.z, b.w));
    }
  } else {
    const int64_t total = rows * cols;
    for (int64_t i = tid; i < total; i += stride) {
      const int64_t r = i / cols, c = i - r * cols;
      dst[r * ldd + c] = __float2bfloat16_rn(src[r * lds + c]);
    }
  }
}

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__global__ void k_split_tf32(const float* __restrict__ src, int64_t lds, float* __restrict__ hi,
                             float* __restrict__ lo, int64_t ldd, int64_t rows, int64_t cols, int vec) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (vec) {  // cols % 4 == 0, aligned rows
    const int64_t per_row = cols / 4, total = rows * per_row;
    for (int64_t i = tid; i < total; i += stride) {
      const int64_t r = i / per_row, c = (i - r * per_row) * 4;
      const float4 a = *reinterpret_cast<const float4*>(src + r * lds + c);
      const float4 b = make_float4(tf32_rna(a.x), tf32_rna(a.y), tf32_rna(a.z), tf32_rna(a.w));
      *reinterpret_cast<float4*>(hi + r * ldd + c) = b;
      *reinterpret_cast<float4*>(lo + r * ldd + c) =
          make_float4(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y), __fsub_rn(a.z, b.z), __fsub_rn(a.w, b.w));
    }
  } else {
    for (int64_t i = tid; i < rows * cols; i += stride) {
      const int64_t r = i / cols, c = i - r * cols;
      const float a = src[r * lds + c], b = tf32_rna(a);
      hi[r * ldd + c] = b;
      lo[r * ldd + c] = __fsub_rn(a, b);
    }
  }
}

__global__ void k_join_tf32(const float* __restrict__ hi, const float* __restrict__ lo, int64_t ld, int64_t rows,
                            int64_t cols, float* __restrict__ out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < rows * cols; i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    out[i] = __fadd_rn(hi[r * ld + c], lo[r * ld + c]);
  }
}

__global__ void k_copy_bf16(const __nv_bfloat16* __restrict__ src, int64_t lds, __nv_bfloat16* __restrict__ dst,
                            int64_t ldd, int64_t rows, int64_t cols) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t total = rows * cols;
  for (int64_t i = tid; i < total; i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    dst[r * ldd + c] = src[r * lds + c];
  }
}

__global__ void k_bf16_to_f32(const __nv_bfloat16* __restrict__ a, int64_t ld, int64_t rows, int64_t cols,
                              float* __restrict__ out) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < rows * cols; i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    out[i] = __bfloat162float(a[r * ld + c]);
  }
}

__global__ void k_copy_f32(const float* __restrict__ a, int64_t lds, int64_t rows, int64_t cols,
                           float* __restrict__ out, int64_t ldd) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < rows * cols; i += stride) {
    const int64_t r = i / cols, c = i - r * cols;
    out[r * ldd + c] = a[r * lds + c];
  }
}

// ------------------------------------------------------------------ loss
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One block of 1024 threads: thread t sums partials t, t+1024, ... in order, then the 32 warps'
// shuffle trees and the 32 warp sums in warp order — a fixed summation order for a fixed n
// (the GEMM epilogue stores one partial per (tile, CTA, warp), so n and every slot are fixed).
__global__ void __launch_bounds__(1024) k_loss_final(int kind, const double* __restrict__ partials, int n,
                                                     int64_t rows, int64_t cols, float* __restrict__ loss) {
  __shared__ double ws[32];
  double v = 0.0;
  for (int i = threadIdx.x; i < n; i += 1024) v += partials[i];
  v = warp_sum_d(v);
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    v = ws[0];
#pragma unroll
    for (int w = 1; w < 32; ++w) v += ws[w];
    const double c = (kind == 0) ? v / (2.0 * static_cast<double>(rows) * static_cast<double>(cols))
                                 : v / static_cast<double>(rows);
    *loss = static_cast<float>(c);
  }
}

// ApplyGradientDescent: w <- fl(w - fl(lr * g))
__device__ __forceinline__ float sgd(float w, float lr, float g) { return __fsub_rn(w, __fmul_rn(lr, g)); }

// ------------------------------------------------------------------ colsum (final pass)
// The fixed summation order of colsum.cuh with 16 threads per column: a block of 1024 threads
// covers 64 columns; warp w handles columns 8 (w % 8) .. +7 and the groups of warp-set w / 8;
// the 32 group sums meet in shared memory and lanes of warp-set 0 fold them in g order.
__global__ void __launch_bounds__(1024) k_colsum_final(const float* __restrict__ ws, int chunks, int64_t cols,
                                                       float* __restrict__ out32, uint16_t* __restrict__ out16,
                                                       Round16 r16, int64_t idx_base, float* __restrict__ bias,
                                                       float lr) {
  __shared__ float tg[8][32][9];  // [column group][g][column] (+1 pad)
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int cw = w & 7, s = w >> 3, co = lane & 7, q = lane >> 3;
  const int64_t c = blockIdx.x * 64LL + cw * 8 + co;
  float t[2];
  colsum_groups2(ws, chunks, cols, c, s, t);
  tg[cw][q + 8 * s][co] = t[0];
  tg[cw][q + 8 * s + 4][co] = t[1];
  __syncthreads();
  if (s == 0 && q == 0 && c < cols) {
    float sum = tg[cw][0][co];
#pragma unroll
    for (int g = 1; g < 32; ++g) sum = __fadd_rn(sum, tg[cw][g][co]);
    if (out32) out32[c] = sum;
    if (out16) out16[c] = static_cast<uint16_t>(round16(__float_as_uint(sum), idx_base + c, r16));
    if (bias) bias[c] = sgd(bias[c], lr, sum);  // N = 1: ApplyGradientDescent on b_l (a9), fused
  }
}

// ------------------------------------------------------------------ f4 channel (backward)
// block: 32 x 8 threads = 256 columns x one 32-row chunk; each thread one column, rows in order
__global__ void k_relugrad_recv(const uint16_t* __restrict__ code, int64_t ldc, const __nv_bfloat16* __restrict__ a,
                                int64_t lda, int64_t rows, int64_t cols, __nv_bfloat16* __restrict__ dz, int64_t ldz,
                                float* __restrict__ colsum_ws) {
  const int64_t c = blockIdx.x * 256LL + threadIdx.y * 32 + threadIdx.x;
  const int64_t r0 = blockIdx.y * 32LL;
  if (c >= cols) return;
  const uint16_t* ab = reinterpret_cast<const uint16_t*>(a);
  uint16_t* zb = reinterpret_cast<uint16_t*>(dz);
  float sum = 0.f;
  for (int64_t r = r0; r < r0 + 32 && r < rows; ++r) {
    const uint32_t h = ab[r * lda + c];
    const bool pos = (h & 0x8000u) == 0 && h != 0 && h <= 0x7F80u;  // a > 0 (bf16 bits)
    const uint16_t q = pos ? code[r * ldc + c] : 0;
    zb[r * ldz + c] = q;
    sum = __fadd_rn(sum, __uint_as_float(static_cast<uint32_t>(q) << 16));
  }
  colsum_ws[blockIdx.y * cols + c] = sum;
}

// ------------------------------------------------------------------ owner reduce
__global__ void k_owner_reduce_t16(const uint16_t* __restrict__ recv, int64_t shard, int nranks,
                                   uint16_t* __restrict__ out, Round16 r16, int64_t idx_base) {
  const float inv = 1.0f / static_cast<float>(nranks);  // exact for power-of-two N (reading A7)
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t nv = shard / 8;  // shard is a multiple of 8 (bucket padding)
  for (int64_t i = tid; i < nv; i += stride) {
    float s[8];
    {
      const uint4 q = reinterpret_cast<const uint4*>(recv)[i];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = __uint_as_float((w[e >> 1] >> ((e & 1) * 16)) << 16);
    }
    for (int r = 1; r < nranks; ++r) {  // left fold in rank order
      const uint4 q = reinterpret_cast<const uint4*>(recv + r * shard)[i];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = __fadd_rn(s[e], __uint_as_float((w[e >> 1] >> ((e & 1) * 16)) << 16));
    }
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const uint32_t lo = round16(__float_as_uint(__fmul_rn(s[e], inv)), idx_base + 8 * i + e, r16);
      const uint32_t hi = round16(__float_as_uint(__fmul_rn(s[e + 1], inv)), idx_base + 8 * i + e + 1, r16);
      o[e >> 1] = lo | (hi << 16);
    }
    reinterpret_cast<uint4*>(out)[i] = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void k_owner_reduce_f32(const float* __restrict__ recv, int64_t shard, int nranks,
                                   float* __restrict__ out) {
  const float inv = 1.0f / static_cast<float>(nranks);
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < shard; i += stride) {
    float s = recv[i];
    for (int r = 1; r < nranks; ++r) s = __fadd_rn(s, recv[r * shard + i]);
    out[i] = __fmul_rn(s, inv);
  }
}

__global__ void k_sum_ranks_f32(RankPtrs src, int nranks, float* __restrict__ dst, size_t count) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += stride) {
    float s = src.p[0][i];
    for (int r = 1; r < nranks; ++r) s = __fadd_rn(s, src.p[r][i]);
    dst[i] = s;
  }
}

__global__ void k_scale_f32(float* __restrict__ x, int64_t n, float scale) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n; i += stride) x[i] = __fmul_rn(x[i], scale);
}

// ------------------------------------------------------------------ SGD apply

__global__ void k_apply_sgd_vec(float* __restrict__ W, const float* __restrict__ g32,
                                const uint16_t* __restrict__ g16, int64_t n8, __nv_bfloat16* __restrict__ wbf,
                                float lr) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = tid; i < n8; i += stride) {
    float4 w0 = reinterpret_cast<float4*>(W)[2 * i], w1 = reinterpret_cast<float4*>(W)[2 * i + 1];
    float g[8];
    if (g16) {
      const uint4 q = reinterpret_cast<const uint4*>(g16)[i];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) g[e] = __uint_as_float((w[e >> 1] >> ((e & 1) * 16)) << 16);
    } else {
      const float4 a = reinterpret_cast<const float4*>(g32)[2 * i], b = reinterpret_cast<const float4*>(g32)[2 * i + 1];
      g[0] = a.x; g[1] = a.y; g[2] = a.z; g[3] = a.w; g[4] = b.x; g[5] = b.y; g[6] = b.z; g[7] = b.w;
    }
    w0.x = sgd(w0.x, lr, g[0]); w0.y = sgd(w0.y, lr, g[1]); w0.z = sgd(w0.z, lr, g[2]); w0.w = sgd(w0.w, lr, g[3]);
    w1.x = sgd(w1.x, lr, g[4]); w1.y = sgd(w1.y, lr, g[5]); w1.z = sgd(w1.z, lr, g[6]); w1.w = sgd(w1.w, lr, g[7]);
    reinterpret_cast<float4*>(W)[2 * i] = w0;
    reinterpret_cast<float4*>(W)[2 * i + 1] = w1;
    if (wbf)
      reinterpret_cast<uint4*>(wbf)[i] = make_uint4(pack2_bf16(w0.x, w0.y), pack2_bf16(w0.z, w0.w),
                                                    pack2_bf16(w1.x, w1.y), pack2_bf16(w1.z, w1.w));
  }
}

__global__ void k_apply_sgd(float* __restrict__ W, const float* __restrict__ g32, const uint16_t* __restrict__ g16,
                            int64_t rows, int64_t cols, __nv_bfloat16* __restrict__ wbf, int64_t ldwb, float lr) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = rows * cols;
  for (int64_t i = tid; i < n; i += stride) {
    const float g = g16 ? __uint_as_float(static_cast<uint32_t>(g16[i]) << 16) : g32[i];
    const float w = sgd(W[i], lr, g);
    W[i] = w;
    if (wbf) {
      const int64_t r = i / cols, c = i - r * cols;
      wbf[r * ldwb + c] = __float2bfloat16_rn(w);
    }
  }
}

__global__ void k_apply_sgd_tf32(float* __restrict__ W, const float* __restrict__ g32,
                                 const uint16_t* __restrict__ g16, int64_t rows, int64_t cols,
                                 float* __restrict__ whi, float* __restrict__ wlo, int64_t ldw, float lr) {
  const int64_t tid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t n = rows * cols;
  for (int64_t i = tid; i < n; i += stride) {
    const float g = g16 ? __uint_as_float(static_cast<uint32_t>(g16[i]) << 16) : g32[i];
    const float w = sgd(W[i], lr, g);
    W[i] = w;
    if (whi) {
      const int64_t r = i / cols, c = i - r * cols;
      const float b = tf32_rna(w);
      whi[r * ldw + c] = b;
      wlo[r * ldw + c] = __fsub_rn(w, b);
    }
  }
}

// ------------------------------------------------------------------ masks
template <typename T>
__global__ void k_relu_mask_bits(const T* __restrict__ a, int64_t ld, int64_t rows, int64_t cols,
                                 uint32_t* __restrict__ bits) {
  const int64_t n = rows * cols;
  const int64_t words = (n + 31) / 32;
  const int lane = threadIdx.x & 31;
  const int64_t warp = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = warp; w < words; w += nwarps) {
    const int64_t i = w * 32 + lane;
    bool p = false;
    if (i < n) {
      const int64_t r = i / cols, c = i - r * cols;
      float v;
      if constexpr (sizeof(T) == 2) v = __bfloat162float(a[r * ld + c]); else v = a[r * ld + c];
      p = v > 0.f;
    }
    const uint32_t b = __ballot_sync(0xffffffffu, p);
    if (lane == 0) bits[w] = b;
  }
}

}  // namespace

cudaError_t launch_truncate16(const float* src, uint16_t* dst, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int vec = al16(src) && al16(dst);
  k_truncate16<<<blocks_for(vec ? (int64_t)n / 8 : (int64_t)n), kThreads, 0, s>>>(src, dst, (int64_t)n, vec);
  return cudaGetLastError();
}

cudaError_t launch_round16(const float* src, uint16_t* dst, size_t n, Round16 r, int64_t idx_base, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  if (!r.stochastic && idx_base == 0) return launch_truncate16(src, dst, n, s);
  k_round16<<<blocks_for((int64_t)n), kThreads, 0, s>>>(src, dst, (int64_t)n, r, idx_base);
  return cudaGetLastError();
}

cudaError_t launch_expand16(const uint16_t* src, float* dst, size_t n, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  const int vec = al16(src) && al16(dst);
  k_expand16<<<blocks_for(vec ? (int64_t)n / 8 : (int64_t)n), kThreads, 0, s>>>(src, dst, (int64_t)n, vec);
  return cudaGetLastError();
}

cudaError_t launch_cast_bf16(const float* src, int64_t lds, __nv_bfloat16* dst, int64_t ldd, int64_t rows,
                             int64_t cols, cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  const int vec = (cols % 8 == 0) && (lds % 4 == 0) && (ldd % 8 == 0) && al16(src) && al16(dst);
  k_cast_bf16<<<blocks_for(vec ? rows * cols / 8 : rows * cols), kThreads, 0, s>>>(src, lds, dst, ldd, rows, cols,
                                                                                  vec);
  return cudaGetLastError();
}

cudaError_t launch_split_tf32(const float* src, int64_t lds, float* hi, float* lo, int64_t ldd, int64_t rows,
                              int64_t cols, cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  const int vec = (cols % 4 == 0) && (lds % 4 == 0) && (ldd % 4 == 0) && al16(src) && al16(hi) && al16(lo);
  k_split_tf32<<<blocks_for(vec ? rows * cols / 4 : rows * cols), kThreads, 0, s>>>(src, lds, hi, lo, ldd, rows,
                                                                                     cols, vec);
  return cudaGetLastError();
}

cudaError_t launch_join_tf32(const float* hi, const float* lo, int64_t ld, int64_t rows, int64_t cols, float* out,
                             cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  k_join_tf32<<<blocks_for(rows * cols), kThreads, 0, s>>>(hi, lo, ld, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_apply_sgd_tf32(float* W, const float* g32, const uint16_t* g16, int64_t rows, int64_t cols,
                                  float* whi, float* wlo, int64_t ldw, float lr, cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return cudaSuccess;
  k_apply_sgd_tf32<<<blocks_for(n), kThreads, 0, s>>>(W, g32, g16, rows, cols, whi, wlo, ldw, lr);
  return cudaGetLastError();
}

cudaError_t launch_copy_bf16(const __nv_bfloat16* src, int64_t lds, __nv_bfloat16* dst, int64_t ldd, int64_t rows,
                             int64_t cols, cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  k_copy_bf16<<<blocks_for(rows * cols), kThreads, 0, s>>>(src, lds, dst, ldd, rows, cols);
  return cudaGetLastError();
}

cudaError_t launch_loss_final(int kind, const double* partials, int n, int64_t rows, int64_t cols, float* loss,
                              cudaStream_t s) {
  k_loss_final<<<1, 1024, 0, s>>>(kind, partials, n, rows, cols, loss);
  return cudaGetLastError();
}

cudaError_t launch_colsum_final(const float* ws, int chunks, int64_t cols, float* out_f32, uint16_t* out_u16,
                                cudaStream_t s, Round16 r, int64_t idx_base, float* bias, float lr) {
  if (cols == 0) return cudaSuccess;
  k_colsum_final<<<static_cast<unsigned>((cols + 63) / 64), 1024, 0, s>>>(ws, chunks, cols, out_f32, out_u16, r,
                                                                           idx_base, bias, lr);
  return cudaGetLastError();
}

cudaError_t launch_owner_reduce_t16(const uint16_t* recv, int64_t shard, int nranks, uint16_t* out,
                                    cudaStream_t s, Round16 r, int64_t idx_base) {
  if (shard == 0) return cudaSuccess;
  k_owner_reduce_t16<<<blocks_for(shard / 8), kThreads, 0, s>>>(recv, shard, nranks, out, r, idx_base);
  return cudaGetLastError();
}

cudaError_t launch_relugrad_recv(const uint16_t* code, int64_t ldc, const __nv_bfloat16* a, int64_t lda, int64_t rows,
                                 int64_t cols, __nv_bfloat16* dz, int64_t ldz, float* colsum_ws, cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  const dim3 grid(static_cast<unsigned>((cols + 255) / 256), static_cast<unsigned>((rows + 31) / 32));
  k_relugrad_recv<<<grid, dim3(32, 8), 0, s>>>(code, ldc, a, lda, rows, cols, dz, ldz, colsum_ws);
  return cudaGetLastError();
}

cudaError_t launch_owner_reduce_f32(const float* recv, int64_t shard, int nranks, float* out, cudaStream_t s) {
  if (shard == 0) return cudaSuccess;
  k_owner_reduce_f32<<<blocks_for(shard), kThreads, 0, s>>>(recv, shard, nranks, out);
  return cudaGetLastError();
}

cudaError_t launch_sum_ranks_f32(RankPtrs src, int nranks, float* dst, size_t count, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_sum_ranks_f32<<<blocks_for(static_cast<int64_t>(count)), kThreads, 0, s>>>(src, nranks, dst, count);
  return cudaGetLastError();
}

cudaError_t launch_scale_f32(float* x, int64_t n, float scale, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  k_scale_f32<<<blocks_for(n), kThreads, 0, s>>>(x, n, scale);
  return cudaGetLastError();
}

cudaError_t launch_apply_sgd(float* W, const float* g32, const uint16_t* g16, int64_t rows, int64_t cols,
                             __nv_bfloat16* wbf, int64_t ldwb, float lr, cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return cudaSuccess;
  const bool dense = (wbf == nullptr) || (ldwb == cols);
  const bool vec = dense && (n % 8 == 0) && al16(W) && (g16 ? al16(g16) : al16(g32)) && (!wbf || al16(wbf));
  if (vec)
    k_apply_sgd_vec<<<blocks_for(n / 8), kThreads, 0, s>>>(W, g32, g16, n / 8, wbf, lr);
  else
    k_apply_sgd<<<blocks_for(n), kThreads, 0, s>>>(W, g32, g16, rows, cols, wbf, ldwb, lr);
  return cudaGetLastError();
}

cudaError_t launch_relu_mask_bits(const __nv_bfloat16* a, int64_t ld, int64_t rows, int64_t cols, uint32_t* bits,
                                  cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return cudaSuccess;
  k_relu_mask_bits<__nv_bfloat16><<<blocks_for(n), kThreads, 0, s>>>(a, ld, rows, cols, bits);
  return cudaGetLastError();
}

cudaError_t launch_relu_mask_bits_f32(const float* a, int64_t ld, int64_t rows, int64_t cols, uint32_t* bits,
                                      cudaStream_t s) {
  const int64_t n = rows * cols;
  if (n == 0) return cudaSuccess;
  k_relu_mask_bits<float><<<blocks_for(n), kThreads, 0, s>>>(a, ld, rows, cols, bits);
  return cudaGetLastError();
}

cudaError_t launch_bf16_to_f32(const __nv_bfloat16* a, int64_t ld, int64_t rows, int64_t cols, float* out,
                               cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  k_bf16_to_f32<<<blocks_for(rows * cols), kThreads, 0, s>>>(a, ld, rows, cols, out);
  return cudaGetLastError();
}

cudaError_t launch_copy_f32(const float* a, int64_t lds, int64_t rows, int64_t cols, float* out, int64_t ldd,
                            cudaStream_t s) {
  if (rows * cols == 0) return cudaSuccess;
  k_copy_f32<<<blocks_for(rows * cols), kThreads, 0, s>>>(a, lds, rows, cols, out, ldd);
  return cudaGetLastError();
}

}  // namespace dflow
