// Bias gradient final pass (NK8, a5): db[c] = sum over the per-32-row column partials
// ws[k, c], k = 0 .. chunks-1, that the dZ-producing GEMM epilogues wrote.  ONE fixed
// summation order, shared by every kernel that forms db (fetch / N = 1 step, the fused NVLink
// db pass, the asynchronous push), so the db a step exchanges is bit-identical to the db
// dflow_fetch_gradients returns:
//
//   t_g = left fold (fp32, RN) of ws[k, c] over k = g, g + 32, g + 64, ...   (g = 0 .. 31)
//   db  = t_0 + t_1 + ... + t_31   (left fold in g order)
//
// Warp layout, no shared memory (the fused-exchange db pass runs beside a GEMM CTA that holds
// 227 KB of the SM's 228 KB): a warp owns 8 consecutive columns; lane (co = lane & 7,
// q = lane >> 3) accumulates the 8 groups g = q + 4 j, j = 0 .. 7 — so each load instruction of
// the warp reads four full 32-byte sectors (4 rows x 8 columns) and every lane keeps 8
// independent loads in flight; the 32 group sums meet by shuffles in lanes q == 0.
#pragma once
#include <cstdint>

namespace dflow {

constexpr int kColsumColsPerWarp = 8;

// Returns db[c] in lanes with (lane >> 3) == 0; every lane of the warp must call it.
__device__ __forceinline__ float colsum_warp(const float* __restrict__ ws, int chunks, int64_t cols, int64_t c) {
  const int lane = threadIdx.x & 31, q = lane >> 3;
  float t[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) t[j] = 0.f;
  if (c < cols) {
    int kb = 0;
    for (; kb + 32 <= chunks; kb += 32) {
      float a[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) a[j] = ws[static_cast<int64_t>(kb + q + 4 * j) * cols + c];
#pragma unroll
      for (int j = 0; j < 8; ++j) t[j] = __fadd_rn(t[j], a[j]);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int k = kb + q + 4 * j;
      if (k < chunks) t[j] = __fadd_rn(t[j], ws[static_cast<int64_t>(k) * cols + c]);
    }
  }
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
#pragma unroll
    for (int qq = 0; qq < 4; ++qq) {  // g = qq + 4 j: ascending g
      const float v = __shfl_sync(0xffffffffu, t[j], (lane & 7) + 8 * qq);
      s = (j == 0 && qq == 0) ? v : __fadd_rn(s, v);
    }
  }
  return s;
}

// The same t_g with more threads per column, for the kernels that may use shared memory:
// lane (co, q) of warp-set s accumulates the groups g = q + 4 j for j in {2 s, 2 s + 1}; the
// caller gathers t_0 .. t_31 and folds them in g order (identical arithmetic to colsum_warp).
__device__ __forceinline__ void colsum_groups2(const float* __restrict__ ws, int chunks, int64_t cols, int64_t c,
                                               int s, float (&t)[2]) {
  const int q = (threadIdx.x & 31) >> 3;
  t[0] = t[1] = 0.f;
  if (c >= cols) return;
  const int g0 = q + 8 * s, g1 = g0 + 4;  // j = 2s, 2s+1
  int kb = 0;
  for (; kb + 128 <= chunks; kb += 128) {  // four rounds of 32 chunks, 8 loads in flight
    float a[4], b[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      a[u] = ws[static_cast<int64_t>(kb + 32 * u + g0) * cols + c];
      b[u] = ws[static_cast<int64_t>(kb + 32 * u + g1) * cols + c];
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      t[0] = __fadd_rn(t[0], a[u]);
      t[1] = __fadd_rn(t[1], b[u]);
    }
  }
  for (; kb < chunks; kb += 32) {
    if (kb + g0 < chunks) t[0] = __fadd_rn(t[0], ws[static_cast<int64_t>(kb + g0) * cols + c]);
    if (kb + g1 < chunks) t[1] = __fadd_rn(t[1], ws[static_cast<int64_t>(kb + g1) * cols + c]);
  }
}

}  // namespace dflow
