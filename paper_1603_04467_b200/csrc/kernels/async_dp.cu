// Asynchronous data-parallel pull / push kernels (f3).  See async_dp.h.
#include <algorithm>
#include <cstdint>

#include "async_dp.h"
#include "colsum.cuh"

namespace dflow {
namespace {

__device__ __forceinline__ float ld_relaxed_sys(const float* p) {
  float v;
  asm volatile("ld.relaxed.sys.global.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}

int grid_for(int64_t n) { return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8))); }

__device__ __forceinline__ float4 ld_relaxed_sys_v4(const float* p) {
  float4 v;
  asm volatile("ld.relaxed.sys.global.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// 4 elements per thread: one 16-byte NVLink load (a 4-group never straddles an owner,
// shard % 8 == 0, nor the W / b boundary or a row, out % 4 == 0); W32 optional (only reads
// of the variable need this replica's fp32 copy; the step needs the bf16 operand and b)
__global__ void k_async_pull_v4(const AsyncLayer a, float* __restrict__ W32, float* __restrict__ b32,
                                __nv_bfloat16* __restrict__ wop, int64_t ldwb) {
  const int64_t nw = a.in * a.out, n4 = (nw + a.out) / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; q < n4; q += stride) {
    const int64_t i = 4 * q;
    const int owner = static_cast<int>(i / a.shard);
    const float4 v = ld_relaxed_sys_v4(a.master[owner] + (i - static_cast<int64_t>(owner) * a.shard));
    if (i < nw) {
      if (W32) *reinterpret_cast<float4*>(W32 + i) = v;
      const __nv_bfloat162 lo = __floats2bfloat162_rn(v.x, v.y), hi = __floats2bfloat162_rn(v.z, v.w);
      uint2 h;
      h.x = *reinterpret_cast<const uint32_t*>(&lo);
      h.y = *reinterpret_cast<const uint32_t*>(&hi);
      *reinterpret_cast<uint2*>(wop + (i / a.out) * ldwb + i % a.out) = h;  // operand copy (reading A13)
    } else {
      *reinterpret_cast<float4*>(b32 + (i - nw)) = v;
    }
  }
}

__global__ void k_async_pull(const AsyncLayer a, float* __restrict__ W32, float* __restrict__ b32,
                             __nv_bfloat16* __restrict__ wop, int64_t ldwb) {
  const int64_t nw = a.in * a.out, p = nw + a.out;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < p; i += stride) {
    const int owner = static_cast<int>(i / a.shard);
    const float v = ld_relaxed_sys(a.master[owner] + (i - static_cast<int64_t>(owner) * a.shard));
    if (i < nw) {
      if (W32) W32[i] = v;
      wop[(i / a.out) * ldwb + i % a.out] = __float2bfloat16_rn(v);  // operand copy (reading A13)
    } else {
      b32[i - nw] = v;
    }
  }
}

__global__ void k_async_publish(const AsyncLayer a, const float* __restrict__ W32, const float* __restrict__ b32) {
  const int64_t nw = a.in * a.out, p = nw + a.out;
  const int64_t lo = static_cast<int64_t>(a.rank) * a.shard;
  const int64_t hi = (lo + a.shard < p) ? lo + a.shard : p;
  float* mine = a.master[a.rank];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = lo + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < hi; i += stride)
    mine[i - lo] = i < nw ? W32[i] : b32[i - nw];
}

__global__ void k_colsum_push(const float* __restrict__ ws, int chunks, const AsyncLayer a, float lr, int coded,
                              Round16 r16) {
  const int64_t cols = a.out;
  const int64_t c = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32 * kColsumColsPerWarp +
                    (threadIdx.x & 7);
  const float s = colsum_warp(ws, chunks, cols, c);  // the fixed order of colsum.cuh
  if ((threadIdx.x & 31) < 8 && c < cols) {
    const int64_t idx = a.in * a.out + c;
    const int owner = static_cast<int>(idx / a.shard);
    const float gh = (coded && owner != a.rank) ? __uint_as_float(round16(__float_as_uint(s), idx, r16) << 16) : s;
    red_add_sys(a.master[owner] + (idx - static_cast<int64_t>(owner) * a.shard), -__fmul_rn(lr, gh));
  }
}

}  // namespace

cudaError_t launch_async_pull(const AsyncLayer& a, float* W32, float* b32, __nv_bfloat16* wop, int64_t ldwb,
                              cudaStream_t s) {
  const bool v4 = (a.out % 4) == 0 && (ldwb % 4) == 0 && (reinterpret_cast<uintptr_t>(wop) & 7) == 0 &&
                  (reinterpret_cast<uintptr_t>(W32) & 15) == 0 && (reinterpret_cast<uintptr_t>(b32) & 15) == 0;
  if (v4)
    k_async_pull_v4<<<grid_for((a.in * a.out + a.out) / 4), 256, 0, s>>>(a, W32, b32, wop, ldwb);
  else
    k_async_pull<<<grid_for(a.in * a.out + a.out), 256, 0, s>>>(a, W32, b32, wop, ldwb);
  return cudaGetLastError();
}

cudaError_t launch_colsum_push(const float* ws, int chunks, const AsyncLayer& a, float lr, int coded, Round16 r,
                               cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, (a.out + 63) / 64));  // 8 warps x 8 columns
  k_colsum_push<<<blocks, 256, 0, s>>>(ws, chunks, a, lr, coded, r);
  return cudaGetLastError();
}

cudaError_t launch_async_publish(const AsyncLayer& a, const float* W32, const float* b32, cudaStream_t s) {
  k_async_publish<<<grid_for(a.shard), 256, 0, s>>>(a, W32, b32);
  return cudaGetLastError();
}

}  // namespace dflow
