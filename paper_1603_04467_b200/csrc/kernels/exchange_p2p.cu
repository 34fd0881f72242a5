// Fused NVLink gradient exchange kernels (see exchange_p2p.h).  Arithmetic is the
// same as the NCCL path (k_owner_reduce_t16): rank-order fp32 fold of the
// expanded values, x (1/N), truncate — so both paths give the same bits.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include "colsum.cuh"
#include "exchange_p2p.h"

namespace dflow {

namespace {

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t globaltimer_ns() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One thread waits until flags[0..n) >= epoch.  The loop is round 1's: the flag load and a
// short sleep.  Only every 2^14 iterations (~2 ms of waiting) does it look at the clock and
// the abort word (host memory, read over PCIe): another wait of this session has given up ->
// give up at once; timeout_ns passed -> raise abort.  (Reading %globaltimer and the abort word
// on every iteration slowed the 8-GPU proxy step by 3.5 %: profiles/r2/ab_r1_r2.)
__device__ __noinline__ bool wait_flags_bounded(const uint32_t* flags, int n, uint32_t epoch, uint32_t* abort,
                                                uint64_t timeout_ns) {
  uint64_t t0 = 0;
  uint32_t spins = 0;
  for (int r = 0; r < n; ++r) {
    while (static_cast<int32_t>(ld_acquire_sys(flags + r) - epoch) < 0) {
      if (abort != nullptr && (++spins & 0x3FFFu) == 0) {
        if (*reinterpret_cast<volatile uint32_t*>(abort) != 0) return false;  // another wait gave up
        const uint64_t now = globaltimer_ns();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > timeout_ns) {
          *reinterpret_cast<volatile uint32_t*>(abort) = 1u;  // any writer writes 1: no atomic needed
          __threadfence_system();
          return false;
        }
      }
      __nanosleep(64);
    }
  }
  return true;
}

// thread 0 of the block waits for flags[0..n) >= epoch; the block proceeds (true) or gives up
// together (false).  The verdict travels through the barrier's reduction, not shared memory:
// these kernels must use NO shared memory, or they cannot sit on an SM beside a resident GEMM
// CTA (227 KB dynamic + 1 KB static of the SM's 228 KB) and the exchange stops overlapping
// the backward.
__device__ __forceinline__ bool block_wait_flags(const uint32_t* flags, int n, uint32_t epoch, uint32_t* abort,
                                                 uint64_t timeout_ns) {
  const bool ok = threadIdx.x != 0 || wait_flags_bounded(flags, n, epoch, abort, timeout_ns);
  return __syncthreads_and(ok) != 0;
}

// The block's peer stores are ordered before thread 0 by the CTA barrier; thread 0's
// system-scope fence is cumulative over them (one fence per block, not per thread: a
// per-thread fence.sc.sys waits out every thread's own NVLink stores and cost ~30 us per
// db pass).  The last block to finish raises `phase` flags flags[j][phase][rank] = epoch
// on every rank j.
__device__ __forceinline__ void grid_signal(const P2PLayer& p, int phase, uint32_t epoch) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence_system();
    const int prev = atomicAdd(&p.done[phase], 1);
    if (prev == static_cast<int>(gridDim.x) - 1) {
      p.done[phase] = 0;
      __threadfence_system();
      for (int j = 0; j < p.world; ++j) st_release_sys(p.flags[j] + phase * kMaxRanks + p.rank, epoch);
    }
  }
}

// db_l in the fixed order of colsum.cuh (no shared memory, so it fits on an SM beside a
// resident GEMM CTA on the exchange stream): bit-identical to the fetched gradient's db.
__global__ void k_colsum_final_p2p(const float* __restrict__ ws, int chunks, int64_t cols, int64_t base_idx,
                                   const P2PLayer p, uint32_t epoch, Round16 r16) {
  const int64_t c = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) / 32 * kColsumColsPerWarp +
                    (threadIdx.x & 7);
  const float sum = colsum_warp(ws, chunks, cols, c);
  if ((threadIdx.x & 31) < 8 && c < cols) {
    const int64_t idx = base_idx + c;
    const int owner = static_cast<int>(idx / p.shard);
    p.recv[owner][static_cast<int64_t>(p.rank) * p.shard + (idx - static_cast<int64_t>(owner) * p.shard)] =
        static_cast<uint16_t>(round16(__float_as_uint(sum), idx, r16));
  }
  grid_signal(p, 0, epoch);
}

__global__ void k_owner_reduce_p2p(const P2PLayer p, uint32_t epoch, Round16 r16) {
  // every rank's contribution has landed (or the wait timed out: no fold, no signal)
  if (!block_wait_flags(p.flags[p.rank], p.world, epoch, p.abort, p.timeout_ns)) return;
  const float inv = 1.0f / static_cast<float>(p.world);
  const uint16_t* recv = p.recv[p.rank];
  const int64_t nv = p.shard / 8;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv; i += stride) {
    float s[8];
    {
      const uint4 q = reinterpret_cast<const uint4*>(recv)[i];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = __uint_as_float((w[e >> 1] >> ((e & 1) * 16)) << 16);
    }
    for (int r = 1; r < p.world; ++r) {  // left fold in rank order (reading A7)
      const uint4 q = reinterpret_cast<const uint4*>(recv + r * p.shard)[i];
      const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) s[e] = __fadd_rn(s[e], __uint_as_float((w[e >> 1] >> ((e & 1) * 16)) << 16));
    }
    uint32_t o[4];
    const int64_t idx0 = static_cast<int64_t>(p.rank) * p.shard + 8 * i;  // bucket position of element 0
#pragma unroll
    for (int e = 0; e < 8; e += 2) {
      const uint32_t lo = round16(__float_as_uint(__fmul_rn(s[e], inv)), idx0 + e, r16);
      const uint32_t hi = round16(__float_as_uint(__fmul_rn(s[e + 1], inv)), idx0 + e + 1, r16);
      o[e >> 1] = lo | (hi << 16);
    }
    if (!p.owner_apply) {
      const uint4 ov = make_uint4(o[0], o[1], o[2], o[3]);
      for (int j = 0; j < p.world; ++j)  // all-gather leg: push q_bar to every rank (NVLink stores)
        reinterpret_cast<uint4*>(p.gath[j] + static_cast<int64_t>(p.rank) * p.shard)[i] = ov;
      continue;
    }
    // owner-apply (a9 on the owner): W <- fl(W - fl(lr * g_hat)) on this rank's fp32 shard,
    // then the new bf16 operand values / fp32 biases go to every rank (the gather leg)
    const int64_t nw = p.in * p.out, nb = nw + p.out;
    float gh[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) gh[e] = __uint_as_float(((o[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu) << 16);
    if (idx0 + 8 <= nw && (p.out % 8) == 0) {
      // 8 consecutive weights of one row: two float4 of the fp32 shard, one 16-byte bf16 store
      // per rank (coalesced NVLink writes)
      float4* w4 = reinterpret_cast<float4*>(p.w32[p.rank] + idx0);
      float4 a = w4[0], b = w4[1];
      float wn[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint32_t h[4];
#pragma unroll
      for (int e = 0; e < 8; ++e) wn[e] = __fsub_rn(wn[e], __fmul_rn(p.lr_w, gh[e]));
#pragma unroll
      for (int e = 0; e < 8; e += 2) {
        const __nv_bfloat162 v = __floats2bfloat162_rn(wn[e], wn[e + 1]);  // operand copy (reading A13)
        h[e >> 1] = *reinterpret_cast<const uint32_t*>(&v);
      }
      w4[0] = make_float4(wn[0], wn[1], wn[2], wn[3]);
      w4[1] = make_float4(wn[4], wn[5], wn[6], wn[7]);
      const int64_t row = idx0 / p.out, col = idx0 - row * p.out;
      const uint4 hv = make_uint4(h[0], h[1], h[2], h[3]);
      if (p.mc_wop) {  // one multicast store: the switch writes every rank's copy
        asm volatile("multimem.st.weak.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(
                         p.mc_wop + row * p.ldwb + col),
                     "r"(hv.x), "r"(hv.y), "r"(hv.z), "r"(hv.w)
                     : "memory");
      } else {
        for (int j = 0; j < p.world; ++j) *reinterpret_cast<uint4*>(p.wop[j] + row * p.ldwb + col) = hv;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int64_t idx = idx0 + e;
        if (idx >= nb) break;  // bucket padding
        if (idx < nw) {
          float* w = p.w32[p.rank] + idx;
          const float wn = __fsub_rn(*w, __fmul_rn(p.lr_w, gh[e]));
          *w = wn;
          const int64_t row = idx / p.out, col = idx - row * p.out;
          const __nv_bfloat16 hh = __float2bfloat16_rn(wn);
          const uint16_t hb = *reinterpret_cast<const uint16_t*>(&hh);
          for (int j = 0; j < p.world; ++j) p.wop[j][row * p.ldwb + col] = hb;
        } else {
          const int64_t c = idx - nw;
          const float bn = __fsub_rn(p.b32[p.rank][c], __fmul_rn(p.lr_b, gh[e]));
          for (int j = 0; j < p.world; ++j) p.b32[j][c] = bn;
        }
      }
    }
  }
  grid_signal(p, 1, epoch);
}

__global__ void k_loss_push(const float* __restrict__ loss, const LossPeers p, int rank, int world, uint32_t epoch) {
  if (threadIdx.x != 0) return;
  const float v = loss[0];
  const int par = static_cast<int>(epoch & 1u);  // two slots: a fast rank's next push never meets an unread value
  for (int j = 0; j < world; ++j) p.slots[j][par * kMaxRanks + rank] = v;
  __threadfence_system();
  for (int j = 0; j < world; ++j) st_release_sys(p.flags[j] + rank, epoch);
}

__global__ void k_loss_gather(const float* slots, const uint32_t* flags, int world, uint32_t epoch,
                              float* __restrict__ out, uint32_t* abort, uint64_t timeout_ns) {
  if (threadIdx.x != 0) return;
  if (!wait_flags_bounded(flags, world, epoch, abort, timeout_ns)) return;
  const volatile float* sl = slots + static_cast<int>(epoch & 1u) * kMaxRanks;
  float sum = sl[0];
  for (int r = 1; r < world; ++r) sum = __fadd_rn(sum, sl[r]);
  out[0] = sum;
}

__global__ void k_gather_w32(const P2PLayer p) {
  const int64_t nw = p.in * p.out;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nw; i += stride) {
    const int owner = static_cast<int>(i / p.shard);
    if (owner != p.rank) p.w32[p.rank][i] = __ldcv(p.w32[owner] + i);
  }
}

__global__ void k_wait_flags(const uint32_t* flags, int n, uint32_t epoch, uint32_t* abort, uint64_t timeout_ns) {
  if (block_wait_flags(flags, n, epoch, abort, timeout_ns)) __threadfence_system();
}

}  // namespace

cudaError_t launch_colsum_final_p2p(const float* ws, int chunks, int64_t cols, int64_t base_idx, const P2PLayer& p,
                                    uint32_t epoch, cudaStream_t s, Round16 r) {
  // 8 warps x 8 columns per block: few blocks, so few system-scope fences in grid_signal
  const unsigned blocks = static_cast<unsigned>(std::max<int64_t>(1, (cols + 63) / 64));
  k_colsum_final_p2p<<<blocks, 256, 0, s>>>(ws, chunks, cols, base_idx, p, epoch, r);
  return cudaGetLastError();
}

cudaError_t launch_owner_reduce_p2p(const P2PLayer& p, uint32_t epoch, cudaStream_t s, Round16 r) {
  const int64_t nv = p.shard / 8;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((nv + 255) / 256, 148 * 2)));
  k_owner_reduce_p2p<<<blocks, 256, 0, s>>>(p, epoch, r);
  return cudaGetLastError();
}

cudaError_t launch_loss_push(const float* loss, const LossPeers& p, int rank, int world, uint32_t epoch,
                             cudaStream_t s) {
  k_loss_push<<<1, 32, 0, s>>>(loss, p, rank, world, epoch);
  return cudaGetLastError();
}

cudaError_t launch_loss_gather(const float* slots, const uint32_t* flags, int world, uint32_t epoch, float* out,
                               uint32_t* abort, uint64_t timeout_ns, cudaStream_t s) {
  k_loss_gather<<<1, 32, 0, s>>>(slots, flags, world, epoch, out, abort, timeout_ns);
  return cudaGetLastError();
}

cudaError_t launch_gather_w32(const P2PLayer& p, cudaStream_t s) {
  const int64_t n = p.in * p.out;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
  k_gather_w32<<<blocks, 256, 0, s>>>(p);
  return cudaGetLastError();
}

cudaError_t launch_wait_flags(const uint32_t* flags, int world, uint32_t epoch, uint32_t* abort, uint64_t timeout_ns,
                              cudaStream_t s) {
  k_wait_flags<<<1, 32, 0, s>>>(flags, world, epoch, abort, timeout_ns);
  return cudaGetLastError();
}

}  // namespace dflow
