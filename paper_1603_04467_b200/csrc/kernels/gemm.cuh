// NK1-NK6: persistent, warp-specialised tcgen05 GEMM for sm_100a with fused
// epilogues (BiasAdd+Relu, loss seed, ReluGrad, db column sums, fp32 store,
// 32->16 truncation, SGD update), in two precisions:
//
//   bf16   C = A B                  kind::f16, bf16 operands (RNE), fp32 accumulate in TMEM
//   3xTF32 C = Ab Bs + As Bb + Ab Bb kind::tf32, every fp32 operand X stored as the pair
//          (Xb = tf32_rna(X), Xs = X - Xb) (reading A14); the two small products first
//
// Operand majors (what the MLP step needs):
//   forward  A_{l-1}[b,in]  (K-major)   x  W_l[in,out]      (MN-major B)
//   dgrad    dZ_l[b,out]    (K-major)   x  W_l as [in,out]  (K-major B: N=in, K=out)
//   wgrad    A_{l-1}[b,in]  (MN-major)  x  dZ_l[b,out]      (MN-major B)
//
// Roles (256 threads): warp 0 = TMA producer, warp 1 = MMA issuer (leader CTA
// only), warp 2 = TMEM allocator, warp 3 = tile scheduler (leader CTA), warps
// 4..7 = epilogue (TMEM lane quarters 0..3).  Pipelines: smem stages full/empty
// (TMA <-> MMA), a double-buffered TMEM accumulator full/empty (MMA <->
// epilogue), and a 2-deep tile-id ring fed by a global atomic counter (dynamic
// persistent schedule over an M-grouped raster, for L2 reuse).
// CG = 2 runs cta_group::2: an MMA of M = 256 spans a CTA pair; each CTA loads
// half of A (its 128 rows) and half of B (BN/2 columns); completions are
// signalled on the leader's barriers; commits multicast to both CTAs.
//
// Shared-memory tiles use the 128-byte swizzle (1024-byte atoms of 8 x 128 B);
// E = element bytes (2 bf16, 4 fp32/tf32), BK = 128/E, K_MMA = 32/E:
//   K-major  tile [rows][BK]                 : SBO = 1024 B, k-step = +32 B
//   MN-major tile [mn/(128/E)][BK][128/E]    : LBO = BK*128 B (next MN chunk),
//                                              SBO = 1024 B (next 8 k-rows), k-step = +K_MMA*128 B
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <type_traits>

#include "async_dp.h"
#include "gemm.h"
#include "ptx.cuh"

namespace dflow {

template <int BN, int CG, bool TF32, bool STG = false>
struct GemmCfg {
  static constexpr int E = TF32 ? 4 : 2;          // operand element bytes
  static constexpr int BM = 128;                  // rows per CTA
  static constexpr int BK = 128 / E;              // one 128-byte swizzle row of K
  static constexpr int KMMA = 32 / E;             // K per tcgen05.mma
  static constexpr int CHUNK = 128 / E;           // MN elements per 128-byte MN-major row
  static constexpr int NOPS = TF32 ? 2 : 1;       // operand parts (big, small)
  static constexpr int BN_CTA = BN / CG;          // B columns loaded by each CTA
  static constexpr int A_TILE = BM * BK * E;      // 16 KB
  static constexpr int B_TILE = BN_CTA * BK * E;  // 16 KB (BN_CTA = 128)
  static constexpr int STAGE_BYTES = NOPS * (A_TILE + B_TILE);
  // BN = 512 (bf16 CTA pair): the tile's accumulator is two N = 256 halves filling all 512
  // TMEM columns (no second buffer); each half is handed to the epilogue / back to the MMA on
  // its own barrier, so the next tile's first half starts while the epilogue drains the second.
  // Each CTA loads its B columns as NH pieces of 128 (piece h feeds half h), so a pair tile
  // reads 25 % fewer operand bytes per FLOP than two 256 x 256 tiles.
  static constexpr int NH = BN > 256 ? 2 : 1;     // accumulator halves per tile
  static constexpr int MMA_N = BN > 256 ? 256 : BN;
  static constexpr int PIECE_COLS = BN_CTA / NH;  // B columns per piece (128)
  static constexpr int TMEM_COLS = NH == 2 ? 512 : 2 * BN;  // two buffers, or the two halves of one
  // tile-id ring depth: the producer runs ~1 tile ahead of the MMA and the epilogue ~1 tile
  // behind it, so the ring must hold >= 3 ids or the producer stalls at tile boundaries
  static constexpr int SCHED_DEPTH = 4;
  static constexpr int BAR_BYTES_MAX = (2 * 8 + 4 + 2 * SCHED_DEPTH) * 8 + 16 + 4 * SCHED_DEPTH;
  // EPI_TRUNC16_P2P staging: per epilogue warp a 32-row x 64-column u16 block (row pitch
  // 72 halves), so peer stores go out as full 128-byte row segments; EPI_ASYNC_PUSH reuses
  // it as 32 rows x 32 fp32 deltas (same 144-byte pitch) for bulk reductions
  static constexpr int STG_PITCH = 72;
  static constexpr int STG_BYTES = STG ? 4 * 32 * STG_PITCH * 2 : 0;
  // as many pipeline stages as the 227 KB opt-in shared memory holds (bf16 256x256 pair: 7,
  // or 6 beside the P2P staging; 3xTF32: 4)
  static constexpr int SMEM_MAX = 227 * 1024;
  static constexpr int STAGE_BUDGET = SMEM_MAX - 1024 - BAR_BYTES_MAX - STG_BYTES;
  static constexpr int STAGES = STAGE_BUDGET / STAGE_BYTES > 8 ? 8 : STAGE_BUDGET / STAGE_BYTES;
  static constexpr int BAR_BYTES = (2 * STAGES + 4 + 2 * SCHED_DEPTH) * 8 + 16 + 4 * SCHED_DEPTH;
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + BAR_BYTES + STG_BYTES + 1024;  // + alignment slack
  static_assert(SMEM_BYTES <= SMEM_MAX, "shared memory budget");
  static constexpr int SCHED_CONSUMERS = (CG == 2) ? 11 : 6;  // producer warp x CG + MMA warp + 4 epilogue warps x CG
  // k-blocks per TMEM accumulation chunk: 3xTF32 flushes every 128 of K into fp32
  // registers (reading A25); bf16 accumulates the whole K in TMEM
  static constexpr int KB_PER_CHUNK = TF32 ? 4 : (1 << 30);
  static_assert(TMEM_COLS >= 32 && TMEM_COLS <= 512 && (TMEM_COLS & (TMEM_COLS - 1)) == 0, "tmem cols");
  static_assert(BN % 32 == 0 && BN_CTA % CHUNK == 0, "tile N");
};

__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int group, int& tm, int& tn) {
  const int per_group = group * tiles_n;
  const int g = t / per_group;
  const int first_m = g * group;
  const int gsize = min(tiles_m - first_m, group);
  const int r = t - g * per_group;
  tm = first_m + r % gsize;
  tn = r / gsize;
}

__device__ __forceinline__ float u32_as_f32(uint32_t x) { return __uint_as_float(x); }

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

// Epilogue traffic that is touched once per launch (targets, masks, the stored activations /
// gradients / weights) can go through L2 with the evict-first (streaming) policy so it does
// not push the operand panels the next tiles reuse out of L2 (args.evict)
template <class T>
__device__ __forceinline__ T ld_once(const T* p, bool cs) {
  return cs ? __ldcs(p) : __ldg(p);
}
template <class T>
__device__ __forceinline__ void st_once(T* p, const T& v, bool cs) {
  if (cs) __stcs(p, v);
  else *p = v;
}

// 256-bit (32-byte) global accesses (sm_100: LDG/STG .256). Each lane of an epilogue warp
// owns one row, so a warp-wide access touches 32 different lines; at 32 bytes per lane the
// L1 data path moves twice the bytes per wavefront of a 16-byte access (args.vec_* == 2).
__device__ __forceinline__ void ld_v8(const void* p, bool cs, uint32_t* r) {
  if (cs)
    asm volatile("ld.global.cs.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
  else
    asm volatile("ld.global.nc.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}
__device__ __forceinline__ void st_v8(void* p, const uint32_t* r, bool cs) {
  if (cs)
    asm volatile("st.global.cs.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
  else
    asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(r[0]), "r"(r[1]), "r"(r[2]),
                 "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
                 : "memory");
}

// tf32 round-to-nearest (ties away), returned in an fp32 container (low 13 bits 0)
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// Store 32 consecutive operand values of one row: bf16 (RNE) or the 3xTF32 pair.
// Returns (in v) the value the next GEMM will see for each element: bf16-rounded
// value, or the exact fp32 value (= big + small) in the 3xTF32 path.
template <bool TF32>
__device__ __forceinline__ void store_operand(float (&v)[32], void* hi_base, void* lo_base, int64_t ld, int64_t gm,
                                              int gn, int N, int vec, bool trunc = false, bool cs = false) {
  const bool full = gn + 32 <= N;
  if constexpr (!TF32) {
    // bf16 operand: RNE (reading A19), or — where the tensor crosses a device (f4 channel,
    // reading A33) — the channel's 16-bit truncation code, which is a bf16 bit pattern.
    // Packed pairwise (one cvt per two values); v is handed back as the stored values (the
    // fused db column sums use them; dead and dropped by the compiler elsewhere)
    uint32_t w[16];
#pragma unroll
    for (int e = 0; e < 16; ++e)
      w[e] = trunc ? ((__float_as_uint(v[2 * e]) >> 16) | (__float_as_uint(v[2 * e + 1]) & 0xFFFF0000u))
                   : pack_bf16x2(v[2 * e], v[2 * e + 1]);
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      v[2 * e] = __uint_as_float(w[e] << 16);
      v[2 * e + 1] = __uint_as_float(w[e] & 0xFFFF0000u);
    }
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(hi_base) + gm * ld + gn;
    if (full && vec == 2) {
      st_v8(o, w, cs);
      st_v8(o + 16, w + 8, cs);
    } else if (full && vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 8)
        st_once(reinterpret_cast<uint4*>(o + j), make_uint4(w[j / 2], w[j / 2 + 1], w[j / 2 + 2], w[j / 2 + 3]), cs);
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (gn + j < N) o[j] = __float2bfloat16_rn(v[j]);
    }
  } else {
    float* oh = reinterpret_cast<float*>(hi_base) + gm * ld + gn;
    float* ol = reinterpret_cast<float*>(lo_base) + gm * ld + gn;
    if (full && vec) {
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        float b[4], s[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          b[e] = tf32_rna(v[j + e]);
          s[e] = __fsub_rn(v[j + e], b[e]);
        }
        st_once(reinterpret_cast<float4*>(oh + j), make_float4(b[0], b[1], b[2], b[3]), cs);
        st_once(reinterpret_cast<float4*>(ol + j), make_float4(s[0], s[1], s[2], s[3]), cs);
      }
    } else {
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (gn + j < N) {
          const float b = tf32_rna(v[j]);
          oh[j] = b;
          ol[j] = __fsub_rn(v[j], b);
        }
    }
  }
}

template <int BN, int CG, bool TF32, bool A_MN, bool B_MN, int EPI>
__global__ void __launch_bounds__(256, 1)
    gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                const __grid_constant__ CUtensorMap tmA2, const __grid_constant__ CUtensorMap tmB2,
                const GemmArgs args) {
  using Cfg = GemmCfg<BN, CG, TF32, EPI == EPI_TRUNC16_P2P || EPI == EPI_ASYNC_PUSH>;
  constexpr int BM = Cfg::BM, BK = Cfg::BK, BN_CTA = Cfg::BN_CTA, STAGES = Cfg::STAGES;
  constexpr int A_TILE = Cfg::A_TILE, B_TILE = Cfg::B_TILE, STAGE_BYTES = Cfg::STAGE_BYTES;
  constexpr int CHUNK = Cfg::CHUNK, KMMA = Cfg::KMMA, NOPS = Cfg::NOPS;
  constexpr int CHUNK_BYTES = BK * 128;  // one MN-major chunk: BK k-rows of 128 bytes
  using OpT = typename std::conditional<TF32, float, __nv_bfloat16>::type;

  extern __shared__ uint8_t smem_raw[];
  uint8_t* tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(tiles + STAGES * STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + STAGES;
  uint64_t* tfull = bars + 2 * STAGES;
  uint64_t* tempty = bars + 2 * STAGES + 2;
  constexpr int SD = Cfg::SCHED_DEPTH;
  uint64_t* sched_full = bars + 2 * STAGES + 4;        // [SD] tile id published (count 1)
  uint64_t* sched_empty = bars + 2 * STAGES + 4 + SD;  // [SD] tile id consumed (leader; SCHED_CONSUMERS arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * STAGES + 4 + 2 * SD);
  int* sched_tile = reinterpret_cast<int*>(tmem_slot + 4);  // [SD]
  uint16_t* stg_base = reinterpret_cast<uint16_t*>(bars) + Cfg::BAR_BYTES / 2;  // P2P staging

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t cta_rank = (CG == 2) ? ptx::cluster_ctarank() : 0;
  const int cluster_id = blockIdx.x / CG;
  const int num_clusters = gridDim.x / CG;
  const int num_tiles = args.tiles_m * args.tiles_n;
  const int num_kb = (args.K + BK - 1) / BK;

  // Dynamic tile scheduler: the leader CTA's warp 3 draws tile ids from a global
  // atomic counter (first tile = cluster id) and publishes them through a 2-deep
  // smem ring in every CTA of the cluster, so the set of tiles in flight stays a
  // contiguous window of the M-grouped raster (L2 reuse) even when SMs drift.
  const uint32_t sched_empty_leader =
      (CG == 2) ? ptx::mapa_shared(ptx::smem_u32(&sched_empty[0]), 0) : ptx::smem_u32(&sched_empty[0]);
  auto next_tile = [&](int& slot, uint32_t& ph, bool whole_warp) -> int {
    ptx::mbar_wait_cluster(ptx::smem_u32(&sched_full[slot]), ph);
    const int t = *reinterpret_cast<volatile int*>(&sched_tile[slot]);
    if (whole_warp) __syncwarp();
    if (!whole_warp || lane == 0) {
      if constexpr (CG == 2) ptx::mbar_arrive_cluster(sched_empty_leader + slot * 8);
      else ptx::mbar_arrive(ptx::smem_u32(&sched_empty[slot]));
    }
    if (++slot == SD) {
      slot = 0;
      ph ^= 1;
    }
    return t;
  };

  if (warp == 0 && lane == 0) {
    ptx::prefetch_tmap(&tmA);
    ptx::prefetch_tmap(&tmB);
    if constexpr (TF32) {
      ptx::prefetch_tmap(&tmA2);
      ptx::prefetch_tmap(&tmB2);
    }
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      ptx::mbar_init(ptx::smem_u32(&full[s]), 1);
      ptx::mbar_init(ptx::smem_u32(&empty[s]), 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(ptx::smem_u32(&tfull[a]), 1);
      ptx::mbar_init(ptx::smem_u32(&tempty[a]), 4 * CG);
    }
    for (int a = 0; a < SD; ++a) {
      ptx::mbar_init(ptx::smem_u32(&sched_full[a]), 1);
      ptx::mbar_init(ptx::smem_u32(&sched_empty[a]), Cfg::SCHED_CONSUMERS);
    }
    ptx::fence_mbarrier_init();
  }
  if (warp == 2) ptx::tmem_alloc<CG>(ptx::smem_u32(tmem_slot), Cfg::TMEM_COLS);
  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    // ===================== TMA producer (warp-uniform; one elected lane issues) =====================
    {
      int stage = 0;
      uint32_t phase = 0;
      int sslot = 0;
      uint32_t sph = 0;
      const uint32_t full0_local = ptx::smem_u32(&full[0]);
      const uint32_t full0 = (CG == 2) ? ptx::mapa_shared(full0_local, 0) : full0_local;
      const uint32_t s_tiles = ptx::smem_u32(tiles);
      // This CTA's (m0, n0) of tile t.
      // n0 = this CTA's first B column of piece 0; piece p starts at n0 + p * (BN / NH)
      auto origin = [&](int t, int& m0, int& n0) {
        int tm, tn;
        tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, tm, tn);
        m0 = tm * (BM * CG) + cta_rank * BM;
        n0 = tn * BN + cta_rank * Cfg::PIECE_COLS;
      };
      constexpr int PIECE_STRIDE = BN / Cfg::NH;              // global columns between pieces
      constexpr int PIECE_BYTES = Cfg::PIECE_COLS * BK * Cfg::E;  // smem bytes of one piece
      // L2 prefetch cursor: walks the same (tile, k-block) sequence `pf` k-blocks ahead of
      // the loads, so the loads hit L2 instead of waiting out DRAM latency. It draws the tile
      // ids from the scheduler ring (one tile ahead of the loads, which take them from t_next).
      const int pf = (args.prefetch > 0 && num_kb > args.prefetch) ? args.prefetch : 0;
      int t = next_tile(sslot, sph, true);
      int pt = t, pkb = 0, pm0 = 0, pn0 = 0, t_next = t;
      if (pf && pt < num_tiles) origin(pt, pm0, pn0);
      auto prefetch_step = [&]() {
        if (pt >= num_tiles) return;
        const int k0 = pkb * BK;
        if (ptx::elect_one()) {
#pragma unroll
          for (int part = 0; part < NOPS; ++part) {
            const CUtensorMap* ma = part ? &tmA2 : &tmA;
            const CUtensorMap* mb = part ? &tmB2 : &tmB;
#pragma unroll
            for (int i = 0; i < (A_MN ? BM / CHUNK : 1); ++i)
              ptx::tma_prefetch_2d(ma, A_MN ? (pm0 + CHUNK * i) : k0, A_MN ? k0 : pm0);
#pragma unroll
            for (int pc = 0; pc < Cfg::NH; ++pc)
#pragma unroll
              for (int i = 0; i < (B_MN ? Cfg::PIECE_COLS / CHUNK : 1); ++i)
                ptx::tma_prefetch_2d(mb, B_MN ? (pn0 + pc * PIECE_STRIDE + CHUNK * i) : k0,
                                     B_MN ? k0 : pn0 + pc * PIECE_STRIDE);
          }
        }
        __syncwarp();
        if (++pkb == num_kb) {
          pkb = 0;
          pt = next_tile(sslot, sph, true);
          t_next = pt;
          if (pt < num_tiles) origin(pt, pm0, pn0);
        }
      };
      for (int i = 0; i < pf; ++i) prefetch_step();
      while (t < num_tiles) {
        int m0, n0;
        origin(t, m0, n0);
        for (int kb = 0; kb < num_kb; ++kb) {
          if (pf) prefetch_step();
          if (args.debug & 4) ptx::mbar_wait_spin(ptx::smem_u32(&empty[stage]), phase ^ 1);
          else ptx::mbar_wait(ptx::smem_u32(&empty[stage]), phase ^ 1);
          const uint32_t fb = full0 + stage * 8;
          const uint32_t s0 = s_tiles + stage * STAGE_BYTES;
          const int k0 = kb * BK;
          if (ptx::elect_one()) {
            if (args.debug & 1) {  // profiling: MMA on stale smem, no TMA traffic
              if (cta_rank == 0) ptx::mbar_arrive(ptx::smem_u32(&full[stage]));
            } else {
              if (cta_rank == 0) ptx::mbar_arrive_expect_tx(ptx::smem_u32(&full[stage]), CG * STAGE_BYTES);
#pragma unroll
              for (int part = 0; part < NOPS; ++part) {
                const CUtensorMap* ma = part ? &tmA2 : &tmA;
                const CUtensorMap* mb = part ? &tmB2 : &tmB;
                const uint32_t sa = s0 + part * A_TILE;
                const uint32_t sb = s0 + NOPS * A_TILE + part * B_TILE;
#pragma unroll
                for (int i = 0; i < (A_MN ? BM / CHUNK : 1); ++i) {
                  const uint32_t dst = sa + i * CHUNK_BYTES;
                  const int c0 = A_MN ? (m0 + CHUNK * i) : k0;
                  const int c1 = A_MN ? k0 : m0;
                  if constexpr (CG == 2) ptx::tma_load_2d_cg2(dst, ma, fb, c0, c1);
                  else ptx::tma_load_2d(dst, ma, fb, c0, c1);
                }
#pragma unroll
                for (int pc = 0; pc < Cfg::NH; ++pc)
#pragma unroll
                  for (int i = 0; i < (B_MN ? Cfg::PIECE_COLS / CHUNK : 1); ++i) {
                    const uint32_t dst = sb + pc * PIECE_BYTES + i * CHUNK_BYTES;
                    const int nn = n0 + pc * PIECE_STRIDE;
                    const int c0 = B_MN ? (nn + CHUNK * i) : k0;
                    const int c1 = B_MN ? k0 : nn;
                    if constexpr (CG == 2) ptx::tma_load_2d_cg2(dst, mb, fb, c0, c1);
                    else ptx::tma_load_2d(dst, mb, fb, c0, c1);
                  }
              }
            }
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        t = pf ? t_next : next_tile(sslot, sph, true);
      }
    }
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA; warp-uniform, one elected lane issues) =====================
    if (cta_rank == 0) {
      constexpr uint32_t idesc = ptx::make_idesc(BM * CG, Cfg::MMA_N, A_MN, B_MN, TF32);
      // smem descriptors of stage 0; a stage / k step only moves the start address
      // (field [0,14) = addr >> 4, < 2^14 for any shared address, so plain adds never carry)
      auto mn_desc = [&](uint32_t addr) {
        // MN-major tf32 operands use the 32-byte-atom 128B swizzle (4-row period, SBO = 4 rows)
        return TF32 ? ptx::smem_desc_sw128_base32(addr, CHUNK_BYTES, 512) : ptx::smem_desc_sw128(addr, CHUNK_BYTES, 1024);
      };
      const uint32_t s_tiles = ptx::smem_u32(tiles);
      uint64_t a_desc0[NOPS], b_desc0[NOPS];
#pragma unroll
      for (int part = 0; part < NOPS; ++part) {
        const uint32_t a = s_tiles + part * A_TILE;
        const uint32_t b = s_tiles + NOPS * A_TILE + part * B_TILE;
        a_desc0[part] = A_MN ? mn_desc(a) : ptx::smem_desc_sw128(a, 16, 1024);
        b_desc0[part] = B_MN ? mn_desc(b) : ptx::smem_desc_sw128(b, 16, 1024);
      }
      constexpr uint32_t KA_STEP = (A_MN ? KMMA * 128 : 32) >> 4;
      constexpr uint32_t KB_STEP = (B_MN ? KMMA * 128 : 32) >> 4;
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      int sslot = 0;
      uint32_t sph = 0;
      for (;;) {
        const int t = next_tile(sslot, sph, true);
        if (t >= num_tiles) break;
        if (num_kb == 0) continue;
        if constexpr (Cfg::NH == 2) {
          // two N = 256 halves in TMEM columns [0, 256) and [256, 512); half 1 waits for the
          // epilogue to hand it back only after half 0's first MMAs are issued
          constexpr uint32_t HB = static_cast<uint32_t>((Cfg::PIECE_COLS * BK * Cfg::E) >> 4);  // piece offset
          ptx::mbar_wait(ptx::smem_u32(&tempty[0]), acc_phase ^ 1);
          ptx::tc_fence_after();
          for (int kb = 0; kb < num_kb; ++kb) {
            ptx::mbar_wait(ptx::smem_u32(&full[stage]), phase);
            ptx::tc_fence_after();
            const uint64_t soff = static_cast<uint64_t>((stage * STAGE_BYTES) >> 4);
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / KMMA; ++k)
                ptx::mma_ss<CG, false>(tmem_base, a_desc0[0] + soff + k * KA_STEP, b_desc0[0] + soff + k * KB_STEP,
                                       idesc, (kb == 0 && k == 0) ? 0u : 1u);
            }
            __syncwarp();
            if (kb == 0) {
              ptx::mbar_wait(ptx::smem_u32(&tempty[1]), acc_phase ^ 1);
              ptx::tc_fence_after();
            }
            if (ptx::elect_one()) {
#pragma unroll
              for (int k = 0; k < BK / KMMA; ++k)
                ptx::mma_ss<CG, false>(tmem_base + 256, a_desc0[0] + soff + k * KA_STEP,
                                       b_desc0[0] + soff + HB + k * KB_STEP, idesc, (kb == 0 && k == 0) ? 0u : 1u);
              ptx::mma_commit<CG>(ptx::smem_u32(&empty[stage]), 0x3);
              if (kb == num_kb - 1) {
                ptx::mma_commit<CG>(ptx::smem_u32(&tfull[0]), 0x3);
                ptx::mma_commit<CG>(ptx::smem_u32(&tfull[1]), 0x3);
              }
            }
            __syncwarp();
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          acc_phase ^= 1;
          continue;
        }
        // K is processed in chunks, each accumulated from zero into one of the two TMEM
        // buffers (bf16: one chunk per tile; 3xTF32: 128-wide K chunks summed in fp32 by the
        // epilogue, because the tensor core truncates when it accumulates, reading A25)
        uint32_t d = 0;
        for (int kb = 0; kb < num_kb; ++kb) {
          const bool chunk_start = (kb % Cfg::KB_PER_CHUNK) == 0;
          const bool chunk_end = (kb % Cfg::KB_PER_CHUNK) == Cfg::KB_PER_CHUNK - 1 || kb == num_kb - 1;
          if (chunk_start) {
            ptx::mbar_wait(ptx::smem_u32(&tempty[acc]), acc_phase ^ 1);
            ptx::tc_fence_after();
            d = tmem_base + acc * BN;
          }
          if (args.debug & 4) ptx::mbar_wait_spin(ptx::smem_u32(&full[stage]), phase);
          else ptx::mbar_wait(ptx::smem_u32(&full[stage]), phase);
          ptx::tc_fence_after();
          const uint64_t soff = static_cast<uint64_t>((stage * STAGE_BYTES) >> 4);
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / KMMA; ++k) {
              const uint32_t first = (chunk_start && k == 0) ? 0u : 1u;
              const uint64_t ao = soff + k * KA_STEP, bo = soff + k * KB_STEP;
              if constexpr (TF32) {
                // small products first (reading A14), then big * big
                ptx::mma_ss<CG, true>(d, a_desc0[0] + ao, b_desc0[1] + bo, idesc, first);
                ptx::mma_ss<CG, true>(d, a_desc0[1] + ao, b_desc0[0] + bo, idesc, 1u);
                ptx::mma_ss<CG, true>(d, a_desc0[0] + ao, b_desc0[0] + bo, idesc, 1u);
              } else {
                ptx::mma_ss<CG, false>(d, a_desc0[0] + ao, b_desc0[0] + bo, idesc, first);
              }
            }
            ptx::mma_commit<CG>(ptx::smem_u32(&empty[stage]), 0x3);
            if (chunk_end) ptx::mma_commit<CG>(ptx::smem_u32(&tfull[acc]), 0x3);
          }
          __syncwarp();
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
          if (chunk_end) {
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 3) {
    // ===================== tile scheduler (one thread of the leader CTA) =====================
    if (cta_rank == 0 && lane == 0) {
      int slot = 0;
      uint32_t ph = 0;
      // Die-aware dynamic schedule (args.die_map; experimental, off by default): the raster's tiles are split
      // at args.die_split into [0, split) for the clusters on die 0 and [split, num_tiles) for
      // die 1 (in proportion to the dies' clusters), so the operand panels of a die's tiles are
      // fetched across the die-to-die fabric once, not by both dies; a cluster draws from its
      // own die's counter (sched[die]) and steals from the other's once its own is exhausted.
      // Without a die map one range holds every tile.
      int my_die = 0;
      if (args.die_map) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        my_die = args.die_map[sm] & 1;
      }
      const int split = args.die_map ? args.die_split : num_tiles;
      // die_mode 2: instead of two ranges of the raster, the two dies sweep the same M-groups
      // side by side, die 0 over N-tiles [0, split), die 1 over [split, tiles_n): the A panels
      // of a group are shared by both dies, every B panel is read by one die only
      const bool nsplit = args.die_map && args.die_mode == 2;
      const int tm_n = args.tiles_m, tn_n = args.tiles_n, grp = args.group_m;
      auto nsplit_tile = [&](int d, int i) -> int {  // the i-th tile of die d -> raster id
        const int n_lo = d ? split : 0, nd = d ? tn_n - split : split;
        const int last_g = (tm_n - 1) / grp;
        const int g = min(i / (grp * nd), last_g);
        const int r = i - g * grp * nd;
        const int gsize = min(tm_n - g * grp, grp);
        const int m_off = r % gsize, n = n_lo + r / gsize;
        return g * grp * tn_n + n * gsize + m_off;
      };
      auto draw = [&]() -> int {
        for (int k = 0; k < 2; ++k) {
          const int d = my_die ^ k;
          int lo, hi;
          if (nsplit) {
            lo = 0;
            hi = tm_n * (d ? tn_n - split : split);
          } else {
            lo = d ? split : 0;
            hi = d ? num_tiles : split;
          }
          if (hi <= lo) continue;
          const int i = atomicAdd(&args.sched[d], 1);
          if (lo + i < hi) return nsplit ? nsplit_tile(d, i) : lo + i;
        }
        return num_tiles;
      };
      int t = args.sched ? draw() : cluster_id;
      for (;;) {
        ptx::mbar_wait(ptx::smem_u32(&sched_empty[slot]), ph ^ 1);
#pragma unroll
        for (int r = 0; r < CG; ++r) {
          const uint32_t tile_addr = (CG == 2) ? ptx::mapa_shared(ptx::smem_u32(&sched_tile[slot]), r)
                                               : ptx::smem_u32(&sched_tile[slot]);
          const uint32_t full_addr = (CG == 2) ? ptx::mapa_shared(ptx::smem_u32(&sched_full[slot]), r)
                                               : ptx::smem_u32(&sched_full[slot]);
          ptx::st_shared_cluster(tile_addr, static_cast<uint32_t>(t));
          ptx::mbar_arrive_cluster(full_addr);
        }
        if (t >= num_tiles) break;
        t = args.sched ? draw() : t + num_clusters;
        if (++slot == SD) {
          slot = 0;
          ph ^= 1;
        }
      }
      if (args.sched) {
        // the last cluster to finish resets the counters for the next launch on this stream
        __threadfence();
        if (atomicAdd(&args.sched[2], 1) == num_clusters - 1) {
          atomicExch(&args.sched[0], 0);
          atomicExch(&args.sched[1], 0);
          atomicExch(&args.sched[2], 0);
        }
      }
    }
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> registers -> global =====================
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const bool ev = args.evict != 0;
    const uint32_t tempty_leader =
        (CG == 2) ? ptx::mapa_shared(ptx::smem_u32(&tempty[0]), 0) : ptx::smem_u32(&tempty[0]);
    int acc = 0;
    uint32_t acc_phase = 0;
    double loss_acc = 0.0;
    int sslot = 0;
    uint32_t sph = 0;
    for (;;) {
      const int t = next_tile(sslot, sph, true);
      if (t >= num_tiles) break;
      int tm, tn;
      tile_coords(t, args.tiles_m, args.tiles_n, args.group_m, tm, tn);
      const int gm = tm * (BM * CG) + cta_rank * BM + q * 32 + lane;
      const bool row_ok = gm < args.M;
      const uint32_t tmem_row = tmem_base + (static_cast<uint32_t>(q * 32) << 16);
      // the tile's bias, lane l holding column 32k + l of chunk k: loaded before the
      // accumulator wait (its latency hides behind the mainloop), broadcast per chunk by shfl
      constexpr bool HAS_BIAS = EPI == EPI_BIAS_RELU || EPI == EPI_BIAS_RELU_LOSS;
      float bl[HAS_BIAS ? BN / 32 : 1];
      if constexpr (HAS_BIAS) {
#pragma unroll
        for (int k = 0; k < BN / 32; ++k) {
          const int gn = tn * BN + k * 32 + lane;
          bl[k] = gn < args.N ? __ldg(args.bias + gn) : 0.f;
        }
      }
      auto hand_back = [&](int slot) {  // hand a TMEM buffer (or half) back to the MMA warp
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          // relaxed: the reads it releases completed at tcgen05.wait::ld; a release.cluster
          // arrive would add a GPU-scope MEMBAR per TMEM hand-back (per 128-deep K chunk on
          // the 3xTF32 path)
          if constexpr (CG == 2) ptx::mbar_arrive_cluster_relaxed(tempty_leader + slot * 8);
          else ptx::mbar_arrive(ptx::smem_u32(&tempty[slot]));
        }
      };
      auto release_tmem = [&]() {
        if constexpr (Cfg::NH == 2) {  // (half 0 went back at the half switch)
          hand_back(1);
          acc_phase ^= 1;
        } else {
          hand_back(acc);
          acc ^= 1;
          if (acc == 0) acc_phase ^= 1;
        }
      };
      // NH == 2: before chunk BN / 64 (the first of half 1) give half 0 back and wait for half 1
      auto half_switch = [&](int c) {
        if constexpr (Cfg::NH == 2) {
          if (c == BN / 64) {
            hand_back(0);
            ptx::mbar_wait(ptx::smem_u32(&tfull[1]), acc_phase);
            ptx::tc_fence_after();
          }
        }
      };
      // 3xTF32: the K chunks arrive one TMEM buffer at a time; sum them in fp32 (RN)
      float kacc[TF32 ? BN : 1];
      if constexpr (TF32) {
        const int nchunks = (num_kb + Cfg::KB_PER_CHUNK - 1) / Cfg::KB_PER_CHUNK;
#pragma unroll
        for (int j = 0; j < BN; ++j) kacc[j] = 0.f;
        for (int ch = 0; ch < nchunks; ++ch) {
          ptx::mbar_wait(ptx::smem_u32(&tfull[acc]), acc_phase);
          ptx::tc_fence_after();
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) {
            uint32_t r[32];
            ptx::tmem_ld_32x32b_x32(tmem_row + acc * BN + c * 32, r);
            ptx::tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) kacc[c * 32 + j] = __fadd_rn(kacc[c * 32 + j], u32_as_f32(r[j]));
          }
          release_tmem();
        }
      } else if (num_kb > 0) {
        ptx::mbar_wait(ptx::smem_u32(&tfull[acc]), acc_phase);
        ptx::tc_fence_after();
        if (args.debug & 2) {  // profiling: hand the accumulator straight back
          half_switch(BN / 64);
          release_tmem();
          continue;
        }
      }
      // EPI_BIAS_RELU_LOSS: the 32 targets y[gm, gn .. gn+31] of a column chunk, loaded one
      // chunk ahead of its use so the DRAM latency overlaps the previous chunk's work
      auto load_y = [&](int c, float (&yv)[32]) {
        const int gn = tn * BN + c * 32;
        if (args.loss_kind != 0 || !row_ok || gn >= args.N) return;
        if (args.debug & 8) {  // profiling: targets taken as 0, no loads
#pragma unroll
          for (int j = 0; j < 32; ++j) yv[j] = 0.f;
          return;
        }
        const float* yrow = args.y + static_cast<int64_t>(gm) * args.ldy + gn;
        if (gn + 32 <= args.N && args.vec_y == 2) {
#pragma unroll
          for (int j = 0; j < 32; j += 8) ld_v8(yrow + j, ev, reinterpret_cast<uint32_t*>(yv + j));
        } else if (gn + 32 <= args.N && args.vec_y) {
#pragma unroll
          for (int j = 0; j < 32; j += 4) {
            const float4 t4 = ld_once(reinterpret_cast<const float4*>(yrow + j), ev);
            yv[j] = t4.x; yv[j + 1] = t4.y; yv[j + 2] = t4.z; yv[j + 3] = t4.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) yv[j] = (gn + j < args.N) ? __ldg(yrow + j) : 0.f;
        }
      };
      // the chunk's streamed operand, loaded one chunk ahead of its use: the targets (loss
      // seed), the bf16 Relu mask (dgrad) or the fp32 master weights (SGD apply) — on the
      // vectorised full-chunk path; ragged chunks load inline in column_chunk
      const bool pre_vec = EPI == EPI_RELUGRAD ? (!TF32 && args.vec_mask != 0)
                                               : EPI == EPI_SGD_APPLY ? args.vec_out32 != 0 : false;
      auto load_pre = [&](int c, float (&p)[32]) {
        if constexpr (EPI == EPI_BIAS_RELU_LOSS) {
          load_y(c, p);
        } else if constexpr (EPI == EPI_RELUGRAD && !TF32) {
          const int gn = tn * BN + c * 32;
          if (!(pre_vec && row_ok && gn + 32 <= args.N)) return;
          const OpT* mrow = reinterpret_cast<const OpT*>(args.mask) + static_cast<int64_t>(gm) * args.ldm + gn;
          uint32_t mw16[16];
          if (args.vec_mask == 2) {
            ld_v8(mrow, ev, mw16);
            ld_v8(mrow + 16, ev, mw16 + 8);
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 8) {
              const uint4 mv = ld_once(reinterpret_cast<const uint4*>(mrow + j), ev);
              mw16[j / 2] = mv.x; mw16[j / 2 + 1] = mv.y; mw16[j / 2 + 2] = mv.z; mw16[j / 2 + 3] = mv.w;
            }
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) p[j] = __uint_as_float(mw16[j]);
        } else if constexpr (EPI == EPI_SGD_APPLY) {
          const int gn = tn * BN + c * 32;
          if (!(pre_vec && row_ok && gn + 32 <= args.N)) return;
          const float* w = args.out_f32 + static_cast<int64_t>(gm) * args.ldo32 + gn;
          if (args.vec_out32 == 2) {
#pragma unroll
            for (int j = 0; j < 32; j += 8) ld_v8(w + j, ev, reinterpret_cast<uint32_t*>(p + j));
          } else {
#pragma unroll
            for (int j = 0; j < 32; j += 4) {
              const float4 w4 = ld_once(reinterpret_cast<const float4*>(w + j), ev);
              p[j] = w4.x; p[j + 1] = w4.y; p[j + 2] = w4.z; p[j + 3] = w4.w;
            }
          }
        } else {
          (void)c;
          (void)p;
        }
      };
      auto column_chunk = [&](int c, uint32_t (&r)[32], const float (&yv)[32], float bias_lane) {
        const int gn = tn * BN + c * 32;
        const bool active = row_ok && gn < args.N;
        const bool full_chunk = gn + 32 <= args.N;
        float bv[HAS_BIAS ? 32 : 1];  // this chunk's 32 bias values (all lanes)
        // profiling (debug 16): the output stores are skipped (issue and L1 cost of the
        // drain without them); debug 32: the bias broadcast is skipped
        const bool skip_st = (args.debug & 16) != 0;
        if constexpr (HAS_BIAS) {
          if (args.debug & 32) {
#pragma unroll
            for (int j = 0; j < 32; ++j) bv[j] = bias_lane;
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) bv[j] = __shfl_sync(0xffffffffu, bias_lane, j);
          }
        } else {
          (void)bias_lane;
          bv[0] = 0.f;
        }
        if constexpr (EPI == EPI_F32) {
          if (active) {
            float* o = args.out_f32 + static_cast<int64_t>(gm) * args.ldo32 + gn;
            if (full_chunk && args.vec_out32) {
#pragma unroll
              for (int j = 0; j < 32; j += 4)
                st_once(reinterpret_cast<uint4*>(o + j), make_uint4(r[j], r[j + 1], r[j + 2], r[j + 3]), ev);
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (gn + j < args.N) o[j] = u32_as_f32(r[j]);
            }
          }
        } else if constexpr (EPI == EPI_TRUNC16) {
          if (active) {
            uint16_t* o = reinterpret_cast<uint16_t*>(args.out) + static_cast<int64_t>(gm) * args.ldo + gn;
            const uint64_t ib = static_cast<uint64_t>(gm) * args.N + gn;  // bucket position of column gn
            auto code = [&](int j) { return round16(r[j], ib + j, args.r16); };
            if (full_chunk && args.vec_out) {
#pragma unroll
              for (int j = 0; j < 32; j += 8) {
                uint4 v;
                v.x = code(j) | (code(j + 1) << 16);
                v.y = code(j + 2) | (code(j + 3) << 16);
                v.z = code(j + 4) | (code(j + 5) << 16);
                v.w = code(j + 6) | (code(j + 7) << 16);
                *reinterpret_cast<uint4*>(o + j) = v;
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (gn + j < args.N) o[j] = static_cast<uint16_t>(code(j));
            }
          }
        } else if constexpr (EPI == EPI_TRUNC16_P2P) {
          // truncate, stage a 32-row x 64-column block per warp in smem, then push it to the
          // owners as 128-byte row segments (8 lanes x 16 B per row: full NVLink writes).
          // 8-element groups never straddle an owner (shard % 8 == 0, N % 8 == 0 on that path)
          uint16_t* stg = stg_base + q * 32 * Cfg::STG_PITCH;
          uint32_t* srow = reinterpret_cast<uint32_t*>(stg + lane * Cfg::STG_PITCH + (c & 1) * 32);
          const uint64_t ib = static_cast<uint64_t>(gm) * args.N + gn;  // bucket position of column gn
          // bulk-store path: the row this lane staged is read by its own bulk copy of the
          // previous chunk pair; wait until that read is done before overwriting it
          const bool bulk = args.p2p_bulk && (args.N % 8) == 0;
          if (bulk && !(c & 1)) ptx::bulk_wait_read_all();
#pragma unroll
          for (int j = 0; j < 16; ++j)
            srow[j] = round16(r[2 * j], ib + 2 * j, args.r16) | (round16(r[2 * j + 1], ib + 2 * j + 1, args.r16) << 16);
          if ((c & 1) && bulk) {
            // each lane ships its own staged row (<= 64 codes, 128 B) with one bulk copy per
            // owner it touches: the TMA engine carries the NVLink stores, the warp moves on
            const int gn0 = tn * BN + (c - 1) * 32;
            const int ncols = min(64, args.N - gn0);
            if (row_ok && ncols > 0) {
              ptx::fence_proxy_async_shared();
              const uint32_t src = ptx::smem_u32(stg + lane * Cfg::STG_PITCH);
              int64_t idx = static_cast<int64_t>(gm) * args.N + gn0;
              int left = ncols, done = 0;
              while (left > 0) {
                const int owner = static_cast<int>(idx / args.p2p_shard);
                const int64_t room = static_cast<int64_t>(owner + 1) * args.p2p_shard - idx;
                const int n = static_cast<int>(left < room ? static_cast<int64_t>(left) : room);  // multiple of 8 (shard, N, gn0)
                uint16_t* dst = args.p2p_recv[owner] + static_cast<int64_t>(args.p2p_rank) * args.p2p_shard +
                                (idx - static_cast<int64_t>(owner) * args.p2p_shard);
                ptx::bulk_store(dst, src + done * 2, n * 2);
                idx += n;
                done += n;
                left -= n;
              }
              ptx::bulk_commit();
            }
          } else if (c & 1) {
            __syncwarp();
            const int gm0 = tm * (BM * CG) + cta_rank * BM + q * 32;
            const int gn0 = tn * BN + (c - 1) * 32;
#pragma unroll
            for (int it = 0; it < 8; ++it) {
              const int p = it * 32 + lane, row = p >> 3, seg = p & 7;
              const int gmr = gm0 + row, gc = gn0 + seg * 8;
              if (gmr < args.M && gc < args.N) {
                const int64_t idx = static_cast<int64_t>(gmr) * args.N + gc;
                const uint16_t* src = stg + row * Cfg::STG_PITCH + seg * 8;
                if (gc + 8 <= args.N && (args.N % 8) == 0) {
                  const int owner = static_cast<int>(idx / args.p2p_shard);
                  uint16_t* dst = args.p2p_recv[owner] + static_cast<int64_t>(args.p2p_rank) * args.p2p_shard +
                                  (idx - static_cast<int64_t>(owner) * args.p2p_shard);
                  *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
                } else {
                  for (int e = 0; e < 8 && gc + e < args.N; ++e) {
                    const int64_t ie = idx + e;
                    const int owner = static_cast<int>(ie / args.p2p_shard);
                    args.p2p_recv[owner][static_cast<int64_t>(args.p2p_rank) * args.p2p_shard +
                                         (ie - static_cast<int64_t>(owner) * args.p2p_shard)] = src[e];
                  }
                }
              }
            }
            __syncwarp();
          }
        } else if constexpr (EPI == EPI_ASYNC_PUSH) {
          // f3: this replica's update of element (m, n) lands in its owner's shard
          // (reading A30: coded when another rank owns it; A31: one reduction, -fl(lr * g_hat))
          if (active) {
            const int64_t ib = static_cast<int64_t>(gm) * args.N + gn;  // bucket position of column gn
            const int64_t shard = args.p2p_shard;
            auto delta = [&](int j, int owner) {
              const float g = u32_as_f32(r[j]);
              const float gh = (args.async_coded && owner != args.p2p_rank)
                                   ? __uint_as_float(round16(r[j], static_cast<uint64_t>(ib + j), args.r16) << 16)
                                   : g;
              return -__fmul_rn(args.sgd_lr, gh);
            };
            if (full_chunk && (args.N % 8) == 0 && args.p2p_bulk) {
              // stage this row's 32 deltas and hand them to the TMA engine as bulk fp32
              // add-reductions into the owners' shards (split at owner boundaries, multiples
              // of 8 elements); each element is still one atomic fp32 add at its owner
              float* srow = reinterpret_cast<float*>(stg_base + q * 32 * Cfg::STG_PITCH + lane * Cfg::STG_PITCH);
              ptx::bulk_wait_read_all();  // this lane's previous row has been read
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const int64_t idx = ib + j;
                const int owner = static_cast<int>(idx / shard);
                *reinterpret_cast<float4*>(srow + j) =
                    make_float4(delta(j, owner), delta(j + 1, owner), delta(j + 2, owner), delta(j + 3, owner));
              }
              ptx::fence_proxy_async_shared();
              const uint32_t src = ptx::smem_u32(srow);
              int64_t idx = ib;
              int left = 32, done = 0;
              while (left > 0) {
                const int owner = static_cast<int>(idx / shard);
                const int64_t room = static_cast<int64_t>(owner + 1) * shard - idx;
                const int n = static_cast<int>(left < room ? static_cast<int64_t>(left) : room);
                ptx::bulk_reduce_add_f32(args.async_master[owner] + (idx - static_cast<int64_t>(owner) * shard),
                                         src + done * 4, n * 4);
                idx += n;
                done += n;
                left -= n;
              }
              ptx::bulk_commit();
            } else if (full_chunk && (args.N % 4) == 0) {
              // 4 consecutive elements share an owner (shard % 8 == 0, ib % 4 == 0): one v4 reduction
#pragma unroll
              for (int j = 0; j < 32; j += 4) {
                const int64_t idx = ib + j;
                const int owner = static_cast<int>(idx / shard);
                float* dst = args.async_master[owner] + (idx - static_cast<int64_t>(owner) * shard);
                red_add_sys_v4(dst, delta(j, owner), delta(j + 1, owner), delta(j + 2, owner), delta(j + 3, owner));
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                if (gn + j >= args.N) continue;
                const int64_t idx = ib + j;
                const int owner = static_cast<int>(idx / shard);
                red_add_sys(args.async_master[owner] + (idx - static_cast<int64_t>(owner) * shard), delta(j, owner));
              }
            }
          }
        } else if constexpr (EPI == EPI_SGD_APPLY) {
          // N = 1: ApplyGradientDescent fused into the dW epilogue (a4 + a9):
          // W <- fl(W - fl(lr * g)) on the fp32 master; the operand copy (bf16 RNE or
          // the tf32 pair) is refreshed from the new W
          if (active) {
            float* w = args.out_f32 + static_cast<int64_t>(gm) * args.ldo32 + gn;
            float v[32];
            if (full_chunk && pre_vec) {  // W prefetched by load_pre
#pragma unroll
              for (int j = 0; j < 32; ++j) v[j] = __fsub_rn(yv[j], __fmul_rn(args.sgd_lr, u32_as_f32(r[j])));
              if (args.vec_out32 == 2) {
#pragma unroll
                for (int j = 0; j < 32; j += 8) {
                  uint32_t w8[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) w8[e] = __float_as_uint(v[j + e]);
                  st_v8(w + j, w8, ev);
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  st_once(reinterpret_cast<float4*>(w + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]), ev);
              }
            } else {
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                v[j] = 0.f;
                if (gn + j < args.N) {
                  v[j] = __fsub_rn(w[j], __fmul_rn(args.sgd_lr, u32_as_f32(r[j])));
                  w[j] = v[j];
                }
              }
            }
            store_operand<TF32>(v, args.out, args.out2, args.ldo, gm, gn, args.N, args.vec_out, false, ev);
          }
        } else if constexpr (EPI == EPI_BIAS_RELU) {
          if (active) {
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const float z = __fadd_rn(u32_as_f32(r[j]), bv[j]);
              v[j] = (z < 0.f) ? 0.f : z;  // Relu; NaN propagates (non-finite guard)
            }
            if (args.out_f32 != nullptr && !skip_st) {
              float* o = args.out_f32 + static_cast<int64_t>(gm) * args.ldo32 + gn;
              if (full_chunk && args.vec_out32) {
#pragma unroll
                for (int j = 0; j < 32; j += 4)
                  st_once(reinterpret_cast<float4*>(o + j), make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]), ev);
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (gn + j < args.N) o[j] = v[j];
              }
            }
            if (args.out != nullptr && !skip_st)
              store_operand<TF32>(v, args.out, args.out2, args.ldo, gm, gn, args.N, args.vec_out,
                                  args.trunc_out != 0, ev);
          }
        } else if constexpr (EPI == EPI_RELUGRAD || EPI == EPI_BIAS_RELU_LOSS) {
          // dz values as stored, 0 outside the matrix; fused db column sums.
          float v[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = 0.f;
          if (active) {
            if constexpr (EPI == EPI_RELUGRAD) {
              const OpT* mrow = reinterpret_cast<const OpT*>(args.mask) + static_cast<int64_t>(gm) * args.ldm + gn;
              if (full_chunk && args.vec_mask) {
                if constexpr (!TF32) {
                  uint32_t mw16[16];  // the 32 bf16 mask values of this chunk (prefetched by load_pre)
#pragma unroll
                  for (int j = 0; j < 16; ++j) mw16[j] = __float_as_uint(yv[j]);
#pragma unroll
                  for (int j = 0; j < 32; j += 8) {
                    const uint32_t* mw = mw16 + j / 2;
#pragma unroll
                    for (int e = 0; e < 8; ++e) {
                      const uint32_t h = (mw[e >> 1] >> ((e & 1) * 16)) & 0xFFFFu;
                      // bf16 > 0  <=>  sign bit clear, not +0, not NaN
                      const bool pos = (h & 0x8000u) == 0 && h != 0 && h <= 0x7F80u;
                      v[j + e] = pos ? u32_as_f32(r[j + e]) : 0.f;
                    }
                  }
                } else {
#pragma unroll
                  for (int j = 0; j < 32; j += 4) {
                    const float4 m4 = ld_once(reinterpret_cast<const float4*>(mrow + j), ev);
                    v[j] = m4.x > 0.f ? u32_as_f32(r[j]) : 0.f;
                    v[j + 1] = m4.y > 0.f ? u32_as_f32(r[j + 1]) : 0.f;
                    v[j + 2] = m4.z > 0.f ? u32_as_f32(r[j + 2]) : 0.f;
                    v[j + 3] = m4.w > 0.f ? u32_as_f32(r[j + 3]) : 0.f;
                  }
                }
              } else {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                  if (gn + j < args.N) v[j] = (static_cast<float>(mrow[j]) > 0.f) ? u32_as_f32(r[j]) : 0.f;
              }
            } else {  // EPI_BIAS_RELU_LOSS: a = relu(acc + b); loss seed (reading A2, A10, A20)
              float* o32 = args.out_f32 ? args.out_f32 + static_cast<int64_t>(gm) * args.ldo32 + gn : nullptr;
              float av[32];
              float part = 0.f;  // this chunk's loss contribution (fp32), folded into loss_acc (fp64)
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                const bool in = gn + j < args.N;
                const float z = __fadd_rn(u32_as_f32(r[j]), bv[j]);
                const float a = (z < 0.f) ? 0.f : z;
                float g;
                if (args.loss_kind == 0) {  // MSE: d = a - y, g = d / (rows*cols) (IEEE, reading A20)
                  const float d = __fsub_rn(a, yv[j]);
                  part = in ? __fmaf_rn(d, d, part) : part;
                  g = args.denom_pow2 ? __fmul_rn(d, args.inv_denom) : __fdiv_rn(d, args.loss_denom);
                } else {                    // SUM: g = 1 / rows
                  part = in ? __fadd_rn(part, a) : part;
                  g = args.seed_const;
                }
                av[j] = a;
                v[j] = (in && a > 0.f) ? g : 0.f;
              }
              loss_acc += static_cast<double>(part);
              if (o32) {
                if (full_chunk && args.vec_out32) {
#pragma unroll
                  for (int j = 0; j < 32; j += 4)
                    st_once(reinterpret_cast<float4*>(o32 + j), make_float4(av[j], av[j + 1], av[j + 2], av[j + 3]), ev);
                } else {
#pragma unroll
                  for (int j = 0; j < 32; ++j)
                    if (gn + j < args.N) o32[j] = av[j];
                }
              }
            }
            if (!skip_st) store_operand<TF32>(v, args.out, args.out2, args.ldo, gm, gn, args.N, args.vec_out, false, ev);
          }
          if (args.colsum_ws != nullptr) {
            // transpose-reduce: after 5 butterfly steps lane l holds the sum over this
            // warp's 32 rows of column gn + l (fixed order -> deterministic)
#pragma unroll
            for (int off = 16; off >= 1; off >>= 1) {
              const bool upper = (lane & off) != 0;
#pragma unroll
              for (int i = 0; i < off; ++i) {
                const float send = upper ? v[i] : v[i + off];
                const float keep = upper ? v[i + off] : v[i];
                v[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, off));
              }
            }
            const int rowblk = (tm * (BM * CG) + cta_rank * BM + q * 32) >> 5;
            if (gn + lane < args.N && rowblk * 32 < args.M)
              args.colsum_ws[static_cast<int64_t>(rowblk) * args.N + gn + lane] = v[0];
          }
        }
        __syncwarp();
      };
      if constexpr (TF32) {
        // (the K-chunk sums already hold 128 registers: one operand buffer, loaded per chunk)
#pragma unroll
        for (int c = 0; c < BN / 32; ++c) {
          float pre[32];
          load_pre(c, pre);
          uint32_t r[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) r[j] = __float_as_uint(kacc[c * 32 + j]);
          column_chunk(c, r, pre, bl[HAS_BIAS ? c : 0]);
        }
      } else {
        // Software-pipelined and rolled (an unrolled epilogue overflows the instruction
        // cache): chunk c + 1's TMEM load and streamed operand are in flight while chunk c is
        // processed, so the drain runs at issue rate, not at TMEM + DRAM latency per chunk —
        // with the 512-wide tile the MMA waits on this drain at every tile boundary.
        auto tmem_issue = [&](int c, uint32_t (&r)[32]) {
          if (num_kb > 0) {
            half_switch(c);
            ptx::tmem_ld_32x32b_x32(tmem_row + acc * BN + c * 32, r);
          }
        };
        auto tmem_land = [&](uint32_t (&r)[32]) {
          if (num_kb > 0) {
            ptx::tmem_ld_wait_regs(r);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) r[j] = 0u;  // K == 0: the empty sum
          }
        };
        // two register sets, alternating roles chunk by chunk (the loop body is one even and
        // one odd chunk, so no copies between them)
        float pa[32], pb[32];
        uint32_t ra[32], rb[32];
        auto step = [&](int c, uint32_t (&rcur)[32], float (&pcur)[32], uint32_t (&rnext)[32], float (&pnext)[32],
                        float bcur) {
          const bool more = c + 1 < BN / 32;
          if (more) {
            load_pre(c + 1, pnext);
            tmem_issue(c + 1, rnext);
          }
          column_chunk(c, rcur, pcur, bcur);
          if (more) tmem_land(rnext);
        };
        load_pre(0, pa);
        tmem_issue(0, ra);
        tmem_land(ra);
        static_assert((BN / 32) % 2 == 0, "chunk pairs");
#pragma unroll 1
        for (int c = 0; c < BN / 32; c += 2) {
          float b0 = 0.f, b1 = 0.f;
          if constexpr (HAS_BIAS) {
            b0 = bl[0];
            b1 = bl[1];
#pragma unroll
            for (int k = 0; k + 2 < BN / 32; ++k) bl[k] = bl[k + 2];
          }
          step(c, ra, pa, rb, pb, b0);
          step(c + 1, rb, pb, ra, pa, b1);
        }
        if (num_kb > 0) release_tmem();
      }
      if constexpr (EPI == EPI_BIAS_RELU_LOSS) {
        // one partial per (tile, CTA of the pair, warp): the slot depends on the tile, not on
        // which CTA the dynamic scheduler gave it to, so k_loss_final's order is fixed
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) loss_acc += __shfl_xor_sync(0xffffffffu, loss_acc, o);
        if (lane == 0 && args.loss_partials)
          args.loss_partials[(static_cast<int64_t>(t) * CG + cta_rank) * 4 + q] = loss_acc;
        loss_acc = 0.0;
      }
    }
    // the owners read these NVLink stores after a later kernel's system-scope flag
    if constexpr (EPI == EPI_TRUNC16_P2P || EPI == EPI_ASYNC_PUSH) {
      if (args.p2p_bulk) ptx::bulk_wait_all();  // this thread's bulk stores / reductions are done
      if constexpr (EPI == EPI_TRUNC16_P2P) __threadfence_system();
    }
  }

  ptx::tc_fence_before();
  if constexpr (CG == 2) ptx::cluster_sync(); else __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<CG>(tmem_base, Cfg::TMEM_COLS);
  }
}

}  // namespace dflow
