// Host launcher for the tcgen05 GEMM family (NK1-NK6): TMA descriptor
// encoding, tile-config choice, persistent grid sizing, cluster launch.
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdio>
#include <map>
#include <cstdlib>
#include <algorithm>
#include <cstring>
#include <mutex>
#include <type_traits>
#include <vector>

#include "gemm.cuh"
#include "gemm.h"
#include "topology.h"

namespace dflow {

static thread_local char g_err[512];
const char* gemm_last_error() { return g_err; }

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D tensor map (bf16 or fp32 elements) over a row-major matrix with `inner`
// contiguous elements per row (logical extent), `outer` rows, pitch `ld` elements,
// 128-byte swizzle, OOB zero fill.
static bool make_tmap(CUtensorMap* m, const void* base, bool f32, int64_t inner, int64_t outer, int64_t ld,
                      uint32_t box_inner, uint32_t box_outer, bool atom32 = false) {
  auto fn = encode_fn();
  if (!fn) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled unavailable");
    return false;
  }
  const int e = f32 ? 4 : 2;
  if (!base || (reinterpret_cast<uintptr_t>(base) & 15) || ((ld * e) & 15)) {
    snprintf(g_err, sizeof g_err, "TMA needs a 16-byte aligned base and row pitch (ld=%lld)", (long long)ld);
    return false;
  }
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld * e)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  // L2 promotion of the operand loads (DFLOW_GEMM_L2PROMO = 0 / 64 / 128 / 256 bytes; A/B knob)
  static const CUtensorMapL2promotion promo = [] {
    const char* e = getenv("DFLOW_GEMM_L2PROMO");
    const int v = e ? atoi(e) : 256;
    return v == 0 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                  : v == 64 ? CU_TENSOR_MAP_L2_PROMOTION_L2_64B
                            : v == 128 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B : CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }();
  CUresult r = fn(m, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  atom32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, promo,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(g_err, sizeof g_err, "cuTensorMapEncodeTiled failed (%d): inner=%lld outer=%lld ld=%lld box=%u,%u",
             (int)r, (long long)inner, (long long)outer, (long long)ld, box_inner, box_outer);
    return false;
  }
  return true;
}

template <int BN, int CG, bool TF32, bool A_MN, bool B_MN, int EPI>
static void* kernel_ptr(int* smem) {
  auto k = &gemm_kernel<BN, CG, TF32, A_MN, B_MN, EPI>;
  constexpr int bytes = GemmCfg<BN, CG, TF32, EPI == EPI_TRUNC16_P2P || EPI == EPI_ASYNC_PUSH>::SMEM_BYTES;
  // the opt-in to >48 KB of dynamic shared memory is per device: set it once per device
  // (threads racing here both set it, which is harmless)
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t bit = 1ull << (dev & 63);
  if (!(attr_set.load(std::memory_order_acquire) & bit)) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    attr_set.fetch_or(bit, std::memory_order_acq_rel);
  }
  *smem = bytes;
  return reinterpret_cast<void*>(k);
}

// The wide pair tile (BN = 512, bf16): the forward, dgrad and wgrad epilogues of the N = 1
// step and the NCCL-schedule exchange (not the fused-channel or asynchronous epilogues).
static void* select_kernel_512(bool a_mn, bool b_mn, int epi, int* smem) {
  if (!a_mn && b_mn) {
    if (epi == EPI_BIAS_RELU) return kernel_ptr<512, 2, false, false, true, EPI_BIAS_RELU>(smem);
    if (epi == EPI_BIAS_RELU_LOSS) return kernel_ptr<512, 2, false, false, true, EPI_BIAS_RELU_LOSS>(smem);
    if (epi == EPI_F32) return kernel_ptr<512, 2, false, false, true, EPI_F32>(smem);
  } else if (!a_mn && !b_mn) {
    if (epi == EPI_RELUGRAD) return kernel_ptr<512, 2, false, false, false, EPI_RELUGRAD>(smem);
    if (epi == EPI_F32) return kernel_ptr<512, 2, false, false, false, EPI_F32>(smem);
  } else if (a_mn && b_mn) {
    if (epi == EPI_F32) return kernel_ptr<512, 2, false, true, true, EPI_F32>(smem);
    if (epi == EPI_TRUNC16) return kernel_ptr<512, 2, false, true, true, EPI_TRUNC16>(smem);
    if (epi == EPI_SGD_APPLY) return kernel_ptr<512, 2, false, true, true, EPI_SGD_APPLY>(smem);
  }
  return nullptr;
}

// The (operand majors, epilogue) combinations the MLP step uses, per tile config.
template <int BN, int CG, bool TF32>
static void* select_kernel(bool a_mn, bool b_mn, int epi, int* smem) {
  if (!a_mn && b_mn) {  // forward: A K-major, W MN-major
    if (epi == EPI_BIAS_RELU) return kernel_ptr<BN, CG, TF32, false, true, EPI_BIAS_RELU>(smem);
    if (epi == EPI_BIAS_RELU_LOSS) return kernel_ptr<BN, CG, TF32, false, true, EPI_BIAS_RELU_LOSS>(smem);
    if (epi == EPI_F32) return kernel_ptr<BN, CG, TF32, false, true, EPI_F32>(smem);
  } else if (!a_mn && !b_mn) {  // dgrad: dZ K-major, W K-major
    if (epi == EPI_RELUGRAD) return kernel_ptr<BN, CG, TF32, false, false, EPI_RELUGRAD>(smem);
    if (epi == EPI_F32) return kernel_ptr<BN, CG, TF32, false, false, EPI_F32>(smem);
    if constexpr (!TF32)  // f4: dA leaving for the previous rank as channel codes
      if (epi == EPI_TRUNC16) return kernel_ptr<BN, CG, TF32, false, false, EPI_TRUNC16>(smem);
  } else if (a_mn && b_mn) {  // wgrad: activations and dZ both MN-major
    if (epi == EPI_F32) return kernel_ptr<BN, CG, TF32, true, true, EPI_F32>(smem);
    if (epi == EPI_TRUNC16) return kernel_ptr<BN, CG, TF32, true, true, EPI_TRUNC16>(smem);
    if (epi == EPI_SGD_APPLY) return kernel_ptr<BN, CG, TF32, true, true, EPI_SGD_APPLY>(smem);
    if (epi == EPI_TRUNC16_P2P) return kernel_ptr<BN, CG, TF32, true, true, EPI_TRUNC16_P2P>(smem);
    if constexpr (!TF32)
      if (epi == EPI_ASYNC_PUSH) return kernel_ptr<BN, CG, TF32, true, true, EPI_ASYNC_PUSH>(smem);
  }
  return nullptr;
}

// The measured SM -> die map of `dev` on the device (int per SM id), or NULL when the
// measurement gave no clean two-die split; *n0 = SMs on die 0, *n = SMs.
static const int* device_die_map(int dev, int* n0, int* n) {
  static std::mutex mu;
  static std::map<int, std::pair<int*, std::pair<int, int>>> maps;
  std::lock_guard<std::mutex> lock(mu);
  auto it = maps.find(dev);
  if (it == maps.end()) {
    std::vector<int> m;
    int* d = nullptr;
    int c0 = 0;
    if (measure_die_map(dev, &m, nullptr) && cudaMalloc(&d, m.size() * sizeof(int)) == cudaSuccess) {
      if (cudaMemcpy(d, m.data(), m.size() * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
        cudaFree(d);
        d = nullptr;
      }
      for (int x : m) c0 += x == 0;
    }
    cudaGetLastError();
    it = maps.emplace(dev, std::make_pair(d, std::make_pair(c0, static_cast<int>(m.size())))).first;
  }
  *n0 = it->second.second.first;
  *n = it->second.second.second;
  return it->second.first;
}

// Tile-scheduler counters [die 0, die 1, done, pad] per (device, stream); zeroed once, and every GEMM
// launch leaves them zero again, so launches serialised on one stream can share them (and
// GEMMs on different streams never do).  Sessions pass their own counters in GemmDesc.sched.
int* gemm_stream_sched(cudaStream_t stream) {
  static std::map<std::pair<int, cudaStream_t>, int*> ptrs;
  static std::mutex mu;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lock(mu);
  int*& slot = ptrs[{dev, stream}];
  if (!slot) {
    void* p = nullptr;
    if (cudaMalloc(&p, 4 * sizeof(int)) != cudaSuccess) return nullptr;
    if (cudaMemset(p, 0, 4 * sizeof(int)) != cudaSuccess) return nullptr;
    slot = static_cast<int*>(p);
  }
  return slot;
}

static bool aligned16(const void* p, int64_t ld, int elem) {
  return p != nullptr && (reinterpret_cast<uintptr_t>(p) & 15) == 0 && ((ld * elem) & 15) == 0;
}

// 2: 32-byte aligned (256-bit epilogue accesses), 1: 16-byte aligned, 0: scalar.
// DFLOW_GEMM_V8=0 caps it at 1 (A/B of the 256-bit accesses).
static int vec_width(const void* p, int64_t ld, int elem) {
  static const int allow_v8 = [] {
    const char* e = getenv("DFLOW_GEMM_V8");
    return e ? atoi(e) : 1;
  }();
  if (!aligned16(p, ld, elem)) return 0;
  const bool a32 = (reinterpret_cast<uintptr_t>(p) & 31) == 0 && ((ld * elem) & 31) == 0;
  return (a32 && allow_v8) ? 2 : 1;
}

cudaError_t gemm_prepare(const GemmDesc& d, int num_sms, GemmPlan* plan) {
  g_err[0] = 0;
  if (d.M <= 0 || d.N <= 0 || d.K < 0 || d.M > (1 << 30) || d.N > (1 << 30) || d.K > (1 << 30)) {
    snprintf(g_err, sizeof g_err, "bad GEMM shape %lld x %lld x %lld", (long long)d.M, (long long)d.N, (long long)d.K);
    return cudaErrorInvalidValue;
  }
  int tile = d.tile;
  if (tile == 0) {
    const int64_t pair_tiles = ((d.M + 255) / 256) * ((d.N + 255) / 256);
    tile = (pair_tiles >= num_sms / 2) ? 2 : 1;
    // the wide pair tile, 256 x 512 per CTA pair, where it fills the machine and the epilogue
    // has a 512-wide variant.  DFLOW_GEMM_TILE512 (A/B knob): 0 off (default), 1 every GEMM
    // kind, 2 the weight gradient only.  It reads 25 % fewer operand bytes per FLOP and runs
    // at a higher power-capped clock, but its single TMEM accumulator exposes the epilogue
    // drain at every tile boundary: the N = 1 step is 5 % slower with it everywhere and
    // unchanged with it on the weight gradient only
    const char* wide_env = getenv("DFLOW_GEMM_TILE512");  // read per plan, like the raster knobs
    const int wide = wide_env ? atoi(wide_env) : 0;
    int dummy = 0;
    const bool wgrad_kind = d.a_mn && d.b_mn;
    if ((wide == 1 || (wide == 2 && wgrad_kind)) && tile == 2 && !d.tf32 &&
        ((d.M + 255) / 256) * ((d.N + 511) / 512) >= num_sms / 2 && select_kernel_512(d.a_mn, d.b_mn, d.epilogue, &dummy))
      tile = 3;
  }
  const bool tf = d.tf32;
  if (tile == 3 && tf) {
    snprintf(g_err, sizeof g_err, "the 512-wide tile is bf16 only");
    return cudaErrorInvalidValue;
  }
  // 3xTF32 pairs use N = 128 so the epilogue can hold a row's fp32 K-chunk sums in registers
  const int BN = tile == 3 ? 512 : (tile == 2 && !tf) ? 256 : 128;
  const int CG = (tile >= 2) ? 2 : 1;
  const int BN_CTA = BN / CG;
  const int BK = tf ? 32 : 64;
  const int CHUNK = BK;  // MN elements per 128-byte row (= BK for both element sizes)
  plan->d = d;
  plan->tile = tile;
  plan->cluster = CG;
  plan->tiles_m = static_cast<int>((d.M + 128 * CG - 1) / (128 * CG));
  plan->tiles_n = static_cast<int>((d.N + BN - 1) / BN);
  void* k = nullptr;
  if (tile == 3)
    k = select_kernel_512(d.a_mn, d.b_mn, d.epilogue, &plan->smem);
  else if (tile == 2)
    k = tf ? select_kernel<128, 2, true>(d.a_mn, d.b_mn, d.epilogue, &plan->smem)
           : select_kernel<256, 2, false>(d.a_mn, d.b_mn, d.epilogue, &plan->smem);
  else
    k = tf ? select_kernel<128, 1, true>(d.a_mn, d.b_mn, d.epilogue, &plan->smem)
           : select_kernel<128, 1, false>(d.a_mn, d.b_mn, d.epilogue, &plan->smem);
  if (!k) {
    snprintf(g_err, sizeof g_err, "unsupported GEMM layout/epilogue (a_mn=%d b_mn=%d epi=%d)", d.a_mn, d.b_mn,
             d.epilogue);
    return cudaErrorInvalidValue;
  }
  plan->kernel = k;
  const int64_t K = d.K > 0 ? d.K : 1;
  // MN-major fp32 (tf32) operands: 32-byte-atom 128B swizzle (the UMMA SWIZZLE_128B_BASE32B layout)
  auto map_a = [&](CUtensorMap* m, const void* p) {
    return d.a_mn ? make_tmap(m, p, tf, d.M, K, d.lda, CHUNK, BK, tf) : make_tmap(m, p, tf, K, d.M, d.lda, BK, 128);
  };
  // K-major B boxes cover one piece of a CTA's B columns (128 rows; the 512-wide tile loads two)
  const uint32_t b_box = tile == 3 ? BN_CTA / 2 : BN_CTA;
  auto map_b = [&](CUtensorMap* m, const void* p) {
    return d.b_mn ? make_tmap(m, p, tf, d.N, K, d.ldb, CHUNK, BK, tf)
                  : make_tmap(m, p, tf, K, d.N, d.ldb, BK, b_box);
  };
  bool ok = map_a(&plan->tmA, d.A) && map_b(&plan->tmB, d.B);
  if (ok && tf) {
    ok = map_a(&plan->tmA2, d.A2) && map_b(&plan->tmB2, d.B2);
  } else if (ok) {
    plan->tmA2 = plan->tmA;
    plan->tmB2 = plan->tmB;
  }
  if (!ok) return cudaErrorInvalidValue;
  GemmArgs& a = plan->args;
  memset(&a, 0, sizeof a);
  a.M = static_cast<int>(d.M);
  a.N = static_cast<int>(d.N);
  a.K = static_cast<int>(d.K);
  a.tiles_m = plan->tiles_m;
  a.tiles_n = plan->tiles_n;
  a.out = d.out;
  a.out2 = d.out2;
  a.ldo = d.ldo;
  a.out_f32 = d.out_f32;
  a.ldo32 = d.ldo32;
  a.bias = d.bias;
  a.mask = d.mask;
  a.ldm = d.ldm;
  const int op_elem = tf ? 4 : 2;
  const int out_elem = (d.epilogue == EPI_TRUNC16) ? 2 : op_elem;
  // (the 256-bit paths exist for the bf16 operand stores, the bf16 mask, the fp32 W of the
  // SGD epilogue and the targets; elsewhere any nonzero width takes the 16-byte path)
  a.vec_out = aligned16(d.out, d.ldo, out_elem) && (!tf || d.epilogue == EPI_TRUNC16 || aligned16(d.out2, d.ldo, 4))
                  ? ((tf || d.epilogue == EPI_TRUNC16) ? 1 : vec_width(d.out, d.ldo, out_elem))
                  : 0;
  a.vec_out32 = vec_width(d.out_f32, d.ldo32, 4);
  a.vec_mask = vec_width(d.mask, d.ldm, op_elem);
  a.y = d.y;
  a.ldy = d.ldy;
  a.loss_kind = d.loss_kind;
  a.loss_denom = static_cast<float>(d.M * d.N);
  const int64_t mn = d.M * d.N;
  a.denom_pow2 = (mn > 0 && (mn & (mn - 1)) == 0) ? 1 : 0;
  a.inv_denom = 1.0f / a.loss_denom;
  a.vec_y = vec_width(d.y, d.ldy, 4);
  a.vec_bias = aligned16(d.bias, 0, 4) ? 1 : 0;
  a.group_m = d.group > 0 ? d.group : 8;
  if (const char* e = getenv("DFLOW_GEMM_GROUP")) a.group_m = atoi(e) > 0 ? atoi(e) : a.group_m;
  // L2 prefetch distance in k-blocks (DFLOW_GEMM_PREFETCH). Off by default: measured on the
  // C3 shapes it costs 20-25% (the extra L2 lookups contend with the loads; profiles/r1_gemm_issue.md)
  a.prefetch = 0;
  if (const char* e = getenv("DFLOW_GEMM_PREFETCH")) a.prefetch = atoi(e) >= 0 ? atoi(e) : a.prefetch;
  if (const char* e = getenv("DFLOW_GEMM_DEBUG")) a.debug = atoi(e);
  a.evict = 1;
  if (const char* e = getenv("DFLOW_GEMM_EVICT")) a.evict = atoi(e) != 0;  // A/B knob
  a.sgd_lr = d.sgd_lr;
  a.sched = d.sched ? d.sched : gemm_stream_sched(nullptr);
  if (!a.sched) {
    snprintf(g_err, sizeof g_err, "could not allocate the tile-scheduler counters");
    return cudaErrorMemoryAllocation;
  }
  a.seed_const = 1.0f / static_cast<float>(d.M);
  a.loss_partials = d.loss_partials;
  a.colsum_ws = d.colsum_ws;
  a.trunc_out = d.trunc_out;
  if (d.epilogue == EPI_TRUNC16_P2P) {
    if (!d.p2p_recv || d.p2p_world < 1 || d.p2p_world > kMaxRanks || d.p2p_shard <= 0 || d.p2p_shard % 8 ||
        d.p2p_rank < 0 || d.p2p_rank >= d.p2p_world) {
      snprintf(g_err, sizeof g_err, "bad peer-to-peer exchange arguments");
      return cudaErrorInvalidValue;
    }
    for (int r = 0; r < d.p2p_world; ++r) a.p2p_recv[r] = d.p2p_recv[r];
    a.p2p_shard = d.p2p_shard;
    a.p2p_rank = d.p2p_rank;
    a.p2p_world = d.p2p_world;
    a.p2p_bulk = d.p2p_bulk;
    if (const char* e = getenv("DFLOW_P2P_BULK")) a.p2p_bulk = atoi(e) != 0;  // A/B knob
  }
  if (d.epilogue == EPI_ASYNC_PUSH) {
    if (!d.async_master || d.p2p_world < 1 || d.p2p_world > kMaxRanks || d.p2p_shard <= 0 || d.p2p_shard % 8 ||
        d.p2p_rank < 0 || d.p2p_rank >= d.p2p_world || tf) {
      snprintf(g_err, sizeof g_err, "bad asynchronous push arguments (bf16 path only)");
      return cudaErrorInvalidValue;
    }
    for (int r = 0; r < d.p2p_world; ++r) a.async_master[r] = d.async_master[r];
    a.async_coded = d.async_coded;
    a.p2p_bulk = d.p2p_bulk;
    if (const char* e = getenv("DFLOW_P2P_BULK")) a.p2p_bulk = atoi(e) != 0;  // A/B knob
    a.p2p_shard = d.p2p_shard;
    a.p2p_rank = d.p2p_rank;
    a.p2p_world = d.p2p_world;
  }
  const bool need_lo = tf && d.epilogue != EPI_F32 && d.epilogue != EPI_TRUNC16;
  if ((d.epilogue == EPI_F32 && !d.out_f32) || (d.epilogue == EPI_TRUNC16 && !d.out) ||
      (d.epilogue == EPI_SGD_APPLY && (!d.out_f32 || !d.out)) ||
      (d.epilogue == EPI_RELUGRAD && (!d.out || !d.mask)) ||
      (d.epilogue == EPI_BIAS_RELU && (!d.bias || (!d.out && !d.out_f32))) ||
      (d.epilogue == EPI_BIAS_RELU_LOSS && (!d.bias || !d.out || (d.loss_kind == 0 && !d.y))) ||
      (need_lo && d.out && !d.out2)) {
    snprintf(g_err, sizeof g_err, "missing GEMM epilogue operand (epi=%d)", d.epilogue);
    return cudaErrorInvalidValue;
  }
  int clusters = num_sms / CG;
  if (d.max_ctas > 0 && d.max_ctas < num_sms) clusters = d.max_ctas / CG;
  const int tiles = plan->tiles_m * plan->tiles_n;
  if (clusters > tiles) clusters = tiles;
  if (clusters < 1) clusters = 1;
  plan->grid = clusters * CG;
  // die-aware schedule: split the raster in proportion to the dies' SMs (topology.cu);
  // DFLOW_GEMM_DIE_SPLIT=0 turns it off (A/B)
  a.die_map = nullptr;
  a.die_split = tiles;
  // experimental, off by default: +3 % sustained GEMM rate on one box, -6 % on another (the
  // measured die map's quality varies per GPU) — DFLOW_GEMM_DIE_SPLIT=1 (two
  // raster ranges) / 2 (N halves of every M-group)
  static const int die_mode = [] {
    const char* e = getenv("DFLOW_GEMM_DIE_SPLIT");
    return e ? atoi(e) : 0;
  }();
  int dev = 0;
  if (die_mode && clusters == num_sms / CG && cudaGetDevice(&dev) == cudaSuccess) {
    int n0 = 0, n = 0;
    const int* dm = device_die_map(dev, &n0, &n);
    if (dm && n == num_sms && (die_mode == 1 || plan->tiles_n >= 2)) {
      a.die_map = dm;
      a.die_mode = die_mode;
      a.die_split = die_mode == 2 ? std::max(1, std::min(plan->tiles_n - 1, (plan->tiles_n * n0 + n / 2) / n))
                                  : static_cast<int>((static_cast<int64_t>(tiles) * n0 + n / 2) / n);
    }
  }
  return cudaSuccess;
}

cudaError_t gemm_launch(const GemmPlan& plan, cudaStream_t stream) {
  cudaLaunchConfig_t cfg;
  memset(&cfg, 0, sizeof cfg);
  cfg.gridDim = dim3(plan.grid, 1, 1);
  cfg.blockDim = dim3(256, 1, 1);
  cfg.dynamicSmemBytes = plan.smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = plan.cluster;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[5] = {const_cast<CUtensorMap*>(&plan.tmA), const_cast<CUtensorMap*>(&plan.tmB),
                   const_cast<CUtensorMap*>(&plan.tmA2), const_cast<CUtensorMap*>(&plan.tmB2),
                   const_cast<GemmArgs*>(&plan.args)};
  cudaError_t e = cudaLaunchKernelExC(&cfg, plan.kernel, args);
  if (e != cudaSuccess) snprintf(g_err, sizeof g_err, "GEMM launch failed: %s", cudaGetErrorString(e));
  return e;
}

}  // namespace dflow
