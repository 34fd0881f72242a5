// extern "C" boundary of libdflow (include/dflow.h).  Argument checking and
// marshalling only; every computation runs in the CUDA kernels behind
// session.cu / kernels/.  No exception crosses this file.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/dflow.h"
#include "common.h"
#include "graph.h"
#include "kernels/elementwise.h"
#include "kernels/gemm.h"
#include "kernels/topology.h"
#include "session.h"
#include "sim.h"

struct dflow_graph {
  dflow::Graph g;
};

namespace dflow {
static thread_local std::string g_last_error;
void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_last_error = buf;
}
void clear_error() { g_last_error.clear(); }
}  // namespace dflow

using dflow::fail;

#define GUARD_BEGIN try {
#define GUARD_END                                                               \
  }                                                                             \
  catch (const std::bad_alloc&) {                                               \
    return fail(DFLOW_OOM, "host allocation failed");                           \
  }                                                                             \
  catch (...) {                                                                 \
    return fail(DFLOW_INVALID_ARGUMENT, "internal error (unexpected exception)"); \
  }

static dflow_status json_out(const std::string& js, char* buf, size_t cap, size_t* needed) {
  if (needed) *needed = js.size() + 1;
  if (!buf || cap < js.size() + 1) {
    if (buf && cap) buf[0] = 0;
    return fail(DFLOW_BUFFER_TOO_SMALL, "JSON needs %zu bytes", js.size() + 1);
  }
  memcpy(buf, js.c_str(), js.size() + 1);
  return DFLOW_OK;
}

extern "C" {

const char* dflow_last_error(void) { return dflow::g_last_error.c_str(); }

const char* dflow_status_name(dflow_status s) {
  switch (s) {
    case DFLOW_OK: return "DFLOW_OK";
    case DFLOW_INVALID_ARGUMENT: return "DFLOW_INVALID_ARGUMENT";
    case DFLOW_DUPLICATE_NAME: return "DFLOW_DUPLICATE_NAME";
    case DFLOW_UNKNOWN_OP: return "DFLOW_UNKNOWN_OP";
    case DFLOW_DANGLING_INPUT: return "DFLOW_DANGLING_INPUT";
    case DFLOW_SHAPE_MISMATCH: return "DFLOW_SHAPE_MISMATCH";
    case DFLOW_NON_DIFFERENTIABLE: return "DFLOW_NON_DIFFERENTIABLE";
    case DFLOW_NON_SCALAR_TARGET: return "DFLOW_NON_SCALAR_TARGET";
    case DFLOW_UNIMPLEMENTED: return "DFLOW_UNIMPLEMENTED";
    case DFLOW_NOT_INITIALIZED: return "DFLOW_NOT_INITIALIZED";
    case DFLOW_CUDA: return "DFLOW_CUDA";
    case DFLOW_NCCL: return "DFLOW_NCCL";
    case DFLOW_OOM: return "DFLOW_OOM";
    case DFLOW_SESSION_POISONED: return "DFLOW_SESSION_POISONED";
    case DFLOW_BUFFER_TOO_SMALL: return "DFLOW_BUFFER_TOO_SMALL";
  }
  return "DFLOW_UNKNOWN_STATUS";
}

const char* dflow_version(void) { return "dflow 0.1 (sm_100a tcgen05)"; }

// ------------------------------------------------------------------ graph
dflow_status dflow_graph_create(dflow_graph** out) {
  GUARD_BEGIN
  if (!out) return fail(DFLOW_INVALID_ARGUMENT, "out is NULL");
  *out = new dflow_graph();
  return DFLOW_OK;
  GUARD_END
}

void dflow_graph_destroy(dflow_graph* g) { delete g; }

dflow_status dflow_graph_num_nodes(const dflow_graph* g, int32_t* out) {
  if (!g || !out) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  *out = static_cast<int32_t>(g->g.nodes.size());
  return DFLOW_OK;
}

dflow_status dflow_node_by_name(const dflow_graph* g, const char* name, dflow_node* out) {
  if (!g || !name || !out) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  auto it = g->g.by_name.find(name);
  if (it == g->g.by_name.end()) return fail(DFLOW_DANGLING_INPUT, "no node named '%s'", name);
  *out = it->second;
  return DFLOW_OK;
}

dflow_status dflow_placeholder(dflow_graph* g, const char* name, dflow_dtype dtype, int rank, const int64_t* dims,
                               dflow_node* out) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return g->g.placeholder(name, dtype, rank, dims, out);
  GUARD_END
}

dflow_status dflow_variable(dflow_graph* g, const char* name, dflow_dtype dtype, int rank, const int64_t* dims,
                            dflow_node* out) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return g->g.variable(name, dtype, rank, dims, out);
  GUARD_END
}

dflow_status dflow_matmul(dflow_graph* g, const char* name, dflow_node a, dflow_node b, int transpose_a,
                          int transpose_b, dflow_node* out) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return g->g.matmul(name, a, b, transpose_a, transpose_b, out);
  GUARD_END
}

dflow_status dflow_add(dflow_graph* g, const char* name, dflow_node a, dflow_node b, dflow_node* out) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return g->g.add(name, a, b, out);
  GUARD_END
}

dflow_status dflow_relu(dflow_graph* g, const char* name, dflow_node x, dflow_node* out) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return g->g.relu(name, x, out);
  GUARD_END
}

dflow_status dflow_loss(dflow_graph* g, const char* name, int kind, dflow_node pred, dflow_node target,
                        dflow_node* out) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return g->g.loss(name, kind, pred, target, out);
  GUARD_END
}

dflow_status dflow_gradients(dflow_graph* g, dflow_node cost, int n, const dflow_node* xs, dflow_node* out_grads) {
  GUARD_BEGIN
  if (!g || n < 0 || (n > 0 && (!xs || !out_grads))) return fail(DFLOW_INVALID_ARGUMENT, "bad arguments");
  std::vector<int> v(xs, xs + n), res;
  dflow_status st = g->g.gradients(cost, v, &res);
  if (st != DFLOW_OK) return st;
  for (int i = 0; i < n; ++i) out_grads[i] = res[i];
  return DFLOW_OK;
  GUARD_END
}

dflow_status dflow_apply_gradient_descent(dflow_graph* g, const char* name, dflow_node var, float lr, dflow_node grad,
                                          dflow_node* out) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return g->g.apply_gradient_descent(name, var, lr, grad, out);
  GUARD_END
}

dflow_status dflow_graph_to_json(const dflow_graph* g, char* buf, size_t cap, size_t* needed) {
  GUARD_BEGIN
  if (!g) return fail(DFLOW_INVALID_ARGUMENT, "graph is NULL");
  return json_out(g->g.to_json(), buf, cap, needed);
  GUARD_END
}

dflow_status dflow_graph_partition(const dflow_graph* g, const int32_t* device_of_node, int32_t n_nodes, int32_t device,
                                   int32_t compress, dflow_graph** out) {
  GUARD_BEGIN
  if (!g || !device_of_node || !out) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  if (n_nodes != static_cast<int32_t>(g->g.nodes.size())) return fail(DFLOW_INVALID_ARGUMENT, "n_nodes != node count");
  std::vector<int> place(device_of_node, device_of_node + n_nodes);
  std::vector<dflow::Graph> parts;
  dflow_status st = dflow::partition(g->g, place, compress != 0, &parts);
  if (st != DFLOW_OK) return st;
  if (device < 0 || device >= static_cast<int32_t>(parts.size())) return fail(DFLOW_INVALID_ARGUMENT, "no such device");
  dflow_graph* r = new dflow_graph();
  r->g = std::move(parts[device]);
  *out = r;
  return DFLOW_OK;
  GUARD_END
}

dflow_status dflow_graph_insert_exchange(const dflow_graph* g, int world, int exchange, dflow_graph** out) {
  GUARD_BEGIN
  if (!g || !out) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  const int ex = exchange & ~DFLOW_EXCHANGE_ASYNC;
  if (world < 1 || ex < DFLOW_EXCHANGE_TRUNC16 || ex > DFLOW_EXCHANGE_SR16 || (exchange & ~0x1FF))
    return fail(DFLOW_INVALID_ARGUMENT, "bad world/exchange");
  dflow_graph* r = new dflow_graph();
  std::vector<int> remap;
  dflow_status st = dflow::insert_exchange(g->g, world, exchange, &r->g, &remap);
  if (st != DFLOW_OK) {
    delete r;
    return st;
  }
  *out = r;
  return DFLOW_OK;
  GUARD_END
}

// ------------------------------------------------------------------ session
dflow_status dflow_nccl_unique_id(uint8_t* out128) {
  if (!out128) return fail(DFLOW_INVALID_ARGUMENT, "out is NULL");
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId size");
  ncclUniqueId id;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) return fail(DFLOW_NCCL, "ncclGetUniqueId: %s", ncclGetErrorString(r));
  memcpy(out128, &id, 128);
  return DFLOW_OK;
}

dflow_status dflow_session_create(const dflow_graph* g, const dflow_options* opt, const uint8_t* nccl_id128,
                                  dflow_session** out) {
  GUARD_BEGIN
  if (!g || !opt || !out) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  return dflow::session_create(g->g, *opt, nccl_id128, nullptr, out);
  GUARD_END
}

void dflow_session_destroy(dflow_session* s) {
  try {
    dflow::session_destroy(s);
  } catch (...) {
  }
}

dflow_status dflow_session_graph_to_json(const dflow_session* s, char* buf, size_t cap, size_t* needed) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return json_out(s->g.to_json(), buf, cap, needed);
  GUARD_END
}

dflow_status dflow_variable_assign(dflow_session* s, dflow_node var, const void* src, int src_on_device,
                                   void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_variable_assign(s, var, src, src_on_device, static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_variable_read(dflow_session* s, dflow_node var, void* dst, int dst_on_device, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_variable_read(s, var, dst, dst_on_device, static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_train_step(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* dev_ptrs,
                              const int64_t* ld, int64_t local_rows, float* loss_out, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_train_step(s, n_feeds, feeds, dev_ptrs, ld, local_rows, loss_out,
                                   static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_train_step_host(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                   const void* const* host_ptrs, const int64_t* ld, int64_t local_rows,
                                   float* loss_out, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_train_step_host(s, n_feeds, feeds, host_ptrs, ld, local_rows, loss_out,
                                        static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_train_step_host_pipelined(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                             const void* const* host_ptrs, const int64_t* ld, int64_t local_rows,
                                             float* prev_loss_out, int32_t* has_loss, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_train_step_host(s, n_feeds, feeds, host_ptrs, ld, local_rows, prev_loss_out,
                                        static_cast<cudaStream_t>(stream), true, has_loss);
  GUARD_END
}

dflow_status dflow_session_last_loss(dflow_session* s, float* loss_out, int32_t* has_loss) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_last_loss(s, loss_out, has_loss);
  GUARD_END
}

dflow_status dflow_forward(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* dev_ptrs,
                           const int64_t* ld, int64_t local_rows, dflow_node fetch, void* out_dev, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_forward(s, n_feeds, feeds, dev_ptrs, ld, local_rows, fetch, out_dev,
                                static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_fetch_gradients(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                   const void* const* dev_ptrs, const int64_t* ld, int64_t local_rows, int n,
                                   const dflow_node* grads, void* const* out_dev, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_fetch_gradients(s, n_feeds, feeds, dev_ptrs, ld, local_rows, n, grads, out_dev,
                                        static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_fetch_relu_masks(dflow_session* s, int layer, uint32_t* out_bits_host) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_fetch_masks(s, layer, out_bits_host);
  GUARD_END
}

dflow_status dflow_session_set_timing(dflow_session* s, int enable) {
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  s->timing = enable != 0;
  s->ranges.clear();  // (a partial DFLOW_TIMING_BATCH window is dropped)
  s->event_next = 0;
  s->timing_pending = 0;
  s->gemm_ms = s->other_ms = s->exchange_ms = 0;
  s->timed_steps = 0;
  return DFLOW_OK;
}

dflow_status dflow_session_sync(dflow_session* s, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_sync(s, static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_session_stats(dflow_session* s, dflow_stats* out) {
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_stats(s, out);
}

// ------------------------------------------------------------------ standalone ops
dflow_status dflow_truncate16(const float* src, uint16_t* dst, size_t n, void* stream) {
  if (n && (!src || !dst)) return fail(DFLOW_INVALID_ARGUMENT, "NULL pointer");
  cudaError_t e = dflow::launch_truncate16(src, dst, n, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "truncate16: %s", cudaGetErrorString(e));
  return DFLOW_OK;
}

dflow_status dflow_round16(const float* src, uint16_t* dst, size_t n, uint32_t key, int stochastic, int64_t idx_base,
                           void* stream) {
  if (n && (!src || !dst)) return fail(DFLOW_INVALID_ARGUMENT, "NULL pointer");
  if (idx_base < 0) return fail(DFLOW_INVALID_ARGUMENT, "negative idx_base");
  cudaError_t e = dflow::launch_round16(src, dst, n, dflow::Round16{key, stochastic ? 1 : 0}, idx_base,
                                        static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "round16: %s", cudaGetErrorString(e));
  return DFLOW_OK;
}

dflow_status dflow_round16_key(uint32_t seed, uint32_t step, uint32_t layer, uint32_t stage, uint32_t rank,
                               uint32_t* key_out) {
  if (!key_out) return fail(DFLOW_INVALID_ARGUMENT, "NULL key_out");
  *key_out = dflow::round16_key(seed, step, layer, stage, rank);
  return DFLOW_OK;
}

dflow_status dflow_expand16(const uint16_t* src, float* dst, size_t n, void* stream) {
  if (n && (!src || !dst)) return fail(DFLOW_INVALID_ARGUMENT, "NULL pointer");
  cudaError_t e = dflow::launch_expand16(src, dst, n, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "expand16: %s", cudaGetErrorString(e));
  return DFLOW_OK;
}

dflow_status dflow_async_pull(dflow_session* s, void* stream) {
  GUARD_BEGIN
  if (!s) return fail(DFLOW_INVALID_ARGUMENT, "session is NULL");
  return dflow::session_async_pull(s, static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_exchange(dflow_session* s, const float* grad_dev, float* out_dev, size_t n, void* stream) {
  GUARD_BEGIN
  if (!s || (n && (!grad_dev || !out_dev))) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  return dflow::session_exchange(s, grad_dev, out_dev, n, static_cast<cudaStream_t>(stream));
  GUARD_END
}

dflow_status dflow_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int a_mn, const void* B,
                             int64_t ldb, int b_mn, int epilogue, void* out, int64_t ldo, float* out_f32,
                             int64_t ldo32, const float* bias, const void* mask, int64_t ldm, int tile,
                             void* stream) {
  GUARD_BEGIN
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(DFLOW_CUDA, "no CUDA device");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  dflow::GemmDesc d{};
  d.M = M; d.N = N; d.K = K;
  d.A = A; d.lda = lda; d.a_mn = a_mn != 0;
  d.B = B; d.ldb = ldb; d.b_mn = b_mn != 0;
  d.epilogue = epilogue;
  d.out = out; d.ldo = ldo;
  d.out_f32 = out_f32; d.ldo32 = ldo32;
  d.bias = bias;
  d.mask = mask; d.ldm = ldm;
  d.tile = tile;
  d.sched = dflow::gemm_stream_sched(static_cast<cudaStream_t>(stream));
  dflow::GemmPlan p;
  cudaError_t e = dflow::gemm_prepare(d, sms, &p);
  if (e != cudaSuccess) return fail(DFLOW_INVALID_ARGUMENT, "%s", dflow::gemm_last_error());
  e = dflow::gemm_launch(p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "%s", dflow::gemm_last_error());
  return DFLOW_OK;
  GUARD_END
}

dflow_status dflow_gemm_3xtf32(int64_t M, int64_t N, int64_t K, const float* A_hi, const float* A_lo, int64_t lda,
                               int a_mn, const float* B_hi, const float* B_lo, int64_t ldb, int b_mn, float* out_f32,
                               int64_t ldo32, int tile, void* stream) {
  GUARD_BEGIN
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(DFLOW_CUDA, "no CUDA device");
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  dflow::GemmDesc d{};
  d.tf32 = true;
  d.M = M; d.N = N; d.K = K;
  d.A = A_hi; d.A2 = A_lo; d.lda = lda; d.a_mn = a_mn != 0;
  d.B = B_hi; d.B2 = B_lo; d.ldb = ldb; d.b_mn = b_mn != 0;
  d.epilogue = dflow::EPI_F32;
  d.out_f32 = out_f32; d.ldo32 = ldo32;
  d.tile = tile;
  d.sched = dflow::gemm_stream_sched(static_cast<cudaStream_t>(stream));
  dflow::GemmPlan p;
  cudaError_t e = dflow::gemm_prepare(d, sms, &p);
  if (e != cudaSuccess) return fail(DFLOW_INVALID_ARGUMENT, "%s", dflow::gemm_last_error());
  e = dflow::gemm_launch(p, static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "%s", dflow::gemm_last_error());
  return DFLOW_OK;
  GUARD_END
}

dflow_status dflow_split_tf32(const float* src, float* hi, float* lo, size_t n, void* stream) {
  if (n && (!src || !hi || !lo)) return fail(DFLOW_INVALID_ARGUMENT, "NULL pointer");
  cudaError_t e = dflow::launch_split_tf32(src, 0, hi, lo, 0, 1, static_cast<int64_t>(n),
                                           static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "split_tf32: %s", cudaGetErrorString(e));
  return DFLOW_OK;
}

dflow_status dflow_device_die_map(int32_t device, int32_t* die_of_sm, int32_t n, double* agreement) {
  GUARD_BEGIN
  std::vector<int> m;
  double a = 0.0;
  const bool ok = dflow::measure_die_map(device, &m, &a);
  if (agreement) *agreement = a;
  for (int i = 0; i < n && i < static_cast<int>(m.size()); ++i) if (die_of_sm) die_of_sm[i] = m[i];
  if (m.empty()) return fail(DFLOW_CUDA, "die probe failed on device %d", device);
  return ok ? DFLOW_OK : fail(DFLOW_UNIMPLEMENTED, "no clean two-die split (agreement %.3f)", a);
  GUARD_END
}

// --------------------------------------------------------- simulated world (tests)
dflow_status dflow_sim_world_create(int32_t world, int32_t device, dflow_sim_world** out) {
  GUARD_BEGIN
  if (!out) return fail(DFLOW_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (world < 1 || world > dflow::kMaxRanks) return fail(DFLOW_INVALID_ARGUMENT, "world must be 1..%d", dflow::kMaxRanks);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(DFLOW_CUDA, "no CUDA device available (dflow has no CPU fallback)");
  }
  if (device < 0 || device >= ndev || cudaSetDevice(device) != cudaSuccess)
    return fail(DFLOW_INVALID_ARGUMENT, "bad device ordinal %d", device);
  dflow_sim_world* w = new dflow_sim_world();
  w->world = world;
  w->device = device;
  w->slot.assign(world, nullptr);
  if (const char* e = getenv("DFLOW_SIM_TIMEOUT_MS")) w->timeout_ms = atoll(e) > 0 ? atoll(e) : w->timeout_ms;
  if (cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete w;
    return fail(DFLOW_CUDA, "stream creation failed");
  }
  *out = w;
  return DFLOW_OK;
  GUARD_END
}

void dflow_sim_world_destroy(dflow_sim_world* w) {
  if (!w) return;
  cudaSetDevice(w->device);
  cudaStreamSynchronize(w->stream);
  cudaStreamDestroy(w->stream);
  delete w;
}

dflow_status dflow_sim_world_stream(dflow_sim_world* w, void** stream_out) {
  if (!w || !stream_out) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  *stream_out = w->stream;
  return DFLOW_OK;
}

dflow_status dflow_sim_world_drop_rank(dflow_sim_world* w, int32_t rank) {
  if (!w || rank < -1 || rank >= w->world) return fail(DFLOW_INVALID_ARGUMENT, "bad rank");
  w->drop_rank = rank;
  return DFLOW_OK;
}

dflow_status dflow_sim_sessions_create(dflow_sim_world* w, const dflow_graph* g, const dflow_options* opt,
                                       dflow_session** out) {
  GUARD_BEGIN
  if (!w || !g || !opt || !out) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  for (int r = 0; r < w->world; ++r) out[r] = nullptr;
  const dflow_status st = dflow::sim_run(w, [&](int r) {
    dflow_options o = *opt;
    o.world = w->world;
    o.rank = r;
    o.device = w->device;
    return dflow::session_create(g->g, o, nullptr, w, &out[r]);
  });
  if (st != DFLOW_OK) {
    const std::string msg = dflow_last_error();
    for (int r = 0; r < w->world; ++r) {
      dflow::session_destroy(out[r]);
      out[r] = nullptr;
    }
    return fail(st, "%s", msg.c_str());
  }
  return DFLOW_OK;
  GUARD_END
}

dflow_status dflow_sim_train_step(dflow_sim_world* w, dflow_session* const* sessions, int n_feeds,
                                  const dflow_node* feeds, const void* const* dev_ptrs, const int64_t* ld,
                                  int64_t local_rows, float* loss_out) {
  GUARD_BEGIN
  if (!w || !sessions || n_feeds < 0 || (n_feeds > 0 && (!feeds || !dev_ptrs || !ld)))
    return fail(DFLOW_INVALID_ARGUMENT, "bad arguments");
  for (int r = 0; r < w->world; ++r)
    if (!sessions[r] || sessions[r]->sim != w || sessions[r]->opt.rank != r)
      return fail(DFLOW_INVALID_ARGUMENT, "sessions[%d] is not rank %d of this world", r, r);
  return dflow::sim_run(w, [&](int r) {
    return dflow::session_train_step(sessions[r], n_feeds, feeds, dev_ptrs + static_cast<size_t>(r) * n_feeds, ld,
                                     local_rows, loss_out ? loss_out + r : nullptr, w->stream);
  });
  GUARD_END
}

dflow_status dflow_sim_exchange(dflow_sim_world* w, dflow_session* const* sessions, const float* const* grads,
                                float* const* outs, size_t n) {
  GUARD_BEGIN
  if (!w || !sessions || !grads || !outs) return fail(DFLOW_INVALID_ARGUMENT, "NULL argument");
  for (int r = 0; r < w->world; ++r)
    if (!sessions[r] || sessions[r]->sim != w || sessions[r]->opt.rank != r)
      return fail(DFLOW_INVALID_ARGUMENT, "sessions[%d] is not rank %d of this world", r, r);
  return dflow::sim_run(
      w, [&](int r) { return dflow::session_exchange(sessions[r], grads[r], outs[r], n, w->stream); });
  GUARD_END
}

}  // extern "C"
