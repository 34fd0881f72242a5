// Replicated train-step session: planner (graph -> fused kernel schedule),
// device state, NCCL exchange, and the step executor.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <string>
#include <vector>

#include "../../include/dflow.h"
#include "comm.h"
#include "graph.h"
#include "kernels/async_dp.h"
#include "kernels/exchange_p2p.h"
#include "kernels/gemm.h"

namespace dflow {

// One Relu(A W + b) block of the chain plus its gradient nodes (session-graph ids).
struct LayerNodes {
  int W = -1, b = -1, mm = -1, add = -1, relu = -1;
  int relugrad = -1, db = -1, dW = -1, dX = -1;
  int apply_W = -1, apply_b = -1;
  float lr_W = 0.f, lr_b = 0.f;
};

// A GEMM operand in HBM: bf16 path -> hi only (bf16); 3xTF32 path -> the pair
// hi = tf32_rna(x), lo = x - hi (fp32 each), same layout (reading A14).
struct Operand {
  void* hi = nullptr;
  void* lo = nullptr;
};

struct Layer {
  LayerNodes n;
  int64_t in = 0, out = 0;
  int64_t ld_out = 0;             // padded leading dim (elements) of [rows, out] operand buffers
  int64_t ld_wb = 0;              // padded leading dim of the weight operand copy [in, ld_wb]
  float* W32 = nullptr;           // fp32 master [in*out] dense
  Operand Wop;                    // operand copy of W [in, ld_wb]
  float* b32 = nullptr;           // fp32 [out]
  Operand A;                      // activation [cap, ld_out] (layers 1..L-1)
  Operand dZ;                     // [cap, ld_out]
  // gradient bucket [dW_l || db_l], padded to Ppad = roundup(P, 8N)
  int64_t P = 0, Ppad = 0, shard = 0;
  float* g32 = nullptr;           // fp32 gradient bucket [Ppad]
  uint16_t* q16 = nullptr;        // TRUNC16 send bucket [Ppad]
  void* recv = nullptr;           // alltoall landing [Ppad] (u16 or f32)
  void* own = nullptr;            // owner's reduced shard [shard]
  void* gath = nullptr;           // allgather landing [Ppad]
  float* colsum_ws = nullptr;     // fused db partials [ceil(cap/32), out]
  P2PLayer p2p;                   // fused NVLink exchange: peer pointers of this layer
  AsyncLayer async;               // asynchronous replicas (f3): every rank's shard of this layer
  GemmPlan fwd, fwd_fetch, fwd_plain, dgrad, wgrad32, wgrad16, wgrad_apply, wgrad_p2p, wgrad_async;
  GemmPlan fwd_send, dgrad_send;  // f4 channel ends: truncation-coded activation out / dA out
  bool has_fwd = false, has_dgrad = false, has_wgrad16 = false, has_wgrad_apply = false, has_wgrad_p2p = false;
};

struct TimedRange {
  int kind;  // 0 gemm, 1 other, 2 exchange
  cudaEvent_t a, b;
  int comm;           // 1: launched on the comm stream
  const char* label;  // GEMM epilogue name (timeline dump)
};

}  // namespace dflow

struct dflow_session {
  dflow::Graph g;                 // rewritten (replicated + compression) graph
  std::vector<int> remap;         // user graph id -> session graph id
  dflow_options opt{};
  int L = 0;
  std::vector<dflow::Layer> layers;
  int x = -1, y = -1, cost = -1, lossgrad = -1, loss_kind = 0;
  dflow_dtype x_dtype = DFLOW_F32;
  bool trainable = false;
  int64_t cap = 0;
  int num_sms = 148;
  int64_t planned_rows = -1;
  bool tf32 = false;              // DFLOW_PRECISION_3XTF32
  int esz = 2;                    // operand element bytes (2 bf16, 4 fp32)
  dflow::Operand A0;              // operand copy of the x feed [cap, ld_A0]
  int64_t ld_A0 = 0;
  float* AL32 = nullptr;          // fp32 last activation [cap, ld_AL32]
  int64_t ld_AL32 = 0;
  double* loss_partials = nullptr;
  float* loss_dev = nullptr;      // [2]: local C_r, reduced sum
  float* loss_host = nullptr;     // pinned
  uint32_t* mask_dev = nullptr;
  int64_t mask_words_cap = 0;
  void* xbuf[4] = {nullptr, nullptr, nullptr, nullptr};  // dflow_exchange scratch (grow-only)
  size_t xbuf_bytes = 0;
  uint32_t xchg_calls = 0;  // standalone dflow_exchange calls (the SR16 step counter there)
  void* host_stage[2] = {nullptr, nullptr};  // device copies of host feeds (e2e path)
  size_t host_stage_bytes[2] = {0, 0};
  cudaStream_t comm = nullptr;
  std::vector<cudaEvent_t> ev_grad, ev_apply;
  // opt.defer_apply: layer l's update (ev_apply[l], comm stream) not yet joined by any
  // stream; the next forward waits per layer, every other entry point joins all
  bool defer = false;
  bool apply_pending = false;
  // N = 1, small layers (all dW grids + the largest dgrad grid <= #SMs): dW_l and db_l run
  // on side[l % 2], concurrently with the next dgrad and with dW_{l-1} (no shared buffers)
  cudaStream_t side[2] = {nullptr, nullptr};
  cudaEvent_t ev_side_join[2] = {nullptr, nullptr};
  int* sched_w = nullptr;  // [2][4] tile-scheduler counters of the dW GEMMs, per side stream
  bool bwd_side = false;
  cudaEvent_t ev_loss = nullptr;
  // loss value landed in loss_host[slot] (after the forward); two slots so a pipelined
  // host step can enqueue step i+1 while step i's loss is still unread
  cudaEvent_t ev_loss_ready[2] = {nullptr, nullptr};
  bool loss_pending[2] = {false, false};
  int loss_slot = 0;
  // e2e path: host feeds are copied on their own stream so step i+1's upload overlaps
  // step i's backward; ev_feeds_free marks the forward done reading the staging buffers
  // (x is uploaded first; y, needed only by the last layer's loss epilogue, uploads while
  // the first layers run: the step's forward waits on ev_h2d, its last GEMM on ev_h2d_y)
  cudaStream_t h2d = nullptr;
  cudaEvent_t ev_h2d = nullptr, ev_h2d_y = nullptr, ev_feeds_free = nullptr;
  cudaEvent_t ev_x_free = nullptr;  // the input cast is done with the x staging buffer
  bool y_upload_pending = false;
  // opt.graphs: captured train steps keyed by their feed signature, replayed on gstream
  struct StepGraph {
    const void* x;
    const void* y;
    int64_t ldx, ldy, rows;
    bool loss;
    bool ywait;
    int slot;  // loss slot the captured copy writes
    cudaGraphExec_t exec;
  };
  std::vector<StepGraph> step_graphs;
  cudaStream_t gstream = nullptr;
  cudaEvent_t ev_gin = nullptr, ev_gout = nullptr;
  bool capturing = false;
  ncclComm_t nccl = nullptr;
  // simulated N-rank world on one GPU (comm.h; the test harness of the N-GPU path): the
  // transport's collectives become host rendezvous + device copies; comm is the world's
  // shared stream (not owned)
  dflow_sim_world* sim = nullptr;
  void* sim_scratch = nullptr;
  size_t sim_scratch_bytes = 0;
  bool comm_owned = true;
  // bounded cross-GPU flag waits (exchange_p2p.h): a wait that times out writes a code here
  // (pinned, mapped) and its kernel returns; the next call poisons the session
  uint32_t* abort_host = nullptr;
  uint32_t* abort_dev = nullptr;
  uint64_t flag_timeout_ns = 0;
  int* sched_fd = nullptr;  // [2][4] tile-scheduler counters of this session's forward / dgrad GEMMs
  // f1 multicast (bf16 owner-apply over NCCL): every layer's bf16 W copy lives in one symmetric
  // NCCL window whose multicast address the owner fold stores through (comm.h)
  dflow::SymRegion* wsym = nullptr;
  bool multicast = false;
  // the cost's cross-replica mean over peer memory (fused channel, no NCCL call in the step):
  // every rank's loss slots / flags in its symmetric allocation; the gather runs on loss_stream
  dflow::LossPeers loss_peers{};
  cudaStream_t loss_stream = nullptr;
  // fused NVLink exchange (opt.p2p): one symmetric allocation per rank, peers via CUDA IPC
  bool p2p = false;
  bool async = false;  // opt.async_dp (f3): sym holds this rank's parameter shards
  // opt.model_parallel (f4): this rank holds layers [mp_lo, mp_hi); channel buffers
  bool mp = false;
  int replicas = 1;    // data-parallel replicas (world, or 1 under model parallelism)
  int mp_lo = 0, mp_hi = 0;
  uint16_t* mp_recv = nullptr;  // codes of dA of layer mp_hi-1 from rank+1 [cap, ld_out]
  void* sym = nullptr;
  void* peer_sym[dflow::kMaxRanks] = {};
  std::vector<void*> ipc_opened;  // CUDA IPC mappings of the peers' allocations (closed at destroy)
  int* p2p_done = nullptr;
  uint32_t epoch = 0;
  bool poisoned = false;
  bool have_forward = false;
  int64_t last_rows = 0;
  // timing / stats
  bool timing = false;
  int timing_pending = 0;  // steps whose events are not read back yet (DFLOW_TIMING_BATCH)
  std::vector<dflow::TimedRange> ranges;
  std::vector<cudaEvent_t> event_pool;
  size_t event_next = 0;
  double gemm_ms = 0, other_ms = 0, exchange_ms = 0;
  int64_t timed_steps = 0;
  int launches = 0, gemm_launches = 0;
  int last_launches = 0, last_gemm_launches = 0;
  int nonfinite = 0;
};

namespace dflow {
// sim != NULL: this session is rank opt.rank of a simulated world on one GPU (comm.h)
dflow_status session_create(const Graph& user, const dflow_options& opt, const uint8_t* nccl_id,
                            dflow_sim_world* sim, dflow_session** out);
void session_destroy(dflow_session* s);
dflow_status session_train_step(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* ptrs,
                                const int64_t* ld, int64_t rows, float* loss_out, cudaStream_t st);
dflow_status session_train_step_host(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                     const void* const* host_ptrs, const int64_t* ld, int64_t rows,
                                     float* loss_out, cudaStream_t st, bool pipelined = false,
                                     int32_t* has_loss = nullptr);
dflow_status session_last_loss(dflow_session* s, float* loss_out, int32_t* has_loss);
dflow_status session_forward(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* ptrs,
                             const int64_t* ld, int64_t rows, dflow_node fetch, void* out, cudaStream_t st);
dflow_status session_fetch_gradients(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                     const void* const* ptrs, const int64_t* ld, int64_t rows, int n,
                                     const dflow_node* grads, void* const* out, cudaStream_t st);
dflow_status session_fetch_masks(dflow_session* s, int layer, uint32_t* bits_host);
dflow_status session_variable_assign(dflow_session* s, dflow_node var, const void* src, int on_dev, cudaStream_t st);
dflow_status session_variable_read(dflow_session* s, dflow_node var, void* dst, int on_dev, cudaStream_t st);
dflow_status session_async_pull(dflow_session* s, cudaStream_t st);
dflow_status session_exchange(dflow_session* s, const float* grad, float* out, size_t n, cudaStream_t st);
dflow_status session_stats(dflow_session* s, dflow_stats* out);
dflow_status session_sync(dflow_session* s, cudaStream_t st);
}  // namespace dflow
