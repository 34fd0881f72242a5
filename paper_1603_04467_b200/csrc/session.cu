// Replicated synchronous train step (§7 :934-941, Fig.7 top) on one GPU
// per replica: planner, device state, NCCL exchange with the §5.5 codec, executor.
//
// Step schedule for rank r (local batch b = B/N, reading A4):
//   cast x -> A0 (bf16)                                   NK13
//   l = 1..L:  A_l = relu(A_{l-1} W_l + b_l)              NK1 (tcgen05 GEMM, fused epilogue)
//              (l = L: + loss seed dZ_L, C_r partials and db_L partials, NK7 fused)
//   l = L..1:  dZ_{l-1} = (dZ_l W_l^T) . 1[A_{l-1} > 0]   NK2 (l > 1; + db_{l-1} partials fused)
//              dW_l = A_{l-1}^T dZ_l  [-> trunc16]        NK3
//              db_l = sum of the per-32-row partials [-> trunc16]   NK8 (final pass)
//              comm stream: alltoall -> owner fold -> allgather (NCCL, NVLink)   NK11
//              W_l, b_l <- W - lr * expand(g_hat)         NK12
#include "session.h"

#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <set>
#include <tuple>

#include "common.h"
#include "kernels/elementwise.h"
#include "sim.h"

namespace dflow {

namespace {

// Tile-raster group (M tiles per group) of one GEMM kind: forward, dgrad or wgrad. The three
// kinds stream different panels, so each has its own A/B knob; 0 leaves the
// plan's default (8); DFLOW_GEMM_GROUP, when set, still overrides every kind.
constexpr int kGroupFwd = 0, kGroupDgrad = 0, kGroupWgrad = 0;
int raster_group(const char* env, int def) {
  const char* e = getenv(env);
  return (e && atoi(e) > 0) ? atoi(e) : def;
}

#define CU(expr)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (expr);                                                             \
    if (e_ != cudaSuccess) {                                                             \
      s->poisoned = true;                                                                \
      return fail(DFLOW_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    }                                                                                    \
  } while (0)

#define NC(expr)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (expr);                                                             \
    if (r_ != ncclSuccess) {                                                              \
      s->poisoned = true;                                                                 \
      return fail(DFLOW_NCCL, "%s failed: %s", #expr, ncclGetErrorString(r_));           \
    }                                                                                     \
  } while (0)

#define ST(expr)                        \
  do {                                  \
    dflow_status st_ = (expr);          \
    if (st_ != DFLOW_OK) return st_;    \
  } while (0)

inline int64_t pad_to(int64_t x, int64_t m) { return (x + m - 1) / m * m; }

dflow_status check_alive(dflow_session* s);
dflow_status setup_multicast(dflow_session* s);
int tbegin(dflow_session* s, int kind, cudaStream_t st);
void tend(dflow_session* s, int idx, cudaStream_t st);
dflow_status check_launch(dflow_session* s, cudaError_t e, int count, const char* what);
cudaError_t record_event(dflow_session* s, cudaEvent_t e, cudaStream_t st);

// Gradients cross the channel as 16-bit codes (TRUNC16 or SR16).
inline bool u16_wire(const dflow_session* s) {
  return s->opt.exchange == DFLOW_EXCHANGE_TRUNC16 || s->opt.exchange == DFLOW_EXCHANGE_SR16;
}

// The coding of layer l's bucket at compression point `stage` (0: this rank as sender,
// 1: this rank as owner of the mean) in the current train step (epoch, 1-based).
inline Round16 round16_of(const dflow_session* s, int l, int stage) {
  if (s->opt.exchange != DFLOW_EXCHANGE_SR16) return Round16{0, 0};
  return Round16{round16_key(s->opt.sr_seed, s->epoch, static_cast<uint32_t>(l), static_cast<uint32_t>(stage),
                             static_cast<uint32_t>(s->opt.rank)),
                 1};
}

int find_node(const Graph& g, Op op, const std::vector<int>& inputs, int ta = -1, int tb = -1) {
  for (size_t i = 0; i < g.nodes.size(); ++i) {
    const Node& n = g.nodes[i];
    if (n.op != op || n.inputs != inputs) continue;
    if (ta >= 0 && (n.transpose_a != ta || n.transpose_b != tb)) continue;
    return static_cast<int>(i);
  }
  return -1;
}

// --------------------------------------------------------------------- planner
dflow_status match_graph(dflow_session* s) {
  const Graph& g = s->g;
  const int n = static_cast<int>(g.nodes.size());
  std::vector<char> used(n, 0);
  int loss = -1;
  for (int i = 0; i < n; ++i)
    if (g.nodes[i].op == Op::Loss) {
      if (loss >= 0) return fail(DFLOW_UNIMPLEMENTED, "planner: more than one Loss node");
      loss = i;
    }
  if (loss < 0) return fail(DFLOW_UNIMPLEMENTED, "planner: the graph has no Loss node");
  s->cost = loss;
  s->loss_kind = g.nodes[loss].loss_kind;
  used[loss] = 1;
  if (s->loss_kind == DFLOW_LOSS_MSE) {
    s->y = g.nodes[loss].inputs[1];
    if (g.nodes[s->y].op != Op::Placeholder || g.nodes[s->y].dtype != DFLOW_F32)
      return fail(DFLOW_UNIMPLEMENTED, "planner: the MSE target must be an fp32 Placeholder");
    used[s->y] = 1;
  }
  // walk the forward chain back from the loss prediction
  std::vector<LayerNodes> rev;
  int cur = g.nodes[loss].inputs[0];
  for (;;) {
    LayerNodes ln;
    const Node& r = g.nodes[cur];
    if (r.op != Op::Relu) return fail(DFLOW_UNIMPLEMENTED, "planner: '%s' is not a Relu block", r.name.c_str());
    ln.relu = cur;
    ln.add = r.inputs[0];
    const Node& a = g.nodes[ln.add];
    if (a.op != Op::Add) return fail(DFLOW_UNIMPLEMENTED, "planner: '%s' is not Add(MatMul, bias)", a.name.c_str());
    ln.mm = a.inputs[0];
    ln.b = a.inputs[1];
    const Node& m = g.nodes[ln.mm];
    const Node& bn = g.nodes[ln.b];
    if (m.op != Op::MatMul || m.transpose_a || m.transpose_b || bn.op != Op::Variable || bn.shape.size() != 1)
      return fail(DFLOW_UNIMPLEMENTED, "planner: '%s' is not Add(MatMul(a, W), b)", a.name.c_str());
    ln.W = m.inputs[1];
    const Node& Wn = g.nodes[ln.W];
    if (Wn.op != Op::Variable || Wn.shape.size() != 2)
      return fail(DFLOW_UNIMPLEMENTED, "planner: '%s' needs a rank-2 Variable weight", m.name.c_str());
    rev.push_back(ln);
    const int prev = m.inputs[0];
    if (g.nodes[prev].op == Op::Placeholder) {
      s->x = prev;
      break;
    }
    cur = prev;
  }
  std::reverse(rev.begin(), rev.end());
  s->L = static_cast<int>(rev.size());
  const Node& xn = g.nodes[s->x];
  if (xn.shape.size() != 2) return fail(DFLOW_UNIMPLEMENTED, "planner: x must be rank 2");
  s->x_dtype = xn.dtype;
  used[s->x] = 1;
  s->layers.assign(s->L, Layer());
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    ly.n = rev[l];
    ly.in = g.nodes[ly.n.W].shape[0];
    ly.out = g.nodes[ly.n.W].shape[1];
    if (g.nodes[ly.n.b].shape[0] != ly.out) return fail(DFLOW_UNIMPLEMENTED, "planner: bias length mismatch");
    if (l > 0 && ly.in != s->layers[l - 1].out) return fail(DFLOW_UNIMPLEMENTED, "planner: layer widths do not chain");
    for (int id : {ly.n.W, ly.n.b, ly.n.mm, ly.n.add, ly.n.relu}) {
      if (used[id]) return fail(DFLOW_UNIMPLEMENTED, "planner: node '%s' is shared between layers", g.nodes[id].name.c_str());
      used[id] = 1;
    }
  }
  if (xn.shape[1] != s->layers[0].in) return fail(DFLOW_UNIMPLEMENTED, "planner: x width != W1 rows");
  // gradient graph: LossGrad -> (ReluGrad -> ReduceSum, MatMul^T...) per layer
  std::vector<int> lg_in = g.nodes[loss].inputs;
  s->lossgrad = find_node(g, Op::LossGrad, lg_in);
  if (s->lossgrad >= 0) {
    if (g.nodes[s->lossgrad].loss_kind != s->loss_kind) return fail(DFLOW_UNIMPLEMENTED, "planner: LossGrad kind");
    used[s->lossgrad] = 1;
    int gin = s->lossgrad;
    for (int l = s->L - 1; l >= 0; --l) {
      Layer& ly = s->layers[l];
      const int aprev = (l == 0) ? s->x : s->layers[l - 1].n.relu;
      ly.n.relugrad = find_node(g, Op::ReluGrad, {gin, ly.n.relu});
      if (ly.n.relugrad < 0)
        return fail(DFLOW_UNIMPLEMENTED, "planner: layer %d has no ReluGrad(g, relu) node on the gradient path", l + 1);
      ly.n.db = find_node(g, Op::ReduceSum, {ly.n.relugrad});
      ly.n.dW = find_node(g, Op::MatMul, {aprev, ly.n.relugrad}, 1, 0);
      ly.n.dX = find_node(g, Op::MatMul, {ly.n.relugrad, ly.n.W}, 0, 1);
      if (ly.n.db < 0 || ly.n.dW < 0)
        return fail(DFLOW_UNIMPLEMENTED, "planner: layer %d gradient nodes (db, dW) not found", l + 1);
      for (int id : {ly.n.relugrad, ly.n.db, ly.n.dW}) used[id] = 1;
      if (ly.n.dX >= 0) used[ly.n.dX] = 1;
      if (l > 0) {
        if (ly.n.dX < 0) return fail(DFLOW_UNIMPLEMENTED, "planner: layer %d has no dX node", l + 1);
        gin = ly.n.dX;
      }
    }
  }
  // ApplyGradientDescent nodes, through the exchange chain the compression pass inserted
  const bool xchg = s->replicas > 1 && s->opt.exchange != DFLOW_EXCHANGE_NONE;
  int applies = 0;
  for (int i = 0; i < n; ++i) {
    const Node& ap = g.nodes[i];
    if (ap.op != Op::ApplyGradientDescent) continue;
    int gid = ap.inputs[1];
    std::vector<int> chain;
    if (xchg && s->async && !u16_wire(s)) {
      // asynchronous FP32 channel: the replica's gradient feeds its apply directly
    } else if (xchg && u16_wire(s)) {
      const bool sr = s->opt.exchange == DFLOW_EXCHANGE_SR16;
      const int e = gid;
      if (g.nodes[e].op != Op::Expand16) return fail(DFLOW_UNIMPLEMENTED, "planner: missing Expand16 before apply");
      int m = g.nodes[e].inputs[0];
      if (!s->async) {  // synchronous: the cross-replica mean sits between the code and the expand
        if (g.nodes[m].op != (sr ? Op::CrossReplicaMeanSR16 : Op::CrossReplicaMeanT16))
          return fail(DFLOW_UNIMPLEMENTED, "planner: missing exchange");
        chain.push_back(m);
        m = g.nodes[m].inputs[0];
      }
      const int t = m;
      if (g.nodes[t].op != (sr ? Op::StochasticRound16 : Op::Truncate16))
        return fail(DFLOW_UNIMPLEMENTED, "planner: missing the 32->16 coding node");
      chain.push_back(e);
      chain.push_back(t);
      gid = g.nodes[t].inputs[0];
    } else if (xchg) {
      if (g.nodes[gid].op != Op::CrossReplicaMean) return fail(DFLOW_UNIMPLEMENTED, "planner: missing exchange");
      chain = {gid};
      gid = g.nodes[gid].inputs[0];
    }
    bool matched = false;
    for (Layer& ly : s->layers) {
      if (ap.inputs[0] == ly.n.W && gid == ly.n.dW && ly.n.apply_W < 0) {
        ly.n.apply_W = i;
        ly.n.lr_W = ap.lr;
        matched = true;
      } else if (ap.inputs[0] == ly.n.b && gid == ly.n.db && ly.n.apply_b < 0) {
        ly.n.apply_b = i;
        ly.n.lr_b = ap.lr;
        matched = true;
      }
      if (matched) break;
    }
    if (!matched)
      return fail(DFLOW_UNIMPLEMENTED, "planner: '%s' does not apply its own layer's gradient", ap.name.c_str());
    used[i] = 1;
    for (int c : chain) used[c] = 1;
    ++applies;
  }
  s->trainable = applies == 2 * s->L;
  if (applies != 0 && !s->trainable)
    return fail(DFLOW_UNIMPLEMENTED, "planner: every W_l and b_l needs exactly one ApplyGradientDescent");
  for (int i = 0; i < n; ++i)
    if (!used[i])
      return fail(DFLOW_UNIMPLEMENTED, "planner: node '%s' (%s) is not part of a fusable MLP train step",
                  g.nodes[i].name.c_str(), op_name(g.nodes[i].op));
  return DFLOW_OK;
}

template <typename T>
dflow_status dmalloc(dflow_session* s, T** p, size_t elems) {
  if (elems == 0) elems = 1;
  void* v = nullptr;
  cudaError_t e = cudaMalloc(&v, elems * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(DFLOW_OOM, "cudaMalloc(%zu bytes) failed: %s", elems * sizeof(T), cudaGetErrorString(e));
  }
  e = cudaMemset(v, 0, elems * sizeof(T));
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "cudaMemset failed: %s", cudaGetErrorString(e));
  *p = static_cast<T*>(v);
  return DFLOW_OK;
}

// bf16 operand, or the fp32 (hi, lo) pair of the 3xTF32 path
dflow_status alloc_operand(dflow_session* s, Operand* op, size_t elems) {
  if (s->tf32) {
    float *h, *l;
    ST(dmalloc(s, &h, elems));
    ST(dmalloc(s, &l, elems));
    op->hi = h;
    op->lo = l;
  } else {
    __nv_bfloat16* h;
    ST(dmalloc(s, &h, elems));
    op->hi = h;
    op->lo = nullptr;
  }
  return DFLOW_OK;
}

void free_operand(Operand& op) {
  if (op.hi) cudaFree(op.hi);
  if (op.lo) cudaFree(op.lo);
  op.hi = op.lo = nullptr;
}

// Refresh the operand copy of a fp32 matrix src [rows, lds] (RNE bf16 or the tf32 split).
cudaError_t to_operand(dflow_session* s, const float* src, int64_t lds, const Operand& op, int64_t ldd, int64_t rows,
                       int64_t cols, cudaStream_t st) {
  if (s->tf32)
    return launch_split_tf32(src, lds, static_cast<float*>(op.hi), static_cast<float*>(op.lo), ldd, rows, cols, st);
  return launch_cast_bf16(src, lds, static_cast<__nv_bfloat16*>(op.hi), ldd, rows, cols, st);
}

// f4: layer-wise placement (reading A32) and the check that the partition pass puts the
// channels exactly where the runtime implements them: per boundary, the activation forward
// and its gradient (dA) backward, both through the 16-bit codec (A33).
dflow_status setup_mp(dflow_session* s) {
  const int N = s->opt.world, L = s->L, R = s->opt.rank;
  if (N > L) return fail(DFLOW_INVALID_ARGUMENT, "model_parallel needs at least as many layers (%d) as ranks (%d)", L, N);
  auto dev = [&](int l) { return (l * N) / L; };
  std::vector<int> place(s->g.nodes.size(), -1);
  for (int l = 0; l < L; ++l) {
    const LayerNodes& n = s->layers[l].n;
    for (int id : {n.W, n.b, n.mm, n.add, n.relu, n.relugrad, n.db, n.dW, n.dX, n.apply_W, n.apply_b})
      if (id >= 0) place[id] = dev(l);
  }
  place[s->x] = 0;
  for (int id : {s->y, s->cost, s->lossgrad})
    if (id >= 0) place[id] = dev(L - 1);
  for (size_t i = 0; i < place.size(); ++i)
    if (place[i] < 0) return fail(DFLOW_UNIMPLEMENTED, "model_parallel: node '%s' has no placement", s->g.nodes[i].name.c_str());
  std::vector<Graph> parts;
  ST(partition(s->g, place, true, &parts));
  std::set<std::tuple<std::string, int, int>> got, want;
  for (const Graph& g : parts)
    for (const Node& n : g.nodes)
      if (n.op == Op::Send) got.insert(std::make_tuple(n.tensor_name, n.send_device, n.recv_device));
  for (int l = 1; l < L; ++l) {
    if (dev(l) == dev(l - 1)) continue;
    want.insert(std::make_tuple(s->g.nodes[s->layers[l - 1].n.relu].name, dev(l - 1), dev(l)));
    if (s->layers[l].n.dX >= 0) want.insert(std::make_tuple(s->g.nodes[s->layers[l].n.dX].name, dev(l), dev(l - 1)));
  }
  if (got != want) return fail(DFLOW_UNIMPLEMENTED, "model_parallel: the partition's channels are not the MLP's boundary pair");
  s->mp_lo = L;
  s->mp_hi = 0;
  for (int l = 0; l < L; ++l)
    if (dev(l) == R) {
      s->mp_lo = std::min(s->mp_lo, l);
      s->mp_hi = std::max(s->mp_hi, l + 1);
    }
  return DFLOW_OK;
}

dflow_status alloc_state(dflow_session* s) {
  const int N = s->replicas;
  const int64_t cap = s->cap;
  s->ld_A0 = pad_to(s->layers[0].in, 8);
  ST(alloc_operand(s, &s->A0, cap * s->ld_A0));
  int64_t max_out = 0;
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    ly.ld_out = pad_to(ly.out, 8);
    ly.ld_wb = pad_to(ly.out, 8);
    ST(dmalloc(s, &ly.W32, ly.in * ly.out));
    ST(alloc_operand(s, &ly.Wop, ly.in * ly.ld_wb));
    ST(dmalloc(s, &ly.b32, ly.out));
    if (l + 1 < s->L) ST(alloc_operand(s, &ly.A, cap * ly.ld_out));
    ST(alloc_operand(s, &ly.dZ, cap * ly.ld_out));
    ly.P = ly.in * ly.out + ly.out;
    ly.Ppad = pad_to(ly.P, 8 * N);
    ly.shard = ly.Ppad / N;
    ST(dmalloc(s, &ly.g32, ly.Ppad));
    ST(dmalloc(s, &ly.colsum_ws, ((cap + 31) / 32) * ly.out));
    if (N > 1 && u16_wire(s) && !s->p2p && !s->async) {
      ST(dmalloc(s, &ly.q16, ly.Ppad));
      uint16_t *r, *o, *gt;
      ST(dmalloc(s, &r, ly.Ppad));
      ST(dmalloc(s, &o, ly.shard));
      ST(dmalloc(s, &gt, ly.Ppad));
      ly.recv = r; ly.own = o; ly.gath = gt;
    } else if (N > 1 && s->opt.exchange == DFLOW_EXCHANGE_FP32 && !s->async) {
      float *r, *o, *gt;
      ST(dmalloc(s, &r, ly.Ppad));
      ST(dmalloc(s, &o, ly.shard));
      ST(dmalloc(s, &gt, ly.Ppad));
      ly.recv = r; ly.own = o; ly.gath = gt;
    }
    max_out = std::max(max_out, ly.out);
  }
  s->ld_AL32 = pad_to(s->layers[s->L - 1].out, 4);
  ST(dmalloc(s, &s->AL32, cap * s->ld_AL32));
  {  // one fp64 loss partial per (tile, CTA, warp) of the last forward GEMM, either tile config
    const int64_t outL = s->layers[s->L - 1].out;
    ST(dmalloc(s, &s->loss_partials, ((cap + 127) / 128) * ((outL + 127) / 128) * 8));
  }
  ST(dmalloc(s, &s->loss_dev, 4));
  s->mask_words_cap = (cap * std::max(max_out, s->layers[0].in) + 31) / 32;
  ST(dmalloc(s, &s->mask_dev, s->mask_words_cap));
  if (cudaMallocHost(&s->loss_host, 4 * sizeof(float)) != cudaSuccess)
    return fail(DFLOW_OOM, "cudaMallocHost failed");
  // the comm stream gets the highest priority: its exchange kernels take SMs at the next
  // GEMM boundary instead of queueing behind the following persistent GEMM's CTAs
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  if (s->sim) {  // simulated world: every rank's work goes to the world's one stream (comm.h)
    s->comm = s->sim->stream;
    s->comm_owned = false;
  } else if (cudaStreamCreateWithPriority(&s->comm, cudaStreamNonBlocking, prio_hi) != cudaSuccess) {
    return fail(DFLOW_CUDA, "stream creation failed");
  }
  // bounded flag waits: the abort word the wait kernels write on a timeout (host-mapped, so
  // it is read without synchronising), and the timeout (DFLOW_P2P_TIMEOUT_MS, default 60 s)
  if (cudaHostAlloc(&s->abort_host, sizeof(uint32_t), cudaHostAllocMapped) != cudaSuccess)
    return fail(DFLOW_OOM, "cudaHostAlloc failed");
  *s->abort_host = 0;
  CU(cudaHostGetDevicePointer(&s->abort_dev, s->abort_host, 0));
  {
    const char* e = getenv("DFLOW_P2P_TIMEOUT_MS");
    const double ms = (e && atof(e) > 0) ? atof(e) : 60000.0;
    s->flag_timeout_ns = static_cast<uint64_t>(ms * 1e6);
  }
  ST(dmalloc(s, &s->sched_fd, 8));  // zeroed: forward [0, 4) and dgrad [4, 8) plans of this session
  s->ev_grad.resize(s->L);
  s->ev_apply.resize(s->L);
  for (int l = 0; l < s->L; ++l) {
    cudaEventCreateWithFlags(&s->ev_grad[l], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&s->ev_apply[l], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&s->ev_loss, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_loss_ready[0], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_loss_ready[1], cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_x_free, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_h2d, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_h2d_y, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_gin, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&s->ev_gout, cudaEventDisableTiming);
  if (cudaStreamCreateWithFlags(&s->gstream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(DFLOW_CUDA, "stream creation failed");
  cudaEventCreateWithFlags(&s->ev_feeds_free, cudaEventDisableTiming);
  if (cudaStreamCreateWithFlags(&s->h2d, cudaStreamNonBlocking) != cudaSuccess)
    return fail(DFLOW_CUDA, "stream creation failed");
  for (int i = 0; i < 2; ++i) {
    if (cudaStreamCreateWithFlags(&s->side[i], cudaStreamNonBlocking) != cudaSuccess)
      return fail(DFLOW_CUDA, "stream creation failed");
    cudaEventCreateWithFlags(&s->ev_side_join[i], cudaEventDisableTiming);
  }
  ST(dmalloc(s, &s->sched_w, 8));  // zeroed: [4] per side stream
  return DFLOW_OK;
}

// Fused NVLink exchange setup: one symmetric allocation per rank (identical layout on
// every rank: per layer the receive area [N * shard], the gathered bucket [N * shard]
// and the flags [2][kMaxRanks]); CUDA IPC handles are exchanged over NCCL and the
// peers' allocations mapped, so kernels can store into them directly over NVLink.
dflow_status setup_p2p(dflow_session* s) {
  const int N = s->opt.world, R = s->opt.rank;
  if (N > kMaxRanks) return fail(DFLOW_INVALID_ARGUMENT, "the p2p exchange supports up to %d ranks", kMaxRanks);
  std::vector<size_t> off_recv(s->L), off_gath(s->L), off_flags(s->L);
  size_t total = 0;
  auto take = [&](size_t bytes) {
    const size_t o = total;
    total += (bytes + 255) / 256 * 256;
    return o;
  };
  for (int l = 0; l < s->L; ++l) {
    off_recv[l] = take(s->layers[l].Ppad * 2);
    off_gath[l] = take(s->layers[l].Ppad * 2);
    off_flags[l] = take(2 * kMaxRanks * sizeof(uint32_t));
  }
  const size_t off_loss = take((2 * kMaxRanks) * sizeof(float) + kMaxRanks * sizeof(uint32_t));
  CU(cudaMalloc(&s->sym, total));
  CU(cudaMemset(s->sym, 0, total));
  CU(cudaMalloc(&s->p2p_done, 2 * s->L * sizeof(int)));
  CU(cudaMemset(s->p2p_done, 0, 2 * s->L * sizeof(int)));
  std::vector<void*> all;
  ST(comm_share_ptrs(s, &s->sym, 1, &all, &s->ipc_opened));
  for (int j = 0; j < N; ++j) {
    s->peer_sym[j] = all[j];
    float* ls = reinterpret_cast<float*>(static_cast<char*>(all[j]) + off_loss);
    s->loss_peers.slots[j] = ls;
    s->loss_peers.flags[j] = reinterpret_cast<uint32_t*>(ls + 2 * kMaxRanks);
  }
  if (cudaStreamCreateWithFlags(&s->loss_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(DFLOW_CUDA, "stream creation failed");
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    for (int j = 0; j < N; ++j) {
      char* b = static_cast<char*>(s->peer_sym[j]);
      ly.p2p.recv[j] = reinterpret_cast<uint16_t*>(b + off_recv[l]);
      ly.p2p.gath[j] = reinterpret_cast<uint16_t*>(b + off_gath[l]);
      ly.p2p.flags[j] = reinterpret_cast<uint32_t*>(b + off_flags[l]);
    }
    ly.p2p.done = s->p2p_done + 2 * l;
    ly.p2p.shard = ly.shard;
    ly.p2p.rank = R;
    ly.p2p.world = N;
    ly.p2p.abort = s->abort_dev;
    ly.p2p.timeout_ns = s->flag_timeout_ns;
  }
  if (s->tf32) return DFLOW_OK;
  ST(setup_multicast(s));
  // owner-apply: every rank maps every peer's W32, b32 and (without
  // multicast) bf16 W copy
  const int per = s->multicast ? 2 * s->L : 3 * s->L;  // allocations per rank
  const int k = s->multicast ? 2 : 3;
  std::vector<void*> mine(per);
  for (int l = 0; l < s->L; ++l) {
    mine[k * l] = s->layers[l].W32;
    mine[k * l + 1] = s->layers[l].b32;
    if (!s->multicast) mine[k * l + 2] = s->layers[l].Wop.hi;
  }
  std::vector<void*> allp;
  ST(comm_share_ptrs(s, mine.data(), per, &allp, &s->ipc_opened));
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    for (int j = 0; j < N; ++j) {
      ly.p2p.w32[j] = static_cast<float*>(allp[j * per + k * l]);
      ly.p2p.b32[j] = static_cast<float*>(allp[j * per + k * l + 1]);
      ly.p2p.wop[j] = s->multicast ? nullptr : static_cast<uint16_t*>(allp[j * per + k * l + 2]);
    }
    ly.p2p.owner_apply = 1;
    ly.p2p.in = ly.in;
    ly.p2p.out = ly.out;
    ly.p2p.ldwb = ly.ld_wb;
    ly.p2p.lr_w = ly.n.lr_W;
    ly.p2p.lr_b = ly.n.lr_b;
  }
  return DFLOW_OK;
}

// f1 multicast gather (bf16 owner-apply over NCCL): move every layer's bf16 W copy into one
// symmetric NCCL window and store through its multicast address, so an owner writes each new
// weight once and the NVSwitch delivers it to all N copies (instead of N unicast NVLink
// stores).  All ranks agree (all-reduce of the outcome) or all keep unicast.
// DFLOW_P2P_MULTICAST=0 disables it.
dflow_status setup_multicast(dflow_session* s) {
  if (s->sim || !s->nccl) return DFLOW_OK;
  if (const char* e = getenv("DFLOW_P2P_MULTICAST"))
    if (atoi(e) == 0) return DFLOW_OK;
  size_t total = 0;
  std::vector<size_t> off(s->L);
  bool shapes_ok = true;
  for (int l = 0; l < s->L; ++l) {
    off[l] = total;
    total += (s->layers[l].in * s->layers[l].ld_wb * 2 + 4095) / 4096 * 4096;
    shapes_ok &= (s->layers[l].out % 8) == 0 && s->layers[l].ld_wb == s->layers[l].out;  // 16-byte rows
  }
  if (!shapes_ok) return DFLOW_OK;  // (the same decision on every rank: shapes are global)
  void *base = nullptr, *mc = nullptr;
  SymRegion* r = nullptr;
  const dflow_status st = comm_symmetric_alloc(s, total, &base, &mc, &r);
  // every rank must take the same path: all-reduce "this rank has a multicast address"
  float* flag = nullptr;
  CU(cudaMalloc(&flag, sizeof(float)));
  const float one = (st == DFLOW_OK && mc) ? 1.f : 0.f;
  CU(cudaMemcpyAsync(flag, &one, sizeof(float), cudaMemcpyHostToDevice, s->comm));
  ST(comm_allreduce_f32(s, flag, flag, 1, s->comm));
  float all = 0.f;
  CU(cudaMemcpyAsync(&all, flag, sizeof(float), cudaMemcpyDeviceToHost, s->comm));
  CU(cudaStreamSynchronize(s->comm));
  cudaFree(flag);
  if (all != static_cast<float>(s->opt.world)) {
    if (r) comm_symmetric_free(s, r);
    clear_error();
    return DFLOW_OK;  // unicast pushes
  }
  s->wsym = r;
  s->multicast = true;
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    cudaFree(ly.Wop.hi);
    ly.Wop.hi = static_cast<char*>(base) + off[l];
    ly.p2p.mc_wop = reinterpret_cast<uint16_t*>(static_cast<char*>(mc) + off[l]);
  }
  return DFLOW_OK;
}

// Asynchronous replicas (f3): every rank allocates its fp32 shard of every layer bucket in
// one symmetric allocation and maps every peer's through CUDA IPC (the same pointer
// exchange as setup_p2p).  Shards start zeroed; dflow_variable_assign publishes them.
dflow_status setup_async(dflow_session* s) {
  const int N = s->opt.world, R = s->opt.rank;
  std::vector<size_t> off(s->L);
  size_t total = 0;
  for (int l = 0; l < s->L; ++l) {
    off[l] = total;
    total += (s->layers[l].shard * sizeof(float) + 255) / 256 * 256;
  }
  CU(cudaMalloc(&s->sym, total));
  CU(cudaMemset(s->sym, 0, total));
  std::vector<void*> all;
  ST(comm_share_ptrs(s, &s->sym, 1, &all, &s->ipc_opened));
  for (int j = 0; j < N; ++j) s->peer_sym[j] = all[j];
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    for (int j = 0; j < N; ++j) ly.async.master[j] = reinterpret_cast<float*>(static_cast<char*>(s->peer_sym[j]) + off[l]);
    ly.async.shard = ly.shard;
    ly.async.in = ly.in;
    ly.async.out = ly.out;
    ly.async.rank = R;
    ly.async.world = N;
  }
  return DFLOW_OK;
}

// The train step's pull (async_dp = 1): layer l's shards are pulled on a side stream while
// the forward of the earlier layers runs; the forward of layer l waits for its own pull
// (ev_apply[l], joined like a deferred update).  The fp32 W copy is not refreshed here
// (dflow_variable_read pulls it).
dflow_status async_pull_pipelined(dflow_session* s, cudaStream_t st) {
  CU(cudaEventRecord(s->ev_side_join[0], st));  // the previous step is done with the operands
  CU(cudaStreamWaitEvent(s->side[0], s->ev_side_join[0], 0));
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    const int t = tbegin(s, 1, s->side[0]);
    cudaError_t e = launch_async_pull(ly.async, nullptr, ly.b32, static_cast<__nv_bfloat16*>(ly.Wop.hi), ly.ld_wb,
                                      s->side[0]);
    tend(s, t, s->side[0]);
    ST(check_launch(s, e, 1, "parameter pull"));
    CU(cudaEventRecord(s->ev_apply[l], s->side[0]));
  }
  s->apply_pending = true;
  return DFLOW_OK;
}

dflow_status async_pull(dflow_session* s, cudaStream_t st) {
  for (Layer& ly : s->layers) {
    const int t = tbegin(s, 1, st);
    cudaError_t e = launch_async_pull(ly.async, ly.W32, ly.b32, static_cast<__nv_bfloat16*>(ly.Wop.hi), ly.ld_wb, st);
    tend(s, t, st);
    ST(check_launch(s, e, 1, "parameter pull"));
  }
  return DFLOW_OK;
}

// loss partials the last forward GEMM's epilogue writes: one per (tile, CTA, epilogue warp)
inline int loss_slots(const GemmPlan& p) { return p.tiles_m * p.tiles_n * p.cluster * 4; }

dflow_status gemm_plan(dflow_session* s, const GemmDesc& d, GemmPlan* p) {
  cudaError_t e = gemm_prepare(d, s->num_sms, p);
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "GEMM plan: %s", gemm_last_error());
  return DFLOW_OK;
}

dflow_status plan_rows(dflow_session* s, int64_t rows) {
  if (rows == s->planned_rows) return DFLOW_OK;
  const int max_ctas = (s->replicas > 1 && s->opt.overlap && s->opt.sm_reserve > 0)
                           ? std::max(2, s->num_sms - s->opt.sm_reserve)
                           : 0;
  const bool tf = s->tf32;
  for (int l = 0; l < s->L; ++l) {
    Layer& ly = s->layers[l];
    const bool last = (l + 1 == s->L);
    const Operand& Aprev = (l == 0) ? s->A0 : s->layers[l - 1].A;
    const int64_t ld_prev = (l == 0) ? s->ld_A0 : s->layers[l - 1].ld_out;
    GemmDesc f{};
    f.tf32 = tf;
    f.M = rows; f.N = ly.out; f.K = ly.in;
    f.A = Aprev.hi; f.A2 = Aprev.lo; f.lda = ld_prev; f.a_mn = false;
    f.B = ly.Wop.hi; f.B2 = ly.Wop.lo; f.ldb = ly.ld_wb; f.b_mn = true;
    f.bias = ly.b32;
    f.max_ctas = max_ctas;
    f.group = raster_group("DFLOW_GEMM_GROUP_FWD", kGroupFwd);
    f.sched = s->sched_fd;  // this session's own counters (never another session's stream)
    if (!last) {
      f.epilogue = EPI_BIAS_RELU;
      f.out = ly.A.hi; f.out2 = ly.A.lo; f.ldo = ly.ld_out;
      ST(gemm_plan(s, f, &ly.fwd));
      if (s->mp && l + 1 == s->mp_hi) {  // f4: this activation crosses to rank+1 as its channel code
        GemmDesc fs = f;
        fs.trunc_out = 1;
        ST(gemm_plan(s, fs, &ly.fwd_send));
      }
    } else {
      // last layer: Relu + loss seed + db partials fused (a1 + a2 + a5); y is patched per call
      f.epilogue = EPI_BIAS_RELU_LOSS;
      f.out = ly.dZ.hi; f.out2 = ly.dZ.lo; f.ldo = ly.ld_out;
      f.loss_kind = s->loss_kind == DFLOW_LOSS_MSE ? 0 : 1;
      f.y = s->AL32; f.ldy = s->ld_AL32;  // placeholder pointer, replaced at launch
      f.loss_partials = s->loss_partials;
      f.colsum_ws = ly.colsum_ws;
      ST(gemm_plan(s, f, &ly.fwd));
      f.out_f32 = s->AL32; f.ldo32 = s->ld_AL32;  // fetch variant also keeps fp32 A_L
      ST(gemm_plan(s, f, &ly.fwd_fetch));
      GemmDesc p = f;  // forward-only without a target: plain Relu, fp32 A_L
      p.epilogue = EPI_BIAS_RELU;
      p.out = nullptr;
      p.out2 = nullptr;
      p.y = nullptr; p.loss_partials = nullptr; p.colsum_ws = nullptr;
      ST(gemm_plan(s, p, &ly.fwd_plain));
    }
    ly.has_fwd = true;
    if (l > 0) {
      const Layer& lp = s->layers[l - 1];
      GemmDesc d{};
      d.tf32 = tf;
      d.M = rows; d.N = ly.in; d.K = ly.out;
      d.A = ly.dZ.hi; d.A2 = ly.dZ.lo; d.lda = ly.ld_out; d.a_mn = false;
      d.B = ly.Wop.hi; d.B2 = ly.Wop.lo; d.ldb = ly.ld_wb; d.b_mn = false;
      d.epilogue = EPI_RELUGRAD;
      d.out = lp.dZ.hi; d.out2 = lp.dZ.lo; d.ldo = lp.ld_out;
      d.mask = lp.A.hi; d.ldm = lp.ld_out;
      d.colsum_ws = lp.colsum_ws;  // db_{l-1} partials fused (a5)
      d.max_ctas = max_ctas;
      d.group = raster_group("DFLOW_GEMM_GROUP_DGRAD", kGroupDgrad);
      d.sched = s->sched_fd + 4;
      ST(gemm_plan(s, d, &ly.dgrad));
      ly.has_dgrad = true;
      if (s->mp && l == s->mp_lo) {  // f4: dA_{l-1} crosses back to rank-1 as channel codes (no mask here)
        GemmDesc ds = d;
        ds.epilogue = EPI_TRUNC16;
        ds.mask = nullptr; ds.ldm = 0; ds.colsum_ws = nullptr;
        ds.out = lp.dZ.hi; ds.out2 = nullptr; ds.ldo = lp.ld_out;
        ST(gemm_plan(s, ds, &ly.dgrad_send));
      }
    }
    GemmDesc w{};
    w.tf32 = tf;
    w.M = ly.in; w.N = ly.out; w.K = rows;
    w.A = Aprev.hi; w.A2 = Aprev.lo; w.lda = ld_prev; w.a_mn = true;
    w.B = ly.dZ.hi; w.B2 = ly.dZ.lo; w.ldb = ly.ld_out; w.b_mn = true;
    w.epilogue = EPI_F32;
    w.out_f32 = ly.g32; w.ldo32 = ly.out;
    w.max_ctas = max_ctas;
    w.group = raster_group("DFLOW_GEMM_GROUP_WGRAD", kGroupWgrad);
    w.sched = s->sched_w + 4 * (l % 2);  // (bwd_side: dW_l runs on side[l % 2])
    ST(gemm_plan(s, w, &ly.wgrad32));
    if (s->replicas == 1 && s->trainable) {
      // no channel (reading A6): ApplyGradientDescent fused into the dW epilogue
      GemmDesc wa = w;
      wa.epilogue = EPI_SGD_APPLY;
      wa.out_f32 = ly.W32; wa.ldo32 = ly.out;
      wa.out = ly.Wop.hi; wa.out2 = ly.Wop.lo; wa.ldo = ly.ld_wb;
      wa.sgd_lr = ly.n.lr_W;
      ST(gemm_plan(s, wa, &ly.wgrad_apply));
      ly.has_wgrad_apply = true;
    }
    if (s->async) {
      // f3: the dW epilogue pushes -lr * g_hat into the owners' shards
      GemmDesc wa = w;
      wa.epilogue = EPI_ASYNC_PUSH;
      wa.out_f32 = nullptr;
      wa.async_master = ly.async.master;
      wa.async_coded = u16_wire(s) ? 1 : 0;
      wa.p2p_bulk = 1;  // bulk fp32 add-reductions through the TMA engine
      wa.p2p_shard = ly.shard;
      wa.p2p_rank = s->opt.rank;
      wa.p2p_world = s->opt.world;
      wa.sgd_lr = ly.n.lr_W;
      ST(gemm_plan(s, wa, &ly.wgrad_async));
    }
    if (s->replicas > 1 && u16_wire(s) && !s->p2p && !s->async) {
      w.epilogue = EPI_TRUNC16;
      w.out_f32 = nullptr;
      w.out = ly.q16; w.out2 = nullptr; w.ldo = ly.out;
      ST(gemm_plan(s, w, &ly.wgrad16));
      ly.has_wgrad16 = true;
    }
    if (s->p2p) {
      // dW tiles truncated and stored straight into the owners' receive slots (f1)
      w.epilogue = EPI_TRUNC16_P2P;
      w.out_f32 = nullptr;
      w.out = nullptr; w.out2 = nullptr;
      w.p2p_recv = ly.p2p.recv;
      w.p2p_shard = ly.p2p.shard;
      w.p2p_rank = s->opt.rank;
      w.p2p_world = s->opt.world;
      w.p2p_bulk = 1;
      ST(gemm_plan(s, w, &ly.wgrad_p2p));
      ly.has_wgrad_p2p = true;
    }
  }
  // N = 1: can the dW GEMMs run beside the dgrads (and each other) without queueing for SMs?
  int wsum = 0, dmax = 0;
  for (int l = 0; l < s->L; ++l) {
    const Layer& ly = s->layers[l];
    wsum += ly.has_wgrad_apply ? ly.wgrad_apply.grid : ly.wgrad32.grid;
    if (ly.has_dgrad) dmax = std::max(dmax, ly.dgrad.grid);
  }
  s->bwd_side = s->replicas == 1 && !s->mp && s->L > 1 && wsum + dmax <= s->num_sms;
  // A/B knob (DFLOW_BWD_SIDE = 0 / 1): force the side-stream dW schedule off / on (on large
  // layers the persistent dW GEMM then only fills the SMs the dgrad's last wave leaves idle)
  if (const char* e = getenv("DFLOW_BWD_SIDE"))
    s->bwd_side = atoi(e) != 0 && s->replicas == 1 && !s->mp && s->L > 1;
  s->planned_rows = rows;
  return DFLOW_OK;
}

// ------------------------------------------------------------------ timing
int tbegin(dflow_session* s, int kind, cudaStream_t st) {
  if (!s->timing) return -1;
  if (s->event_next + 2 > s->event_pool.size()) {
    for (int i = 0; i < 64; ++i) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      s->event_pool.push_back(e);
    }
  }
  TimedRange r{kind, s->event_pool[s->event_next], s->event_pool[s->event_next + 1], st == s->comm ? 1 : 0,
               nullptr};
  s->event_next += 2;
  cudaEventRecord(r.a, st);
  s->ranges.push_back(r);
  return static_cast<int>(s->ranges.size()) - 1;
}

void tend(dflow_session* s, int idx, cudaStream_t st) {
  if (idx >= 0) cudaEventRecord(s->ranges[idx].b, st);
}

dflow_status launch_gemm(dflow_session* s, const GemmPlan& p, cudaStream_t st) {
  const int t = tbegin(s, 0, st);
  static const char* kEpi[] = {"F32", "TRUNC16", "BIAS_RELU", "RELUGRAD", "BIAS_RELU_LOSS", "SGD_APPLY",
                               "TRUNC16_P2P", "ASYNC_PUSH"};
  if (t >= 0 && p.d.epilogue >= 0 && p.d.epilogue < 8) s->ranges[t].label = kEpi[p.d.epilogue];
  cudaError_t e = gemm_launch(p, st);
  tend(s, t, st);
  if (e != cudaSuccess) {
    s->poisoned = true;
    return fail(DFLOW_CUDA, "%s", gemm_last_error());
  }
  s->launches++;
  s->gemm_launches++;
  return DFLOW_OK;
}

dflow_status check_launch(dflow_session* s, cudaError_t e, int count, const char* what) {
  if (e != cudaSuccess) {
    s->poisoned = true;
    return fail(DFLOW_CUDA, "%s launch failed: %s", what, cudaGetErrorString(e));
  }
  s->launches += count;
  return DFLOW_OK;
}

// ------------------------------------------------------------------ feeds
struct Feeds {
  const void* x = nullptr;
  int64_t ldx = 0;
  const float* y = nullptr;
  int64_t ldy = 0;
};

dflow_status resolve_feeds(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* ptrs,
                           const int64_t* ld, Feeds* f) {
  if (n_feeds < 0 || (n_feeds > 0 && (!feeds || !ptrs || !ld))) return fail(DFLOW_INVALID_ARGUMENT, "bad feed arrays");
  for (int i = 0; i < n_feeds; ++i) {
    if (feeds[i] < 0 || feeds[i] >= static_cast<int>(s->remap.size()))
      return fail(DFLOW_INVALID_ARGUMENT, "feed %d is not a node of the session's graph", i);
    const int sid = s->remap[feeds[i]];
    if (sid == s->x) {
      f->x = ptrs[i];
      f->ldx = ld[i];
    } else if (sid == s->y && s->y >= 0) {
      f->y = static_cast<const float*>(ptrs[i]);
      f->ldy = ld[i];
    } else {
      return fail(DFLOW_INVALID_ARGUMENT, "feed '%s' is not the x or y placeholder", s->g.nodes[sid].name.c_str());
    }
  }
  return DFLOW_OK;
}

// Every entry point: a CUDA/NCCL error, a failed step or a timed-out cross-GPU flag wait
// (the abort word a wait kernel wrote) poisons the session (abort and
// restart from the last checkpoint, which here is the caller's).
dflow_status check_alive(dflow_session* s) {
  if (s->abort_host && *static_cast<volatile uint32_t*>(s->abort_host) != 0 && !s->poisoned) {
    s->poisoned = true;
    return fail(DFLOW_SESSION_POISONED,
                "a cross-GPU flag wait timed out (a peer rank died or fell out of step); session poisoned");
  }
  if (s->poisoned) return fail(DFLOW_SESSION_POISONED, "session poisoned by an earlier CUDA/NCCL error or timeout");
  return DFLOW_OK;
}

dflow_status check_rows(dflow_session* s, int64_t rows) {
  ST(check_alive(s));
  if (rows <= 0 || rows > s->cap)
    return fail(DFLOW_INVALID_ARGUMENT, "local_rows %lld outside 1..max_local_rows=%lld", (long long)rows,
                (long long)s->cap);
  if (cudaSetDevice(s->opt.device) != cudaSuccess) return fail(DFLOW_CUDA, "cudaSetDevice failed");
  return plan_rows(s, rows);
}

// ------------------------------------------------------------------ phases
enum FwdMode { FWD_TRAIN = 0, FWD_FETCH = 1, FWD_ONLY = 2 };

dflow_status run_forward(dflow_session* s, const Feeds& f, int64_t rows, cudaStream_t st, int mode) {
  if (!f.x) return fail(DFLOW_INVALID_ARGUMENT, "x must be fed");
  const int64_t in = s->layers[0].in;
  if (f.ldx < in) return fail(DFLOW_INVALID_ARGUMENT, "ld of x < its width");
  int t = tbegin(s, 1, st);
  cudaError_t e = (s->x_dtype == DFLOW_F32)
                      ? to_operand(s, static_cast<const float*>(f.x), f.ldx, s->A0, s->ld_A0, rows, in, st)
                      : launch_copy_bf16(static_cast<const __nv_bfloat16*>(f.x), f.ldx,
                                         static_cast<__nv_bfloat16*>(s->A0.hi), s->ld_A0, rows, in, st);
  tend(s, t, st);
  ST(check_launch(s, e, 1, "input cast"));
  CU(record_event(s, s->ev_x_free, st));  // (a host-fed pipelined step may upload the next x now)
  // defer_apply: layer l's update of the previous step may still be in flight on the
  // exchange stream; each GEMM waits for exactly the parameters it reads
  const bool pending = s->apply_pending;
  s->apply_pending = false;
  for (int l = 0; l + 1 < s->L; ++l) {
    if (pending) CU(cudaStreamWaitEvent(st, s->ev_apply[l], 0));
    ST(launch_gemm(s, s->layers[l].fwd, st));
  }
  if (pending) CU(cudaStreamWaitEvent(st, s->ev_apply[s->L - 1], 0));
  // last layer: Relu + loss seed (+ db_L partials) fused into the GEMM epilogue (a1+a2+a5)
  Layer& last = s->layers[s->L - 1];
  const bool need_y = s->loss_kind == DFLOW_LOSS_MSE;
  if (mode == FWD_ONLY && need_y && !f.y) {
    ST(launch_gemm(s, last.fwd_plain, st));  // forward fetch without a target: no loss
  } else {
    if (need_y && !f.y) return fail(DFLOW_INVALID_ARGUMENT, "y must be fed (MSE loss)");
    if (need_y && f.ldy < last.out) return fail(DFLOW_INVALID_ARGUMENT, "ld of y < its width");
    GemmPlan& p = (mode == FWD_TRAIN) ? last.fwd : last.fwd_fetch;
    p.args.y = f.y;
    p.args.ldy = f.ldy;
    if (s->y_upload_pending) {  // host-fed y still uploading under layers 1..L-1
      // (inside a step-graph capture this becomes an external event-wait node)
      CU(cudaStreamWaitEvent(st, s->ev_h2d_y, s->capturing ? cudaEventWaitExternal : 0));
      s->y_upload_pending = false;
    }
    ST(launch_gemm(s, p, st));
    const int t = tbegin(s, 1, st);
    cudaError_t e2 = launch_loss_final(s->loss_kind == DFLOW_LOSS_MSE ? 0 : 1, s->loss_partials, loss_slots(p), rows,
                                       last.out, s->loss_dev, st);
    tend(s, t, st);
    ST(check_launch(s, e2, 1, "loss reduction"));
  }
  s->have_forward = true;
  s->last_rows = rows;
  return DFLOW_OK;
}

// Exchange + apply of layer l (comm stream when N > 1).
// joined: the exchange stream already waits for this layer's gradient (ev_grad[l]).
dflow_status exchange_apply(dflow_session* s, int l, cudaStream_t st, bool joined) {
  Layer& ly = s->layers[l];
  const int N = s->replicas;
  const int64_t nW = ly.in * ly.out;
  cudaStream_t cs = st;
  const uint16_t* g16 = nullptr;
  const float* g32 = ly.g32;
  if (N > 1) {
    cs = s->comm;
    if (!joined) {
      CU(cudaEventRecord(s->ev_grad[l], st));
      CU(cudaStreamWaitEvent(cs, s->ev_grad[l], 0));
    }
    const int t = tbegin(s, 2, cs);
    const Round16 own_code = round16_of(s, l, 1);  // the owner's coding of the mean (a8)
    switch (s->opt.exchange) {
      case DFLOW_EXCHANGE_TRUNC16:
      case DFLOW_EXCHANGE_SR16: {
        if (s->p2p) {
          // fused NVLink path: contributions already sit in our receive slots (pushed by the
          // peers' dW epilogues); fold, push q_bar to every rank, wait for every owner
          // (simulated world: every rank's contributions are enqueued before any owner folds,
          // and every owner's fold before any rank waits for the gather — comm.h)
          ST(comm_rendezvous(s));
          ST(check_launch(s, launch_owner_reduce_p2p(ly.p2p, s->epoch, cs, own_code), 1, "owner reduce (p2p)"));
          ST(comm_rendezvous(s));
          ST(check_launch(s, launch_wait_flags(ly.p2p.flags[s->opt.rank] + kMaxRanks, N, s->epoch, s->abort_dev,
                                               s->flag_timeout_ns, cs),
                          1, "gather wait (p2p)"));
          if (ly.p2p.owner_apply) {  // the owners already updated W, b here (a9 on the owner)
            tend(s, t, cs);
            CU(cudaEventRecord(s->ev_apply[l], cs));
            return DFLOW_OK;
          }
          g16 = ly.p2p.gath[s->opt.rank];
          g32 = nullptr;
          break;
        }
        ST(comm_alltoall(s, ly.q16, ly.recv, ly.shard * 2, cs));
        ST(check_launch(s, launch_owner_reduce_t16(static_cast<uint16_t*>(ly.recv), ly.shard, N,
                                                   static_cast<uint16_t*>(ly.own), cs, own_code,
                                                   static_cast<int64_t>(s->opt.rank) * ly.shard),
                        1, "owner reduce"));
        ST(comm_allgather(s, ly.own, ly.gath, ly.shard * 2, cs));
        g16 = static_cast<const uint16_t*>(ly.gath);
        g32 = nullptr;
        break;
      }
      case DFLOW_EXCHANGE_FP32: {
        ST(comm_alltoall(s, ly.g32, ly.recv, ly.shard * 4, cs));
        ST(check_launch(s, launch_owner_reduce_f32(static_cast<float*>(ly.recv), ly.shard, N,
                                                   static_cast<float*>(ly.own), cs), 1, "owner reduce"));
        ST(comm_allgather(s, ly.own, ly.gath, ly.shard * 4, cs));
        g32 = static_cast<const float*>(ly.gath);
        break;
      }
      case DFLOW_EXCHANGE_FP32_NCCL: {
        ST(comm_allreduce_f32(s, ly.g32, ly.g32, ly.P, cs));
        ST(check_launch(s, launch_scale_f32(ly.g32, ly.P, 1.0f / static_cast<float>(N), cs), 1, "scale"));
        break;
      }
      default:
        break;  // NONE: local gradient (timing only)
    }
    tend(s, t, cs);
  }
  const int t = tbegin(s, 1, cs);
  const bool w_done = (N == 1 && ly.has_wgrad_apply);  // W already updated by the dW epilogue
  cudaError_t e = cudaSuccess;
  if (!w_done)
    e = s->tf32 ? launch_apply_sgd_tf32(ly.W32, g32, g16, ly.in, ly.out, static_cast<float*>(ly.Wop.hi),
                                        static_cast<float*>(ly.Wop.lo), ly.ld_wb, ly.n.lr_W, cs)
                : launch_apply_sgd(ly.W32, g32, g16, ly.in, ly.out, static_cast<__nv_bfloat16*>(ly.Wop.hi),
                                   ly.ld_wb, ly.n.lr_W, cs);
  if (e == cudaSuccess)
    e = launch_apply_sgd(ly.b32, g32 ? g32 + nW : nullptr, g16 ? g16 + nW : nullptr, 1, ly.out, nullptr, 0,
                         ly.n.lr_b, cs);
  tend(s, t, cs);
  ST(check_launch(s, e, w_done ? 1 : 2, "apply"));
  if (N > 1) CU(cudaEventRecord(s->ev_apply[l], cs));
  return DFLOW_OK;
}

// mode 0: train (TRUNC16 buckets + exchange + apply); 1: fetch (fp32 grads, no exchange)
dflow_status run_backward(dflow_session* s, int64_t rows, cudaStream_t st, int mode) {
  if (mode == 0 && s->async) {  // f3: push every layer's update into the owners' shards, no exchange
    for (int l = s->L - 1; l >= 0; --l) {
      Layer& ly = s->layers[l];
      if (l > 0) ST(launch_gemm(s, ly.dgrad, st));
      const Round16 code = round16_of(s, l, 0);
      ly.wgrad_async.args.r16 = code;
      ST(launch_gemm(s, ly.wgrad_async, st));
      const int t = tbegin(s, 1, st);
      cudaError_t e = launch_colsum_push(ly.colsum_ws, static_cast<int>((rows + 31) / 32), ly.async, ly.n.lr_b,
                                         u16_wire(s) ? 1 : 0, code, st);
      tend(s, t, st);
      ST(check_launch(s, e, 1, "bias-gradient push"));
    }
    return DFLOW_OK;
  }
  const bool t16 = mode == 0 && s->replicas > 1 && u16_wire(s);
  // defer_apply: the order L..1 with the last two dW swapped — ..., dgrad(2), dW_1, dW_2 —
  // so layer 1's exchange runs under dW_2 and layer 2's (the last) under the next step's
  // forward of layer 1; the step does not join the exchange stream.  dgrad(l) still reads
  // W_l before this rank's dW_l contribution can let an owner overwrite it.  (Running every
  // dgrad first and the dW in order 1..L hides the same tail but puts each exchange under a
  // dW GEMM's own NVLink stores: measured slower at N = 4.)
  const bool defer = mode == 0 && s->defer && s->L >= 2;
  for (int i = 0; i < s->L; ++i) {
    int l = s->L - 1 - i;
    if (defer && l <= 1) l = 1 - l;  // positions L-2, L-1 run layers 0, 1 (0-based)
    Layer& ly = s->layers[l];
    if (!defer || l >= 2) {
      if (l > 0) ST(launch_gemm(s, ly.dgrad, st));
    } else if (l == 0) {
      ST(launch_gemm(s, s->layers[1].dgrad, st));  // dZ_1 for dW_1 (layer 1's dgrad, 0-based)
    }
    const bool p2p = t16 && s->p2p;
    const Round16 send_code = round16_of(s, l, 0);  // this rank's coding of its gradient (a6)
    GemmPlan& wp = p2p ? ly.wgrad_p2p
                       : t16 ? ly.wgrad16 : (mode == 0 && ly.has_wgrad_apply ? ly.wgrad_apply : ly.wgrad32);
    wp.args.r16 = send_code;
    // small N = 1 steps: dW_l (+ its update) and db_l beside dgrad(l-1) on the side stream
    // (dgrad(l), which reads W_l, is already enqueued before the fork)
    const bool side = mode == 0 && s->bwd_side;
    cudaStream_t wst = st;
    if (side) {
      CU(cudaEventRecord(s->ev_grad[l], st));
      CU(cudaStreamWaitEvent(s->side[l % 2], s->ev_grad[l], 0));
      wst = s->side[l % 2];
    }
    // (fault injection of the simulated world: a "dead" rank sends no contributions)
    const bool dropped = p2p && comm_dropped(s);
    if (!dropped) ST(launch_gemm(s, wp, wst));
    // db_l: the producing epilogue left per-32-row column partials; sum them in order.
    // N > 1: on the exchange stream, under the next dgrad (it only feeds the exchange)
    const bool on_comm = mode == 0 && s->replicas > 1;
    cudaStream_t cst = wst;
    if (on_comm) {
      CU(cudaEventRecord(s->ev_grad[l], st));
      CU(cudaStreamWaitEvent(s->comm, s->ev_grad[l], 0));
      cst = s->comm;
    }
    const int t = tbegin(s, 1, cst);
    const int chunks = static_cast<int>((rows + 31) / 32);
    // N = 1: W was updated by the dW epilogue; the b_l update rides on this pass too
    const bool fused_b = mode == 0 && s->replicas == 1 && ly.has_wgrad_apply;
    cudaError_t e = dropped ? cudaSuccess
                  : p2p ? launch_colsum_final_p2p(ly.colsum_ws, chunks, ly.out, ly.in * ly.out, ly.p2p, s->epoch, cst,
                                                  send_code)
                        : launch_colsum_final(ly.colsum_ws, chunks, ly.out,
                                              (t16 || fused_b) ? nullptr : ly.g32 + ly.in * ly.out,
                                              t16 ? ly.q16 + ly.in * ly.out : nullptr, cst, send_code,
                                              ly.in * ly.out, fused_b ? ly.b32 : nullptr, ly.n.lr_b);
    tend(s, t, cst);
    ST(check_launch(s, e, 1, "bias-gradient column sum"));
    if (mode == 0 && !fused_b) ST(exchange_apply(s, l, st, on_comm));
  }
  if (mode == 0 && s->bwd_side) {  // join the side streams (the updates) back into st
    for (int i = 0; i < 2; ++i) {
      CU(cudaEventRecord(s->ev_side_join[i], s->side[i]));
      CU(cudaStreamWaitEvent(st, s->ev_side_join[i], 0));
    }
  }
  if (defer) s->apply_pending = true;  // joined per layer by the next forward
  else if (mode == 0 && s->replicas > 1) CU(cudaStreamWaitEvent(st, s->ev_apply[0], 0));
  return DFLOW_OK;
}

// Orders st after every pending update (defer_apply).
dflow_status join_apply(dflow_session* s, cudaStream_t st) {
  if (!s->apply_pending) return DFLOW_OK;
  for (int l = 0; l < s->L; ++l) CU(cudaStreamWaitEvent(st, s->ev_apply[l], 0));
  s->apply_pending = false;
  return DFLOW_OK;
}

// ---------------------------------------------------------------- f4 model parallelism
// Rank r runs layers [mp_lo, mp_hi) of one replica.  Channels (readings A32-A33) on `st`:
// forward, the activation of layer mp_hi-1 (as truncation codes) to rank r+1; backward,
// dA of layer mp_lo (codes) to rank r-1.  NCCL point-to-point moves the bytes.
dflow_status run_forward_mp(dflow_session* s, const Feeds& f, int64_t rows, cudaStream_t st) {
  const int R = s->opt.rank, N = s->opt.world, lo = s->mp_lo, hi = s->mp_hi;
  if (lo == 0) {
    if (!f.x) return fail(DFLOW_INVALID_ARGUMENT, "x must be fed");
    const int t = tbegin(s, 1, st);
    cudaError_t e = (s->x_dtype == DFLOW_F32)
                        ? to_operand(s, static_cast<const float*>(f.x), f.ldx, s->A0, s->ld_A0, rows, s->layers[0].in, st)
                        : launch_copy_bf16(static_cast<const __nv_bfloat16*>(f.x), f.ldx,
                                           static_cast<__nv_bfloat16*>(s->A0.hi), s->ld_A0, rows, s->layers[0].in, st);
    tend(s, t, st);
    ST(check_launch(s, e, 1, "input cast"));
  } else {
    const Layer& lp = s->layers[lo - 1];  // the received codes are the bf16 operand bits
    ST(comm_recv(s, lp.A.hi, static_cast<size_t>(rows * lp.ld_out) * 2, R - 1, st));
  }
  for (int l = lo; l < hi; ++l) {
    Layer& ly = s->layers[l];
    if (l + 1 < s->L) {
      ST(launch_gemm(s, (l + 1 == hi) ? ly.fwd_send : ly.fwd, st));
      continue;
    }
    // last layer (last rank): Relu + loss seed + db partials
    const bool need_y = s->loss_kind == DFLOW_LOSS_MSE;
    if (need_y && !f.y) return fail(DFLOW_INVALID_ARGUMENT, "y must be fed (MSE loss)");
    if (need_y && f.ldy < ly.out) return fail(DFLOW_INVALID_ARGUMENT, "ld of y < its width");
    ly.fwd.args.y = f.y;
    ly.fwd.args.ldy = f.ldy;
    if (s->y_upload_pending) {  // host-fed y
      CU(cudaStreamWaitEvent(st, s->ev_h2d_y, 0));
      s->y_upload_pending = false;
    }
    ST(launch_gemm(s, ly.fwd, st));
    const int t = tbegin(s, 1, st);
    cudaError_t e = launch_loss_final(need_y ? 0 : 1, s->loss_partials, loss_slots(ly.fwd), rows, ly.out, s->loss_dev, st);
    tend(s, t, st);
    ST(check_launch(s, e, 1, "loss reduction"));
  }
  if (R + 1 < N) {
    const Layer& ll = s->layers[hi - 1];
    ST(comm_send(s, ll.A.hi, static_cast<size_t>(rows * ll.ld_out) * 2, R + 1, st));
  }
  s->have_forward = true;
  s->last_rows = rows;
  return DFLOW_OK;
}

dflow_status run_backward_mp(dflow_session* s, int64_t rows, cudaStream_t st) {
  const int R = s->opt.rank, N = s->opt.world, lo = s->mp_lo, hi = s->mp_hi;
  for (int l = hi - 1; l >= lo; --l) {
    Layer& ly = s->layers[l];
    if (l == hi - 1 && R + 1 < N) {
      // the received dA codes, masked by this rank's own activation (ReluGrad on the
      // channel's output) -> dZ and its per-32-row column partials
      ST(comm_recv(s, s->mp_recv, static_cast<size_t>(rows * ly.ld_out) * 2, R + 1, st));
      const int t = tbegin(s, 1, st);
      cudaError_t e = launch_relugrad_recv(s->mp_recv, ly.ld_out, static_cast<const __nv_bfloat16*>(ly.A.hi), ly.ld_out,
                                           rows, ly.out, static_cast<__nv_bfloat16*>(ly.dZ.hi), ly.ld_out,
                                           ly.colsum_ws, st);
      tend(s, t, st);
      ST(check_launch(s, e, 1, "channel ReluGrad"));
    }
    if (l > lo) {
      ST(launch_gemm(s, ly.dgrad, st));
    } else if (l > 0) {  // l == lo on rank > 0: dA_{lo-1} leaves as codes
      ST(launch_gemm(s, ly.dgrad_send, st));
      const Layer& lp = s->layers[l - 1];
      ST(comm_send(s, lp.dZ.hi, static_cast<size_t>(rows * lp.ld_out) * 2, R - 1, st));
    }
    ST(launch_gemm(s, ly.wgrad_apply, st));  // this rank's own update (no replicas: reading A6)
    const int t = tbegin(s, 1, st);
    cudaError_t e = launch_colsum_final(ly.colsum_ws, static_cast<int>((rows + 31) / 32), ly.out,
                                        ly.g32 + ly.in * ly.out, nullptr, st);
    tend(s, t, st);
    ST(check_launch(s, e, 1, "bias-gradient column sum"));
    ST(exchange_apply(s, l, st, false));  // replicas == 1: the bias update
  }
  return DFLOW_OK;
}

dflow_status finish_timing(dflow_session* s, cudaStream_t st) {
  if (!s->timing) return DFLOW_OK;
  CU(cudaStreamSynchronize(st));
  if (s->comm) CU(cudaStreamSynchronize(s->comm));
  // DFLOW_TIMELINE=<prefix>: the last timed step's launches as <prefix>.rank<R>.json
  // (start / end in ms from the step's first launch, stream, kind, GEMM epilogue)
  if (const char* tl = getenv("DFLOW_TIMELINE")) {
    if (!s->ranges.empty()) {
      std::string path = std::string(tl) + ".rank" + std::to_string(s->opt.rank) + ".json";
      if (FILE* f = fopen(path.c_str(), "w")) {
        fprintf(f, "[");
        for (size_t i = 0; i < s->ranges.size(); ++i) {
          const TimedRange& r = s->ranges[i];
          float t0 = 0, t1 = 0;
          cudaEventElapsedTime(&t0, s->ranges[0].a, r.a);
          cudaEventElapsedTime(&t1, s->ranges[0].a, r.b);
          fprintf(f, "%s{\"kind\": %d, \"comm\": %d, \"label\": \"%s\", \"t0\": %.4f, \"t1\": %.4f}",
                  i ? ", " : "", r.kind, r.comm, r.label ? r.label : "", t0, t1);
        }
        fprintf(f, "]\n");
        fclose(f);
      }
    }
  }
  for (const TimedRange& r : s->ranges) {
    float ms = 0;
    cudaEventElapsedTime(&ms, r.a, r.b);
    if (r.kind == 0) s->gemm_ms += ms;
    else if (r.kind == 1) s->other_ms += ms;
    else s->exchange_ms += ms;
  }
  s->ranges.clear();
  s->event_next = 0;
  return DFLOW_OK;
}

// The loss is final when the forward ends (k_loss_final): its device->host copy is
// enqueued right after the forward and waited for after the backward has been enqueued,
// so the host returns while the backward and the update still run (stream-ordered).
// Event record that may sit inside a step-graph capture (and is waited on outside it).
cudaError_t record_event(dflow_session* s, cudaEvent_t e, cudaStream_t st) {
  return s->capturing ? cudaEventRecordWithFlags(e, st, cudaEventRecordExternal) : cudaEventRecord(e, st);
}

dflow_status enqueue_loss(dflow_session* s, cudaStream_t st, bool want) {
  if (s->mp) {  // f4: the last rank computed C; every rank reports it
    ST(comm_broadcast_f32(s, s->loss_dev, 1, s->opt.world - 1, st));
    CU(cudaMemcpyAsync(s->loss_host + s->loss_slot, s->loss_dev, sizeof(float), cudaMemcpyDeviceToHost, st));
    CU(record_event(s, s->ev_loss_ready[s->loss_slot], st));
    s->loss_pending[s->loss_slot] = true;
    return DFLOW_OK;
  }
  if (s->replicas > 1 && !s->async && s->p2p) {
    // fused channel: push C_r to every rank (always: a rank's peers may want the mean), gather
    // the N values only when this caller wants C — no collective, so ranks may differ
    ST(check_launch(s, launch_loss_push(s->loss_dev, s->loss_peers, s->opt.rank, s->opt.world, s->epoch, st), 1,
                    "loss push"));
    if (!want) return DFLOW_OK;
    CU(cudaEventRecord(s->ev_loss, st));
    CU(cudaStreamWaitEvent(s->loss_stream, s->ev_loss, 0));
    ST(comm_rendezvous(s));  // (simulated world: every rank's push is enqueued first)
    ST(check_launch(s, launch_loss_gather(s->loss_peers.slots[s->opt.rank], s->loss_peers.flags[s->opt.rank],
                                          s->opt.world, s->epoch, s->loss_dev + 1, s->abort_dev,
                                          s->flag_timeout_ns, s->loss_stream),
                    1, "loss gather"));
    CU(cudaMemcpyAsync(s->loss_host + s->loss_slot, s->loss_dev + 1, sizeof(float), cudaMemcpyDeviceToHost,
                       s->loss_stream));
    CU(cudaEventRecord(s->ev_loss_ready[s->loss_slot], s->loss_stream));
  } else if (s->replicas > 1 && !s->async) {  // (asynchronous replicas report their own C_r)
    CU(cudaEventRecord(s->ev_loss, st));
    CU(cudaStreamWaitEvent(s->comm, s->ev_loss, 0));
    ST(comm_allreduce_f32(s, s->loss_dev, s->loss_dev + 1, 1, s->comm));
    CU(cudaMemcpyAsync(s->loss_host + s->loss_slot, s->loss_dev + 1, sizeof(float), cudaMemcpyDeviceToHost,
                       s->comm));
    CU(cudaEventRecord(s->ev_loss_ready[s->loss_slot], s->comm));
  } else {
    CU(cudaMemcpyAsync(s->loss_host + s->loss_slot, s->loss_dev, sizeof(float), cudaMemcpyDeviceToHost, st));
    CU(record_event(s, s->ev_loss_ready[s->loss_slot], st));
  }
  s->loss_pending[s->loss_slot] = true;
  return DFLOW_OK;
}

dflow_status wait_loss(dflow_session* s, float* loss_out, int slot) {
  if (!s->loss_pending[slot]) return DFLOW_OK;
  s->loss_pending[slot] = false;
  CU(cudaEventSynchronize(s->ev_loss_ready[slot]));
  ST(check_alive(s));
  float v = s->loss_host[slot];
  if (s->replicas > 1 && !s->async) v /= static_cast<float>(s->opt.world);
  if (loss_out) *loss_out = v;
  s->nonfinite = std::isfinite(v) ? 0 : 1;
  return DFLOW_OK;
}

int layer_of_variable(dflow_session* s, int sid, bool* is_bias) {
  for (int l = 0; l < s->L; ++l) {
    if (s->layers[l].n.W == sid) { *is_bias = false; return l; }
    if (s->layers[l].n.b == sid) { *is_bias = true; return l; }
  }
  return -1;
}

}  // namespace

// ===================================================================== API
dflow_status session_create(const Graph& user, const dflow_options& opt, const uint8_t* nccl_id,
                            dflow_sim_world* sim, dflow_session** out) {
  if (!out) return fail(DFLOW_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (opt.world < 1 || opt.rank < 0 || opt.rank >= opt.world)
    return fail(DFLOW_INVALID_ARGUMENT, "need 0 <= rank < world");
  if (opt.precision != DFLOW_PRECISION_BF16 && opt.precision != DFLOW_PRECISION_3XTF32)
    return fail(DFLOW_INVALID_ARGUMENT, "unknown precision");
  if (opt.exchange < DFLOW_EXCHANGE_TRUNC16 || opt.exchange > DFLOW_EXCHANGE_SR16)
    return fail(DFLOW_INVALID_ARGUMENT, "unknown exchange mode");
  if (opt.max_local_rows <= 0) return fail(DFLOW_INVALID_ARGUMENT, "max_local_rows must be > 0");
  if (opt.world > 1 && !nccl_id && !sim) return fail(DFLOW_INVALID_ARGUMENT, "world > 1 needs an NCCL unique id");
  if (sim && (opt.world != sim->world || opt.device != sim->device))
    return fail(DFLOW_INVALID_ARGUMENT, "a simulated rank needs the world's size and device");
  if (opt.world > kMaxRanks && (sim || (opt.p2p && !opt.model_parallel) || opt.async_dp))
    return fail(DFLOW_INVALID_ARGUMENT, "at most %d ranks", kMaxRanks);
  dflow_session* s = new dflow_session();
  s->sim = sim;
  s->opt = opt;
  s->cap = opt.max_local_rows;
  s->tf32 = opt.precision == DFLOW_PRECISION_3XTF32;
  s->esz = s->tf32 ? 4 : 2;
  s->mp = opt.model_parallel != 0 && opt.world > 1;
  s->replicas = s->mp ? 1 : opt.world;  // data-parallel replicas (model parallelism: one)
  if (s->mp && (opt.async_dp || opt.precision != DFLOW_PRECISION_BF16)) {
    delete s;
    return fail(DFLOW_INVALID_ARGUMENT, "model_parallel runs the bf16 path without async_dp");
  }
  s->async = opt.async_dp != 0 && opt.world > 1;
  if (s->async && (s->tf32 || !(opt.exchange == DFLOW_EXCHANGE_TRUNC16 || opt.exchange == DFLOW_EXCHANGE_SR16 ||
                                 opt.exchange == DFLOW_EXCHANGE_FP32))) {
    delete s;
    return fail(DFLOW_INVALID_ARGUMENT, "async_dp needs the bf16 path and a TRUNC16, SR16 or FP32 channel");
  }
  if (s->async && opt.world > kMaxRanks) {
    delete s;
    return fail(DFLOW_INVALID_ARGUMENT, "async_dp supports up to %d ranks", kMaxRanks);
  }
  s->defer = opt.defer_apply != 0 && !s->async && !s->mp && opt.world > 1;
  s->p2p = !s->async && !s->mp && opt.p2p && opt.world > 1 &&
           (opt.exchange == DFLOW_EXCHANGE_TRUNC16 || opt.exchange == DFLOW_EXCHANGE_SR16);
  dflow_status st = insert_exchange(user, s->replicas, opt.exchange | (s->async ? DFLOW_EXCHANGE_ASYNC : 0), &s->g,
                                    &s->remap);
  if (st == DFLOW_OK) st = match_graph(s);
  if (st == DFLOW_OK && s->mp) st = setup_mp(s);
  if (st == DFLOW_OK && s->tf32 && s->x_dtype != DFLOW_F32)
    st = fail(DFLOW_INVALID_ARGUMENT, "the 3xTF32 path needs an fp32 x placeholder");
  if (st != DFLOW_OK) {
    delete s;
    return st;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    delete s;
    return fail(DFLOW_CUDA, "no CUDA device available (dflow has no CPU fallback)");
  }
  if (opt.device < 0 || opt.device >= ndev || cudaSetDevice(opt.device) != cudaSuccess) {
    delete s;
    return fail(DFLOW_INVALID_ARGUMENT, "bad device ordinal %d", opt.device);
  }
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, opt.device);
  if (prop.major != 10) {
    delete s;
    return fail(DFLOW_CUDA, "dflow kernels are built for sm_100a; device is sm_%d%d", prop.major, prop.minor);
  }
  s->num_sms = prop.multiProcessorCount;
  if (st == DFLOW_OK) st = alloc_state(s);
  if (st == DFLOW_OK && s->mp && s->mp_hi < s->L)
    st = dmalloc(s, &s->mp_recv, s->cap * s->layers[s->mp_hi - 1].ld_out);
  if (st == DFLOW_OK) st = comm_init(s, nccl_id);
  if (st == DFLOW_OK && s->p2p) st = setup_p2p(s);
  if (st == DFLOW_OK && s->async) st = setup_async(s);
  if (st != DFLOW_OK) {
    session_destroy(s);
    return st;
  }
  *out = s;
  return DFLOW_OK;
}

void session_destroy(dflow_session* s) {
  if (!s) return;
  cudaSetDevice(s->opt.device);
  cudaDeviceSynchronize();
  for (void* p : s->ipc_opened) cudaIpcCloseMemHandle(p);
  if (s->sym) cudaFree(s->sym);
  if (s->p2p_done) cudaFree(s->p2p_done);
  if (s->wsym) comm_symmetric_free(s, s->wsym);
  s->wsym = nullptr;
  comm_destroy(s);
  if (s->abort_host) cudaFreeHost(s->abort_host);
  if (s->sched_fd) cudaFree(s->sched_fd);
  for (Layer& ly : s->layers) {
    for (void* p : {(void*)ly.W32, (void*)ly.b32, (void*)ly.g32, (void*)ly.q16, ly.recv, ly.own, ly.gath,
                    (void*)ly.colsum_ws})
      if (p) cudaFree(p);
    if (!s->multicast) free_operand(ly.Wop);  // (multicast: the window region, freed below)
    free_operand(ly.A);
    free_operand(ly.dZ);
  }
  free_operand(s->A0);
  if (s->mp_recv) cudaFree(s->mp_recv);
  if (s->sched_w) cudaFree(s->sched_w);
  for (void* p : {(void*)s->AL32, (void*)s->loss_partials, (void*)s->loss_dev, (void*)s->mask_dev, s->host_stage[0],
                  s->host_stage[1], s->xbuf[0], s->xbuf[1], s->xbuf[2], s->xbuf[3]})
    if (p) cudaFree(p);
  if (s->loss_host) cudaFreeHost(s->loss_host);
  for (cudaEvent_t e : {s->ev_loss_ready[0], s->ev_loss_ready[1], s->ev_x_free})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : s->ev_grad) cudaEventDestroy(e);
  for (cudaEvent_t e : s->ev_apply) cudaEventDestroy(e);
  for (cudaEvent_t e : s->event_pool) cudaEventDestroy(e);
  if (s->ev_loss) cudaEventDestroy(s->ev_loss);
  for (auto& g : s->step_graphs) cudaGraphExecDestroy(g.exec);
  for (cudaEvent_t e : {s->ev_h2d, s->ev_h2d_y, s->ev_feeds_free, s->ev_gin, s->ev_gout})
    if (e) cudaEventDestroy(e);
  if (s->gstream) cudaStreamDestroy(s->gstream);
  if (s->h2d) cudaStreamDestroy(s->h2d);
  for (int i = 0; i < 2; ++i) {
    if (s->side[i]) cudaStreamDestroy(s->side[i]);
    if (s->ev_side_join[i]) cudaEventDestroy(s->ev_side_join[i]);
  }
  if (s->comm && s->comm_owned) cudaStreamDestroy(s->comm);
  if (s->loss_stream) cudaStreamDestroy(s->loss_stream);
  cudaGetLastError();
  delete s;
}

// wait = false (pipelined host steps): the loss copy is enqueued into slot s->loss_slot and
// left pending; the caller collects it later with wait_loss.
// The feeds a train step needs, checked before anything is enqueued.
dflow_status validate_train_feeds(dflow_session* s, const Feeds& f) {
  const bool need_x = !s->mp || s->mp_lo == 0;
  const bool need_y = s->loss_kind == DFLOW_LOSS_MSE && (!s->mp || s->mp_hi == s->L);
  if (need_x && !f.x) return fail(DFLOW_INVALID_ARGUMENT, "x must be fed");
  if (need_x && f.ldx < s->layers[0].in) return fail(DFLOW_INVALID_ARGUMENT, "ld of x < its width");
  if (need_y && !f.y) return fail(DFLOW_INVALID_ARGUMENT, "y must be fed (MSE loss)");
  if (need_y && f.ldy < s->layers[s->L - 1].out) return fail(DFLOW_INVALID_ARGUMENT, "ld of y < its width");
  return DFLOW_OK;
}

dflow_status session_train_step_impl(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* ptrs,
                                     const int64_t* ld, int64_t rows, float* loss_out, cudaStream_t st, bool wait) {
  if (!s->trainable) return fail(DFLOW_UNIMPLEMENTED, "graph has no ApplyGradientDescent nodes to run");
  ST(check_rows(s, rows));
  Feeds f;
  ST(resolve_feeds(s, n_feeds, feeds, ptrs, ld, &f));
  ST(validate_train_feeds(s, f));  // a rejected call changes nothing, not even the step counter
  s->epoch++;  // p2p exchange flags / SR16 draws of this step
  // one step's work on `stream` (also what a step graph captures)
  auto body = [&](cudaStream_t stream) -> dflow_status {
    s->launches = s->gemm_launches = 0;
    if (s->async && s->opt.async_dp == 1) ST(async_pull_pipelined(s, stream));  // the replica reads the shared parameters
    if (s->mp) {  // f4: this rank's layers of the one replica
      ST(run_forward_mp(s, f, rows, stream));
      CU(record_event(s, s->ev_x_free, stream));
      CU(record_event(s, s->ev_feeds_free, stream));
      ST(enqueue_loss(s, stream, true));  // every rank takes part in the loss broadcast
      ST(run_backward_mp(s, rows, stream));
    } else {
      ST(run_forward(s, f, rows, stream, FWD_TRAIN));
      CU(record_event(s, s->ev_feeds_free, stream));  // x and y are not read after the forward
      // synchronous replicas: every rank takes part in the loss exchange whether or not it
      // asked for the value (the NCCL schedule's all-reduce is a collective; the fused
      // channel's push is one-sided and only a caller that wants C gathers)
      if (loss_out || (s->replicas > 1 && !s->async)) ST(enqueue_loss(s, stream, loss_out != nullptr));
      ST(run_backward(s, rows, stream, 0));
    }
    s->last_launches = s->launches;
    s->last_gemm_launches = s->gemm_launches;
    return DFLOW_OK;
  };
  if (s->opt.graphs && s->opt.world == 1 && !s->timing) {
    dflow_session::StepGraph* g = nullptr;
    const bool ywait = s->y_upload_pending;  // host-fed y: the graph holds an external wait before the last GEMM
    for (auto& e : s->step_graphs)
      if (e.x == f.x && e.y == f.y && e.ldx == f.ldx && e.ldy == f.ldy && e.rows == rows &&
          e.loss == (loss_out != nullptr) && e.ywait == ywait && e.slot == s->loss_slot)
        g = &e;
    s->y_upload_pending = false;
    if (!g) {
      s->y_upload_pending = ywait;
      CU(cudaStreamBeginCapture(s->gstream, cudaStreamCaptureModeThreadLocal));
      s->capturing = true;
      const dflow_status r = body(s->gstream);
      s->capturing = false;
      cudaGraph_t graph = nullptr;
      const cudaError_t ec = cudaStreamEndCapture(s->gstream, &graph);
      if (r != DFLOW_OK) {
        if (graph) cudaGraphDestroy(graph);
        return r;
      }
      CU(ec);
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      CU(ei);
      if (s->step_graphs.size() >= 8) {  // bounded cache: drop the oldest
        cudaGraphExecDestroy(s->step_graphs.front().exec);
        s->step_graphs.erase(s->step_graphs.begin());
      }
      s->step_graphs.push_back({f.x, f.y, f.ldx, f.ldy, rows, loss_out != nullptr, ywait, s->loss_slot, exec});
      g = &s->step_graphs.back();
    }
    CU(cudaEventRecord(s->ev_gin, st));
    CU(cudaStreamWaitEvent(s->gstream, s->ev_gin, 0));
    CU(cudaGraphLaunch(g->exec, s->gstream));
    CU(cudaEventRecord(s->ev_gout, s->gstream));
    CU(cudaStreamWaitEvent(st, s->ev_gout, 0));
    if (loss_out) s->loss_pending[s->loss_slot] = true;
  } else {
    const dflow_status r = body(st);
    if (r != DFLOW_OK) {  // part of the step may be enqueued: the replicas are out of step
      s->poisoned = true;
      return r;
    }
  }
  CU(cudaGetLastError());
  if (wait) {
    if (loss_out) ST(wait_loss(s, loss_out, s->loss_slot));
    else s->loss_pending[s->loss_slot] = false;  // (the all-reduced copy lands unread)
  }
  if (s->timing) {
    // DFLOW_TIMING_BATCH=k: read the events back every k steps only, so the timeline
    // (DFLOW_TIMELINE) shows k consecutive steps running back to back, overlaps included
    static const int batch = [] {
      const char* e = getenv("DFLOW_TIMING_BATCH");
      return (e && atoi(e) > 1) ? atoi(e) : 1;
    }();
    if (++s->timing_pending >= batch) {
      ST(finish_timing(s, st));
      s->timed_steps += s->timing_pending;
      s->timing_pending = 0;
    }
  }
  return DFLOW_OK;
}

dflow_status session_train_step(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* ptrs,
                                const int64_t* ld, int64_t rows, float* loss_out, cudaStream_t st) {
  return session_train_step_impl(s, n_feeds, feeds, ptrs, ld, rows, loss_out, st, true);
}

// pipelined: returns once the step is enqueued; *loss_out = the previous pipelined step's
// loss (its copy was enqueued with that step; waiting for it here cannot stall the device)
dflow_status session_train_step_host(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                     const void* const* host_ptrs, const int64_t* ld, int64_t rows,
                                     float* loss_out, cudaStream_t st, bool pipelined, int32_t* has_loss) {
  ST(check_alive(s));
  if (n_feeds < 0 || n_feeds > 2 || (n_feeds > 0 && (!feeds || !host_ptrs || !ld)))
    return fail(DFLOW_INVALID_ARGUMENT, "bad feed arrays");
  const void* dptrs[2];
  int sids[2] = {-1, -1};
  for (int i = 0; i < n_feeds; ++i) {
    sids[i] = (feeds[i] >= 0 && feeds[i] < (int)s->remap.size()) ? s->remap[feeds[i]] : -1;
    if (sids[i] < 0) return fail(DFLOW_INVALID_ARGUMENT, "bad feed node");
  }
  if (has_loss) *has_loss = 0;
  // x first, then y (its upload overlaps the first layers of the forward); each waits for
  // the previous step to be done with its staging buffer (x: the input cast; y: the loss GEMM)
  for (int pass = 0; pass < 2; ++pass) {
    CU(cudaStreamWaitEvent(s->h2d, pass == 0 ? s->ev_x_free : s->ev_feeds_free, 0));
    for (int i = 0; i < n_feeds; ++i) {
      if ((sids[i] == s->y) != (pass == 1)) continue;
      const size_t esz = (sids[i] == s->x && s->x_dtype == DFLOW_BF16) ? 2 : 4;
      const size_t bytes = static_cast<size_t>(rows) * ld[i] * esz;
      if (s->host_stage_bytes[i] < bytes) {
        if (s->host_stage[i]) cudaFree(s->host_stage[i]);
        s->host_stage[i] = nullptr;
        if (cudaMalloc(&s->host_stage[i], bytes) != cudaSuccess) return fail(DFLOW_OOM, "staging buffer");
        s->host_stage_bytes[i] = bytes;
      }
      CU(cudaMemcpyAsync(s->host_stage[i], host_ptrs[i], bytes, cudaMemcpyHostToDevice, s->h2d));
      dptrs[i] = s->host_stage[i];
    }
    CU(cudaEventRecord(pass == 0 ? s->ev_h2d : s->ev_h2d_y, s->h2d));
  }
  CU(cudaStreamWaitEvent(st, s->ev_h2d, 0));
  s->y_upload_pending = true;
  float loss = 0.f;
  if (pipelined) {
    const int prev = s->loss_slot ^ 1;
    s->loss_slot = prev ^ 1;  // this step's loss goes to the current slot
    const dflow_status r = session_train_step_impl(s, n_feeds, feeds, dptrs, ld, rows, &loss, st, false);
    s->y_upload_pending = false;
    if (r != DFLOW_OK) return r;
    const bool had = s->loss_pending[prev];
    ST(wait_loss(s, &loss, prev));  // the previous step's loss (its host buffers are free now too)
    s->loss_slot = prev;            // the next pipelined step writes the other slot
    if (had) {
      if (loss_out) *loss_out = loss;
      if (has_loss) *has_loss = 1;
    }
    return DFLOW_OK;
  }
  const dflow_status r = session_train_step(s, n_feeds, feeds, dptrs, ld, rows, &loss, st);
  s->y_upload_pending = false;
  if (r != DFLOW_OK) return r;
  if (loss_out) *loss_out = loss;
  else CU(cudaEventSynchronize(s->ev_h2d_y));  // host_ptrs are reusable on return
  return DFLOW_OK;
}

// The loss of the last pipelined host step (waits for it), if one is pending.
dflow_status session_last_loss(dflow_session* s, float* loss_out, int32_t* has_loss) {
  ST(check_alive(s));
  if (has_loss) *has_loss = 0;
  for (int k = 0; k < 2; ++k) {
    const int slot = s->loss_slot ^ 1 ^ k;  // the most recent pipelined step wrote loss_slot ^ 1
    if (!s->loss_pending[slot]) continue;
    float v = 0.f;
    ST(wait_loss(s, &v, slot));
    if (loss_out) *loss_out = v;
    if (has_loss) *has_loss = 1;
    return DFLOW_OK;
  }
  return DFLOW_OK;
}

dflow_status session_forward(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* ptrs,
                             const int64_t* ld, int64_t rows, dflow_node fetch, void* out, cudaStream_t st) {
  if (s->mp) return fail(DFLOW_UNIMPLEMENTED, "model_parallel sessions run train steps only");
  ST(check_rows(s, rows));
  Feeds f;
  ST(resolve_feeds(s, n_feeds, feeds, ptrs, ld, &f));
  if (fetch < 0 || fetch >= (int)s->remap.size() || !out) return fail(DFLOW_INVALID_ARGUMENT, "bad fetch");
  const int sid = s->remap[fetch];
  if (sid == s->cost && s->loss_kind == DFLOW_LOSS_MSE && !f.y)
    return fail(DFLOW_INVALID_ARGUMENT, "fetching the MSE cost needs y");
  ST(run_forward(s, f, rows, st, FWD_ONLY));
  if (sid == s->cost) {
    CU(cudaMemcpyAsync(out, s->loss_dev, sizeof(float), cudaMemcpyDeviceToDevice, st));
    return DFLOW_OK;
  }
  for (int l = 0; l < s->L; ++l) {
    if (s->layers[l].n.relu != sid) continue;
    const Layer& ly = s->layers[l];
    cudaError_t e;
    if (l + 1 == s->L)
      e = launch_copy_f32(s->AL32, s->ld_AL32, rows, ly.out, static_cast<float*>(out), ly.out, st);
    else if (s->tf32)
      e = launch_join_tf32(static_cast<const float*>(ly.A.hi), static_cast<const float*>(ly.A.lo), ly.ld_out, rows,
                           ly.out, static_cast<float*>(out), st);
    else
      e = launch_bf16_to_f32(static_cast<const __nv_bfloat16*>(ly.A.hi), ly.ld_out, rows, ly.out,
                             static_cast<float*>(out), st);
    return check_launch(s, e, 1, "fetch copy");
  }
  return fail(DFLOW_UNIMPLEMENTED, "forward fetch must be a Relu node or the cost");
}

dflow_status session_fetch_gradients(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                     const void* const* ptrs, const int64_t* ld, int64_t rows, int n,
                                     const dflow_node* grads, void* const* out, cudaStream_t st) {
  if (s->mp) return fail(DFLOW_UNIMPLEMENTED, "model_parallel sessions run train steps only");
  if (s->lossgrad < 0) return fail(DFLOW_UNIMPLEMENTED, "graph has no gradient nodes");
  ST(check_rows(s, rows));
  Feeds f;
  ST(resolve_feeds(s, n_feeds, feeds, ptrs, ld, &f));
  if (n < 0 || (n > 0 && (!grads || !out))) return fail(DFLOW_INVALID_ARGUMENT, "bad fetch arrays");
  ST(run_forward(s, f, rows, st, FWD_FETCH));
  ST(run_backward(s, rows, st, 1));
  for (int i = 0; i < n; ++i) {
    const int sid = (grads[i] >= 0 && grads[i] < (int)s->remap.size()) ? s->remap[grads[i]] : -1;
    bool done = false;
    for (int l = 0; l < s->L && !done; ++l) {
      Layer& ly = s->layers[l];
      if (sid == ly.n.dW) {
        CU(cudaMemcpyAsync(out[i], ly.g32, ly.in * ly.out * sizeof(float), cudaMemcpyDeviceToDevice, st));
        done = true;
      } else if (sid == ly.n.db) {
        CU(cudaMemcpyAsync(out[i], ly.g32 + ly.in * ly.out, ly.out * sizeof(float), cudaMemcpyDeviceToDevice, st));
        done = true;
      } else if (sid == ly.n.dX && l == 0) {
        // dx = dZ_1 W_1^T (Fig.5), fp32, written straight by the GEMM epilogue
        GemmDesc d{};
        d.tf32 = s->tf32;
        d.M = rows; d.N = ly.in; d.K = ly.out;
        d.A = ly.dZ.hi; d.A2 = ly.dZ.lo; d.lda = ly.ld_out; d.a_mn = false;
        d.B = ly.Wop.hi; d.B2 = ly.Wop.lo; d.ldb = ly.ld_wb; d.b_mn = false;
        d.epilogue = EPI_F32;
        d.out_f32 = static_cast<float*>(out[i]); d.ldo32 = ly.in;
        d.sched = s->sched_fd + 4;
        GemmPlan p;
        ST(gemm_plan(s, d, &p));
        ST(launch_gemm(s, p, st));
        done = true;
      }
    }
    if (!done) return fail(DFLOW_UNIMPLEMENTED, "fetchable gradients are dW_l, db_l and dx");
  }
  return DFLOW_OK;
}

dflow_status session_fetch_masks(dflow_session* s, int layer, uint32_t* bits_host) {
  ST(check_alive(s));
  if (layer < 1 || layer > s->L || !bits_host) return fail(DFLOW_INVALID_ARGUMENT, "layer must be 1..L");
  if (!s->have_forward) return fail(DFLOW_NOT_INITIALIZED, "no forward pass has run yet");
  const Layer& ly = s->layers[layer - 1];
  const int64_t rows = s->last_rows;
  const int64_t words = (rows * ly.out + 31) / 32;
  // the forward ran on the caller's stream, which may be non-blocking: order after everything
  CU(cudaDeviceSynchronize());
  cudaStream_t st = nullptr;
  cudaError_t e;
  if (layer == s->L)
    e = launch_relu_mask_bits_f32(s->AL32, s->ld_AL32, rows, ly.out, s->mask_dev, st);
  else if (s->tf32)  // mask from the tf32 big part (reading A24)
    e = launch_relu_mask_bits_f32(static_cast<const float*>(ly.A.hi), ly.ld_out, rows, ly.out, s->mask_dev, st);
  else
    e = launch_relu_mask_bits(static_cast<const __nv_bfloat16*>(ly.A.hi), ly.ld_out, rows, ly.out, s->mask_dev, st);
  if (e != cudaSuccess) {
    s->poisoned = true;
    return fail(DFLOW_CUDA, "mask kernel: %s", cudaGetErrorString(e));
  }
  CU(cudaMemcpy(bits_host, s->mask_dev, words * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return DFLOW_OK;
}

dflow_status session_variable_assign(dflow_session* s, dflow_node var, const void* src, int on_dev, cudaStream_t st) {
  ST(check_alive(s));
  if (var < 0 || var >= (int)s->remap.size() || !src) return fail(DFLOW_INVALID_ARGUMENT, "bad variable");
  bool is_bias;
  const int l = layer_of_variable(s, s->remap[var], &is_bias);
  if (l < 0) return fail(DFLOW_INVALID_ARGUMENT, "node is not a Variable of the planned MLP");
  cudaSetDevice(s->opt.device);
  ST(join_apply(s, st));
  Layer& ly = s->layers[l];
  float* dst = is_bias ? ly.b32 : ly.W32;
  const size_t bytes = (is_bias ? ly.out : ly.in * ly.out) * sizeof(float);
  if (on_dev) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  } else {
    // stream-ordered: cudaMemcpy from pageable memory may return before the DMA lands and
    // is ordered on the legacy stream only, so a kernel on a non-blocking `st` (the weight
    // cast below) could read stale W
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
  }
  if (!is_bias) {
    cudaError_t e = to_operand(s, ly.W32, ly.out, ly.Wop, ly.ld_wb, ly.in, ly.out, st);
    if (e != cudaSuccess) {
      s->poisoned = true;
      return fail(DFLOW_CUDA, "weight cast: %s", cudaGetErrorString(e));
    }
  }
  if (s->async) CU(launch_async_publish(ly.async, ly.W32, ly.b32, st));  // this rank's shard of the shared copy
  if (!on_dev) CU(cudaStreamSynchronize(st));
  return DFLOW_OK;
}

dflow_status session_variable_read(dflow_session* s, dflow_node var, void* dst, int on_dev, cudaStream_t st) {
  ST(check_alive(s));
  if (var < 0 || var >= (int)s->remap.size() || !dst) return fail(DFLOW_INVALID_ARGUMENT, "bad variable");
  bool is_bias;
  const int l = layer_of_variable(s, s->remap[var], &is_bias);
  if (l < 0) return fail(DFLOW_INVALID_ARGUMENT, "node is not a Variable of the planned MLP");
  cudaSetDevice(s->opt.device);
  ST(join_apply(s, st));
  Layer& ly = s->layers[l];
  if (s->async) ST(async_pull(s, st));  // the shared parameters, not this replica's last pull
  if (s->p2p && ly.p2p.owner_apply && !is_bias)  // owner-apply: other shards live with their owners
    CU(launch_gather_w32(ly.p2p, st));
  const float* src = is_bias ? ly.b32 : ly.W32;
  const size_t bytes = (is_bias ? ly.out : ly.in * ly.out) * sizeof(float);
  if (on_dev) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToDevice, st));
  } else {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  return DFLOW_OK;
}

dflow_status session_async_pull(dflow_session* s, cudaStream_t st) {
  ST(check_alive(s));
  if (!s->async) return fail(DFLOW_INVALID_ARGUMENT, "not an async_dp session");
  cudaSetDevice(s->opt.device);
  return async_pull(s, st);
}

dflow_status session_exchange(dflow_session* s, const float* grad, float* out, size_t n, cudaStream_t st) {
  ST(check_alive(s));
  const int N = s->opt.world;
  cudaSetDevice(s->opt.device);
  ST(join_apply(s, st));
  if (N == 1 || s->opt.exchange == DFLOW_EXCHANGE_NONE) {  // no channel, no codec (reading A6)
    CU(cudaMemcpyAsync(out, grad, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
    return DFLOW_OK;
  }
  const int64_t npad = pad_to(static_cast<int64_t>(n), 8 * N), shard = npad / N;
  const bool w16 = u16_wire(s);
  const size_t esz = w16 ? 2 : 4;
  // SR16 draws of standalone exchange i (1-based): step i, layer 0 (reading A27)
  const uint32_t xstep = ++s->xchg_calls;
  const bool sr = s->opt.exchange == DFLOW_EXCHANGE_SR16;
  const uint32_t R = static_cast<uint32_t>(s->opt.rank);
  const Round16 send_code{sr ? round16_key(s->opt.sr_seed, xstep, 0, 0, R) : 0u, sr ? 1 : 0};
  const Round16 own_code{sr ? round16_key(s->opt.sr_seed, xstep, 0, 1, R) : 0u, sr ? 1 : 0};
  if (s->xbuf_bytes < static_cast<size_t>(npad) * 4) {  // grow-only scratch (send, recv, own, gath)
    CU(cudaStreamSynchronize(st));
    CU(cudaStreamSynchronize(s->comm));
    for (void*& p : s->xbuf) {
      if (p) cudaFree(p);
      p = nullptr;
    }
    s->xbuf_bytes = 0;
    for (void*& p : s->xbuf) CU(cudaMalloc(&p, static_cast<size_t>(npad) * 4));
    s->xbuf_bytes = static_cast<size_t>(npad) * 4;
  }
  void *send = s->xbuf[0], *recv = s->xbuf[1], *own = s->xbuf[2], *gath = s->xbuf[3];
  CU(cudaMemsetAsync(send, 0, npad * esz, st));
  cudaError_t e = cudaSuccess;
  if (w16) {
    e = launch_round16(grad, static_cast<uint16_t*>(send), n, send_code, 0, st);
  } else {
    e = cudaMemcpyAsync(send, grad, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
  }
  CU(e);
  CU(cudaEventRecord(s->ev_loss, st));
  CU(cudaStreamWaitEvent(s->comm, s->ev_loss, 0));
  cudaStream_t cs = s->comm;
  if (w16) {
    ST(comm_alltoall(s, send, recv, shard * 2, cs));
    CU(launch_owner_reduce_t16(static_cast<uint16_t*>(recv), shard, N, static_cast<uint16_t*>(own), cs, own_code,
                               static_cast<int64_t>(s->opt.rank) * shard));
    ST(comm_allgather(s, own, gath, shard * 2, cs));
    CU(launch_expand16(static_cast<uint16_t*>(gath), out, n, cs));
  } else if (s->opt.exchange == DFLOW_EXCHANGE_FP32) {
    ST(comm_alltoall(s, send, recv, shard * 4, cs));
    CU(launch_owner_reduce_f32(static_cast<float*>(recv), shard, N, static_cast<float*>(own), cs));
    ST(comm_allgather(s, own, gath, shard * 4, cs));
    CU(cudaMemcpyAsync(out, gath, n * sizeof(float), cudaMemcpyDeviceToDevice, cs));
  } else {
    ST(comm_allreduce_f32(s, static_cast<const float*>(send), static_cast<float*>(gath), npad, cs));
    CU(launch_scale_f32(static_cast<float*>(gath), npad, 1.0f / N, cs));
    CU(cudaMemcpyAsync(out, gath, n * sizeof(float), cudaMemcpyDeviceToDevice, cs));
  }
  // stream-ordered completion: later work on `st` sees `out`
  CU(cudaEventRecord(s->ev_loss, cs));
  CU(cudaStreamWaitEvent(st, s->ev_loss, 0));
  return DFLOW_OK;
}

dflow_status session_sync(dflow_session* s, cudaStream_t st) {
  ST(check_alive(s));
  cudaSetDevice(s->opt.device);
  return join_apply(s, st);
}

dflow_status session_stats(dflow_session* s, dflow_stats* out) {
  if (!out) return fail(DFLOW_INVALID_ARGUMENT, "out is NULL");
  memset(out, 0, sizeof *out);
  out->launches_per_step = s->last_launches;
  out->gemm_launches_per_step = s->last_gemm_launches;
  out->layers = s->L;
  out->nonfinite = s->nonfinite;
  out->gemm_ms = s->gemm_ms;
  out->other_ms = s->other_ms;
  out->exchange_ms = s->exchange_ms;
  out->timed_steps = s->timed_steps;
  const int64_t b = s->planned_rows > 0 ? s->planned_rows : 0;
  double f = 0;
  for (int l = 0; l < s->L; ++l) {
    const double io = static_cast<double>(s->layers[l].in) * s->layers[l].out;
    f += 2.0 * b * io * (l > 0 ? 3 : 2);
  }
  out->gemm_flops_per_step = f;
  out->multicast = s->multicast ? 1 : 0;
  return DFLOW_OK;
}

}  // namespace dflow
