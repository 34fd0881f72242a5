/* dflow.h — C ABI of the B200-native replicated Relu(XW+b) MLP train step
 * (arXiv 1603.04467, "TensorFlow: Large-Scale Machine Learning on
 * Heterogeneous Distributed Systems").
 *
 * The calls follow the paper's statement of the problem:
 *   1. build a dataflow graph of ops              PAPER.md §2 :159-185, Fig.1 :100-106
 *   2. add its gradient graph                     PAPER.md §4.1 :494-518 ("[db,dW,dx] = tf.gradients(C,[b,W,x])" :512)
 *   3. Run it with feeds and fetches              PAPER.md §2 :237-254, §4.2 :564-572
 *   4. as a synchronously replicated train step   PAPER.md §7 :932-945 (Fig.7 top)
 *      whose cross-device gradient transfers are compressed 32->16->32
 *                                                 PAPER.md §5.5 :805-821
 *
 * Conventions (all functions):
 *   - Return dflow_status; DFLOW_OK == 0.  No exception or abort crosses the ABI.
 *     dflow_last_error() gives a thread-local message for the last failure.
 *   - Pointers are plain host or device pointers; sizes are element counts.
 *     Matrices are row-major with an explicit leading dimension (elements).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - A CUDA or NCCL failure inside a session poisons it: every later call on that
 *     session returns DFLOW_SESSION_POISONED; destroy and recreate it (the paper's
 *     "aborted and restarted").
 *   - No CPU fallback: without a usable sm_100 GPU, compute entry points return
 *     DFLOW_CUDA.  Graph-building entry points are host-only and need no GPU.
 */
#ifndef DFLOW_H_
#define DFLOW_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef int32_t dflow_status;
#define DFLOW_OK 0
#define DFLOW_INVALID_ARGUMENT 1
#define DFLOW_DUPLICATE_NAME 2      /* SPEC.md:122 add_node errors */
#define DFLOW_UNKNOWN_OP 3
#define DFLOW_DANGLING_INPUT 4
#define DFLOW_SHAPE_MISMATCH 5
#define DFLOW_NON_DIFFERENTIABLE 6  /* SPEC.md:358 add_gradients errors */
#define DFLOW_NON_SCALAR_TARGET 7
#define DFLOW_UNIMPLEMENTED 8       /* graph is not a chain the GPU planner can fuse */
#define DFLOW_NOT_INITIALIZED 9
#define DFLOW_CUDA 10
#define DFLOW_NCCL 11
#define DFLOW_OOM 12
#define DFLOW_SESSION_POISONED 13
#define DFLOW_BUFFER_TOO_SMALL 14

/* Thread-local, valid until the next dflow_* call on this thread. */
const char* dflow_last_error(void);
/* Static string naming a status code, e.g. "DFLOW_SHAPE_MISMATCH". */
const char* dflow_status_name(dflow_status s);
/* Library version string. */
const char* dflow_version(void);

typedef enum { DFLOW_F32 = 1, DFLOW_BF16 = 7, DFLOW_U16 = 8 } dflow_dtype;
typedef int32_t dflow_node; /* node id; every hot-path op has exactly one output (port 0) */
typedef struct dflow_graph dflow_graph;
typedef struct dflow_session dflow_session;

#define DFLOW_BATCH (-1)   /* unknown (batch) dimension; only Placeholders may have it */
#define DFLOW_LOSS_MSE 0   /* C = sum((a - y)^2) / (2 * rows * cols)   (reading A2) */
#define DFLOW_LOSS_SUM 1   /* C = sum(a) / rows                        (reading A2) */

/* ------------------------------------------------------------------ graph
 * Host-only, caller-owned.  Node names match [A-Za-z0-9_./]+ and are unique.
 * A failing call leaves the graph unchanged.              */
dflow_status dflow_graph_create(dflow_graph** out);
void dflow_graph_destroy(dflow_graph* g);
dflow_status dflow_graph_num_nodes(const dflow_graph* g, int32_t* out);
dflow_status dflow_node_by_name(const dflow_graph* g, const char* name, dflow_node* out);

/* Placeholder: a fed input ("tf.placeholder"); dims may hold DFLOW_BATCH. */
dflow_status dflow_placeholder(dflow_graph* g, const char* name, dflow_dtype dtype, int rank,
                               const int64_t* dims, dflow_node* out);
/* Variable: persistent mutable tensor; static dims. */
dflow_status dflow_variable(dflow_graph* g, const char* name, dflow_dtype dtype, int rank,
                            const int64_t* dims, dflow_node* out);
/* MatMul(a, b) = op(a) op(b) (Table 1); rank-2 operands. */
dflow_status dflow_matmul(dflow_graph* g, const char* name, dflow_node a, dflow_node b, int transpose_a,
                          int transpose_b, dflow_node* out);
/* Add(a, b): same shapes, or b rank-1 broadcast over the rows of a (BiasAdd, Fig.1 "Wx+b"). */
dflow_status dflow_add(dflow_graph* g, const char* name, dflow_node a, dflow_node b, dflow_node* out);
/* Relu(x) = max(x, 0). */
dflow_status dflow_relu(dflow_graph* g, const char* name, dflow_node x, dflow_node* out);
/* Scalar cost C ("C = [...]"; reading A2).  target = -1 for DFLOW_LOSS_SUM. */
dflow_status dflow_loss(dflow_graph* g, const char* name, int kind, dflow_node pred, dflow_node target,
                        dflow_node* out);
/* Gradient graph: appends one gradient-function node per op on
 * the paths xs -> cost, named grad/<forward-name>/<suffix>, partials summed by AddN,
 * ZerosLike for sources C does not depend on.  out_grads[i] = dC/dxs[i].        */
dflow_status dflow_gradients(dflow_graph* g, dflow_node cost, int n, const dflow_node* xs,
                             dflow_node* out_grads);
/* ApplyGradientDescent: var <- var - lr * grad. */
dflow_status dflow_apply_gradient_descent(dflow_graph* g, const char* name, dflow_node var, float lr,
                                          dflow_node grad, dflow_node* out);
/* JSON {"version":1,"nodes":[{name, op, inputs, attrs, dtype, shape}]}.  Writes at
 * most cap bytes (NUL-terminated); *needed = full length + 1.  Returns
 * DFLOW_BUFFER_TOO_SMALL if cap < *needed. */
dflow_status dflow_graph_to_json(const dflow_graph* g, char* buf, size_t cap, size_t* needed);

/* Compression-insertion pass alone (host only): *out = a new graph equal to g with,
 * for world > 1, Truncate16 -> CrossReplicaMeanT16 -> Expand16 (TRUNC16) or
 * CrossReplicaMean (FP32 modes) between every gradient and its ApplyGradientDescent
 * (PAPER.md:813-821 on the :934-941 channel).  world == 1 / NONE: a copy (reading A6).
 * The caller owns *out (dflow_graph_destroy).  Node ids of g keep their meaning for
 * every node of g in *out only through dflow_node_by_name.                       */
dflow_status dflow_graph_insert_exchange(const dflow_graph* g, int world, int exchange, dflow_graph** out);

/* Partition pass (f4): device_of_node[i] (n_nodes = every node of g, in
 * id order) places node i; *out receives device `device`'s subgraph, in which every
 * cross-device edge x -> y is replaced by Recv [-> Expand16] (one per endpoint and
 * destination, shared by all its consumers there) and the producers' side gets
 * [Truncate16 ->] Send (compress = 1: the channel codec of PAPER.md:813-821, reading A33).
 * Send/Recv carry tensor_name, send_device, recv_device.  Caller owns *out.           */
dflow_status dflow_graph_partition(const dflow_graph* g, const int32_t* device_of_node, int32_t n_nodes, int32_t device,
                                   int32_t compress, dflow_graph** out);

/* ---------------------------------------------------------------- session
 * One session per (rank, GPU).  dflow_session_create copies the graph (an
 * immutable snapshot), runs the replication + compression-insertion pass and
 * the planner (matches MatMul->Add->Relu chains + loss + gradient graph onto
 * fused kernels; any unmatched node -> DFLOW_UNIMPLEMENTED), allocates all
 * device state on `device`, and (world > 1) initialises NCCL from nccl_id.   */
#define DFLOW_PRECISION_BF16 0    /* bf16 operands, fp32 accumulate/master weights (reading A13) */
#define DFLOW_PRECISION_3XTF32 1  /* fp32-faithful 3xTF32 split (reading A14)                      */
#define DFLOW_EXCHANGE_TRUNC16 0  /* alltoall(u16) + owner fold + allgather(u16) (readings A5-A7) */
#define DFLOW_EXCHANGE_FP32 1     /* same schedule with fp32 payloads (deterministic)              */
#define DFLOW_EXCHANGE_FP32_NCCL 2 /* ncclAllReduce(sum, fp32) then x 1/N (library baseline)        */
#define DFLOW_EXCHANGE_NONE 3     /* debug/timing only: no exchange (N>1 results are wrong)        */
#define DFLOW_EXCHANGE_ASYNC 0x100 /* flag for dflow_graph_insert_exchange: the asynchronous-replica
                                      channel (f3): code -> expand -> apply, no cross-replica mean */
#define DFLOW_EXCHANGE_SR16 4     /* TRUNC16's schedule with both 32->16 codings done by stochastic
                                     rounding (f2; "probabilistic rounding";
                                     readings A26-A28; draws keyed by options.sr_seed)           */

typedef struct {
  int32_t world;          /* N replicas (one process or thread per GPU)                      */
  int32_t rank;           /* this replica, 0..N-1; gets rows [rank*b, (rank+1)*b) (reading A4) */
  int32_t device;         /* CUDA device ordinal                                              */
  int32_t precision;      /* DFLOW_PRECISION_*                                                */
  int32_t exchange;       /* DFLOW_EXCHANGE_*                                                 */
  int32_t overlap;        /* 1: per-layer exchange on a comm stream overlapped with backward  */
  int32_t sm_reserve;     /* SMs left free by the GEMMs for concurrent NCCL kernels          */
  int64_t max_local_rows; /* capacity b_max of every activation buffer                        */
  int32_t p2p;            /* TRUNC16, N > 1: 1 = fused NVLink exchange (the dW epilogue stores the
                             truncated tiles into the owners' buffers through CUDA IPC peer
                             pointers; owner fold + all-gather by peer stores); 0 = NCCL calls  */
  uint32_t sr_seed;       /* SR16: seed of the counter-based draw streams (reading A27)        */
  int32_t async_dp;       /* world > 1, bf16: 1 = asynchronous replicas (f3):
                             each train step pulls the shared (sharded) parameters over NVLink,
                             computes its gradient and pushes -lr * g_hat into the owners'
                             shards with NVLink reductions — no mean, no barrier (readings
                             A29-A31; exchange TRUNC16 / SR16 / FP32 = the coding of the
                             cross-device pushes); 2 = the same without the automatic pull
                             (the client calls dflow_async_pull)                             */
  int32_t model_parallel; /* world > 1, bf16: 1 = layer-wise model parallelism (f4):
                             one replica; rank r holds layers [floor(r L / N), floor((r+1) L / N))
                             (reading A32), the activation crossing to the next rank and the
                             gradient crossing back travel through Send/Recv with the 16-bit
                             channel codec (A33); every rank applies its own layers' updates.
                             Every rank calls dflow_train_step with the full batch (x used
                             on rank 0, y on the last rank); the loss is broadcast.         */
  int32_t graphs;         /* world == 1: 1 = capture the train step into a CUDA graph per feed
                             signature (x, y pointers, leading dims, rows) and replay it — one
                             launch per step instead of ~4L host launches (latency-bound C2);
                             the captured kernels and their arguments are the same             */
  int32_t defer_apply;    /* synchronous world > 1 (not async_dp / model_parallel): 1 = the backward
                             runs layers L..1 with the last two dW swapped (..., dgrad 2, dW 1,
                             dW 2) and the step does not join the exchange stream: the update of
                             layer l is waited for right before the next forward of layer l, so
                             the last exchange (layer 2) overlaps the next step's layer 1 instead
                             of ending the step.  Every later dflow
                             call on any stream is ordered after the pending updates; a plain
                             synchronize of `stream` alone is not (dflow_session_sync joins them).
                             Same arithmetic, same bits as 0                                   */
} dflow_options;

/* 128-byte NCCL unique id for rank 0 to broadcast (e.g. via torch.distributed). */
dflow_status dflow_nccl_unique_id(uint8_t* out128);
dflow_status dflow_session_create(const dflow_graph* g, const dflow_options* opt, const uint8_t* nccl_id128,
                                  dflow_session** out);
void dflow_session_destroy(dflow_session* s);
/* JSON of the rewritten graph the session executes (after the compression pass). */
dflow_status dflow_session_graph_to_json(const dflow_session* s, char* buf, size_t cap, size_t* needed);

/* Variables: fp32 [dims] row-major, dense.  src/dst on host (flag 0) or device (1).
 * Assign also refreshes the bf16 working copy.  Stream-ordered on `stream`;
 * host copies are synchronous.                                                */
dflow_status dflow_variable_assign(dflow_session* s, dflow_node var, const void* src, int src_on_device,
                                   void* stream);
dflow_status dflow_variable_read(dflow_session* s, dflow_node var, void* dst, int dst_on_device, void* stream);

/* Run(targets = all ApplyGradientDescent nodes, fetch = C, feeds) on this rank's
 * shard: forward, gradient graph, compressed exchange, update.  feeds[i] is a
 * Placeholder; dev_ptrs[i] its device data (fp32 or bf16 per the placeholder's
 * dtype) [local_rows, ld[i]], borrowed and stream-ordered on `stream`.
 * local_rows = B / N.  loss_out (host) receives C = mean_r C_r: the call waits
 * only until the forward has produced it (Fig. 1: C is a
 * forward node of the graph, fetched by s.run);
 * the backward, exchange and update stay enqueued on `stream` and complete in
 * stream order (later work on `stream` sees the updated weights).  The feeds are
 * not read after the forward.  NULL = no host wait at all.                    */
dflow_status dflow_train_step(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* dev_ptrs,
                              const int64_t* ld, int64_t local_rows, float* loss_out, void* stream);
/* Same, with HOST feed buffers (pinned for async copies): copies in, steps, and
 * reads the loss back — the end-to-end path.  The upload runs on the session's
 * own copy stream, ordered after the previous step's forward (the last reader of
 * the staging buffers), so step i+1's upload overlaps step i's backward when the
 * caller loops.  host_ptrs may be reused as soon as the call returns.          */
dflow_status dflow_train_step_host(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                   const void* const* host_ptrs, const int64_t* ld, int64_t local_rows,
                                   float* loss_out, void* stream);
/* Pipelined end-to-end step (PAPER.md:239-254 Run with feeds, fetch = C; the feed copies are the
 * client -> device transfers of :564-572): the same step, but the call returns as soon as the uploads and
 * the step are enqueued, so the host can enqueue step i+1 while step i runs and the PCIe link
 * stays busy (x of step i+1 uploads as soon as step i's input cast has read its staging
 * buffer, y as soon as step i's loss GEMM has).  Every step still copies its loss to the host;
 * *prev_loss_out receives the loss of the PREVIOUS pipelined call (*has_loss = 1; 0 on the
 * first call), which that step's forward produced.  host_ptrs of a call must stay unchanged
 * until the next pipelined call (or dflow_session_last_loss) returns.                      */
dflow_status dflow_train_step_host_pipelined(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                             const void* const* host_ptrs, const int64_t* ld, int64_t local_rows,
                                             float* prev_loss_out, int32_t* has_loss, void* stream);
/* Waits for and returns the loss of the last pipelined host step (*has_loss = 0 if none). */
dflow_status dflow_session_last_loss(dflow_session* s, float* loss_out, int32_t* has_loss);
/* async_dp sessions: this replica's local parameters (and operand copies) <- the current
 * shared shards of every rank (NVLink loads), stream-ordered on `stream`.  The updates
 * other replicas push concurrently may or may not be included (no lock, reading A29). */
dflow_status dflow_async_pull(dflow_session* s, void* stream);
/* Fig.1 "s.run(C, feed_dict={x: input})": forward only, no update.  fetch is a
 * Relu node (writes fp32 [local_rows, out] dense) or the cost (writes 1 fp32). */
dflow_status dflow_forward(dflow_session* s, int n_feeds, const dflow_node* feeds, const void* const* dev_ptrs,
                           const int64_t* ld, int64_t local_rows, dflow_node fetch, void* out_dev, void* stream);
/* Fetch gradient nodes (fp32, dense, shapes as in the graph, batch = local_rows)
 * without exchange or update (Fig.5: [db, dW, dx]).                           */
dflow_status dflow_fetch_gradients(dflow_session* s, int n_feeds, const dflow_node* feeds,
                                   const void* const* dev_ptrs, const int64_t* ld, int64_t local_rows, int n,
                                   const dflow_node* grads, void* const* out_dev, void* stream);
/* Masks 1[A_l > 0] of layer `layer` (1-based) from the most recent forward on
 * this rank, bit-packed row-major (bit i of word i/32), ceil(rows*out/32) words,
 * written to HOST memory.  Input to the oracle's mask-locked mode (reading A22). */
dflow_status dflow_fetch_relu_masks(dflow_session* s, int layer, uint32_t* out_bits_host);

typedef struct {
  int32_t launches_per_step; /* dflow kernels launched by one dflow_train_step     */
  int32_t gemm_launches_per_step;
  int32_t layers;
  int32_t nonfinite;         /* non-finite guard: last step's loss was NaN/Inf */
  double gemm_ms;            /* accumulated device time of GEMM launches (timing on) */
  double other_ms;           /* accumulated device time of the other kernels       */
  double exchange_ms;        /* accumulated device time of the exchange            */
  int64_t timed_steps;
  double gemm_flops_per_step; /* algorithmic GEMM FLOPs of one step on this rank    */
  int32_t multicast;         /* 1: the fused exchange's gather leg stores through an NVLink
                                SHARP multicast address (one multimem.st per weight vector)  */
} dflow_stats;
/* Orders `stream` after every update still pending on the session's exchange stream
 * (options.defer_apply: the ApplyGradientDescent nodes of the last step, PAPER.md:262-268,
 * may still be running); a no-op otherwise.  Errors: DFLOW_SESSION_POISONED, DFLOW_CUDA. */
dflow_status dflow_session_sync(dflow_session* s, void* stream);
/* Per-kernel CUDA-event timing inside dflow_train_step (off by default). */
dflow_status dflow_session_set_timing(dflow_session* s, int enable);
dflow_status dflow_session_stats(dflow_session* s, dflow_stats* out);

/* ------------------------------------------------------- standalone ops
 * Bit-exact codec (reading A5): dst[i] = bits(src[i]) >> 16,
 * and dst[i] = float(bits = src[i] << 16).  Device pointers, n elements.       */
dflow_status dflow_truncate16(const float* src, uint16_t* dst, size_t n, void* stream);
/* a6 with either coding, on one device buffer: dst[i] = 16-bit code of src[i] at bucket
 * position idx_base + i — (bits + r) >> 16 with r = mix32((idx) ^ key) >> 16 when
 * stochastic (SR16, readings A26-A27), else bits >> 16.  Stream-ordered.        */
dflow_status dflow_round16(const float* src, uint16_t* dst, size_t n, uint32_t key, int stochastic, int64_t idx_base,
                           void* stream);
/* The SR16 stream key of one compression point (reading A27): stage 0 = a sender's
 * coding of its gradient, stage 1 = the owner's coding of the mean; step = the
 * session's 1-based step (train steps and standalone exchanges count separately,
 * see dflow_exchange); layer = bucket id (0-based layer; 0 for dflow_exchange).    */
dflow_status dflow_round16_key(uint32_t seed, uint32_t step, uint32_t layer, uint32_t stage, uint32_t rank,
                               uint32_t* key_out);
dflow_status dflow_expand16(const uint16_t* src, float* dst, size_t n, void* stream);
/* Exchange alone (a6-a8) on this session's communicator: grad_dev fp32 [n] on
 * every rank -> out_dev fp32 [n] = the g_hat every replica applies.           */
dflow_status dflow_exchange(dflow_session* s, const float* grad_dev, float* out_dev, size_t n, void* stream);
/* One GEMM through the tcgen05 kernel family (layout/epilogue unit tests):
 *   C[m,n] = sum_k A(m,k) B(k,n);  a_mn=0: A(m,k)=A[m*lda+k], 1: A[k*lda+m];
 *   b_mn=0: B(k,n)=B[n*ldb+k], 1: B[k*ldb+n]; bf16 operands, lda/ldb % 8 == 0.
 *   epilogue 0: out_f32 = acc; 1: out (u16) = bits(acc)>>16;
 *   2: relu(acc + bias) -> out (bf16) and/or out_f32; 3: out (bf16) = acc*1[mask>0].
 *   tile 0 auto, 1 = 128x128 single CTA, 2 = 256x256 CTA pair.                 */
dflow_status dflow_gemm_bf16(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, int a_mn, const void* B,
                             int64_t ldb, int b_mn, int epilogue, void* out, int64_t ldo, float* out_f32,
                             int64_t ldo32, const float* bias, const void* mask, int64_t ldm, int tile,
                             void* stream);

/* One 3xTF32 GEMM (fp32-faithful path, reading A14): every fp32 operand X is
 * passed as the pair (X_hi = tf32_rna(X), X_lo = X - X_hi), same layout and
 * leading dim (% 4 == 0); out_f32 = A_hi B_lo + A_lo B_hi + A_hi B_hi (fp32
 * accumulate).  Majors and tiles as dflow_gemm_bf16; epilogue fp32 store only. */
dflow_status dflow_gemm_3xtf32(int64_t M, int64_t N, int64_t K, const float* A_hi, const float* A_lo, int64_t lda,
                               int a_mn, const float* B_hi, const float* B_lo, int64_t ldb, int b_mn, float* out_f32,
                               int64_t ldo32, int tile, void* stream);
/* The tf32 split itself (NK13, 3xTF32 path): hi = tf32_rna(src), lo = src - hi, n elements. */
dflow_status dflow_split_tf32(const float* src, float* hi, float* lo, size_t n, void* stream);

/* Die of every SM of `device` (0 / 1), measured once by L2 hit latencies: an SM reaches L2 lines
 * homed on its own die faster than lines on the other die (B200: two dies, split L2).  The
 * GEMM's tile scheduler uses it to keep each die on its own half of the output.  die_of_sm:
 * [n] (SM id order); *agreement: the weakest SM's agreement with its die's near/far pattern.
 * DFLOW_UNIMPLEMENTED when the measurement gives no clean two-die split.                  */
dflow_status dflow_device_die_map(int32_t device, int32_t* die_of_sm, int32_t n, double* agreement);

/* ------------------------------------------- simulated world (test harness)
 * The N-GPU replicated step (§7 :934-941; §5.5 :813-821 channel) run by N sessions
 * ("ranks") of one process on ONE GPU, so its kernels can be checked against the oracle on a
 * single device at any N <= 8.  Each rank is a full session (its own parameters, activations,
 * buckets, receive areas and flags) created with the same options as on N GPUs; the fused
 * NVLink exchange stores into the other ranks' buffers on the same device (the peer pointers
 * of CUDA IPC become the peers' own pointers), and the NCCL collectives become host
 * rendezvous + device copies.  One host thread per rank enqueues on the world's single
 * stream, every cross-rank wait is rendezvoused on the host first, so the device never
 * waits on work that is not ahead of it in the stream.  Not a transport for real training.
 *   - The sim_* calls are synchronous (they return after the world's stream is idle).
 *   - Sessions of a world may also be used directly (dflow_variable_assign/read,
 *     dflow_fetch_gradients, and dflow_train_step of async_dp sessions, which issue no
 *     collective) with the world's stream; a collective reached by fewer than N ranks
 *     fails after DFLOW_SIM_TIMEOUT_MS (default 120 s) with DFLOW_NCCL.
 *   - Destroy the sessions (dflow_session_destroy) before the world.                   */
typedef struct dflow_sim_world dflow_sim_world;
dflow_status dflow_sim_world_create(int32_t world, int32_t device, dflow_sim_world** out);
void dflow_sim_world_destroy(dflow_sim_world* w);
/* The world's stream (cudaStream_t as void*): pass it to direct calls on its sessions. */
dflow_status dflow_sim_world_stream(dflow_sim_world* w, void** stream_out);
/* Fault injection: rank `rank` (-1 = none) sends no gradient contributions in later train
 * steps (a peer that died mid-step); the other ranks' bounded flag waits time out
 * (DFLOW_P2P_TIMEOUT_MS) and every session of the world becomes DFLOW_SESSION_POISONED.   */
dflow_status dflow_sim_world_drop_rank(dflow_sim_world* w, int32_t rank);
/* Creates all world-size ranks' sessions (options as dflow_session_create; world, rank and
 * device are taken from the world).  out: [world] sessions.                             */
dflow_status dflow_sim_sessions_create(dflow_sim_world* w, const dflow_graph* g, const dflow_options* opt,
                                       dflow_session** out);
/* dflow_train_step on every rank concurrently.  dev_ptrs: [world][n_feeds] (rank-major);
 * feeds and ld shared by all ranks; loss_out: [world] or NULL.                            */
dflow_status dflow_sim_train_step(dflow_sim_world* w, dflow_session* const* sessions, int n_feeds,
                                  const dflow_node* feeds, const void* const* dev_ptrs, const int64_t* ld,
                                  int64_t local_rows, float* loss_out);
/* dflow_exchange on every rank concurrently: grads[r], outs[r] device fp32 [n].           */
dflow_status dflow_sim_exchange(dflow_sim_world* w, dflow_session* const* sessions, const float* const* grads,
                                float* const* outs, size_t n);

#ifdef __cplusplus
}
#endif
#endif /* DFLOW_H_ */
