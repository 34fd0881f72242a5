// Cross-replica transport (see comm.h): NCCL, or the simulated N-rank world on one GPU.
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>

#include "comm.h"
#include "common.h"
#include "kernels/elementwise.h"
#include "session.h"
#include "sim.h"

namespace dflow {

namespace {

#define CU(expr)                                                                                          \
  do {                                                                                                    \
    cudaError_t e_ = (expr);                                                                              \
    if (e_ != cudaSuccess) {                                                                              \
      s->poisoned = true;                                                                                 \
      return fail(DFLOW_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    }                                                                                                     \
  } while (0)

#define NC(expr)                                                              \
  do {                                                                        \
    ncclResult_t r_ = (expr);                                                 \
    if (r_ != ncclSuccess) {                                                  \
      s->poisoned = true;                                                     \
      return fail(DFLOW_NCCL, "%s failed: %s", #expr, ncclGetErrorString(r_)); \
    }                                                                         \
  } while (0)

#define ST(expr)                     \
  do {                               \
    dflow_status st_ = (expr);       \
    if (st_ != DFLOW_OK) return st_; \
  } while (0)

// All ranks of the simulated world arrive; fails (and breaks the world, so every other
// waiter fails too instead of hanging) after the world's timeout.
dflow_status sim_barrier(dflow_session* s) {
  dflow_sim_world* w = s->sim;
  std::unique_lock<std::mutex> lk(w->mu);
  if (w->broken) {
    s->poisoned = true;
    return fail(DFLOW_NCCL, "simulated world is broken (an earlier rendezvous failed)");
  }
  const uint64_t g = w->gen;
  if (++w->arrived == w->world) {
    w->arrived = 0;
    ++w->gen;
    w->cv.notify_all();
    return DFLOW_OK;
  }
  const bool ok = w->cv.wait_for(lk, std::chrono::milliseconds(w->timeout_ms), [&] { return w->gen != g || w->broken; });
  if (!ok || w->gen == g) {
    w->broken = true;
    w->cv.notify_all();
    s->poisoned = true;
    return fail(DFLOW_NCCL, "simulated rendezvous timed out (rank %d): a rank did not reach the same collective",
                s->opt.rank);
  }
  return DFLOW_OK;
}

// publish this rank's pointer, rendezvous; afterwards w->slot[i] is rank i's pointer until
// the closing rendezvous of the same collective
dflow_status sim_publish(dflow_session* s, const void* p) {
  s->sim->slot[s->opt.rank] = p;
  return sim_barrier(s);
}

dflow_status ensure_scratch(dflow_session* s, size_t bytes) {
  if (s->sim_scratch_bytes >= bytes) return DFLOW_OK;
  if (s->sim_scratch) cudaFree(s->sim_scratch);
  s->sim_scratch = nullptr;
  s->sim_scratch_bytes = 0;
  CU(cudaMalloc(&s->sim_scratch, bytes));
  s->sim_scratch_bytes = bytes;
  return DFLOW_OK;
}

}  // namespace

bool comm_simulated(const dflow_session* s) { return s->sim != nullptr; }

bool comm_dropped(const dflow_session* s) { return s->sim && s->sim->drop_rank == s->opt.rank; }

dflow_status comm_init(dflow_session* s, const uint8_t* nccl_id) {
  if (s->opt.world <= 1 || s->sim) return DFLOW_OK;
  ncclUniqueId id;
  memcpy(&id, nccl_id, sizeof id);
  ncclResult_t r = ncclCommInitRank(&s->nccl, s->opt.world, id, s->opt.rank);
  if (r != ncclSuccess) return fail(DFLOW_NCCL, "ncclCommInitRank failed: %s", ncclGetErrorString(r));
  return DFLOW_OK;
}

void comm_destroy(dflow_session* s) {
  if (s->nccl) ncclCommDestroy(s->nccl);
  s->nccl = nullptr;
  if (s->sim_scratch) cudaFree(s->sim_scratch);
  s->sim_scratch = nullptr;
}

dflow_status comm_rendezvous(dflow_session* s) { return s->sim ? sim_barrier(s) : DFLOW_OK; }

dflow_status comm_alltoall(dflow_session* s, const void* send, void* recv, size_t bytes, cudaStream_t st) {
  if (!s->sim) {
    NC(ncclAlltoAll(send, recv, bytes, ncclUint8, s->nccl, st));
    return DFLOW_OK;
  }
  ST(sim_publish(s, send));
  const int N = s->opt.world, R = s->opt.rank;
  for (int i = 0; i < N; ++i)
    CU(cudaMemcpyAsync(static_cast<char*>(recv) + i * bytes, static_cast<const char*>(s->sim->slot[i]) + R * bytes,
                       bytes, cudaMemcpyDeviceToDevice, st));
  return sim_barrier(s);
}

dflow_status comm_allgather(dflow_session* s, const void* send, void* recv, size_t bytes, cudaStream_t st) {
  if (!s->sim) {
    NC(ncclAllGather(send, recv, bytes, ncclUint8, s->nccl, st));
    return DFLOW_OK;
  }
  ST(sim_publish(s, send));
  for (int i = 0; i < s->opt.world; ++i)
    CU(cudaMemcpyAsync(static_cast<char*>(recv) + i * bytes, s->sim->slot[i], bytes, cudaMemcpyDeviceToDevice, st));
  return sim_barrier(s);
}

dflow_status comm_allreduce_f32(dflow_session* s, const float* send, float* recv, size_t n, cudaStream_t st) {
  if (!s->sim) {
    NC(ncclAllReduce(send, recv, n, ncclFloat32, ncclSum, s->nccl, st));
    return DFLOW_OK;
  }
  // every rank sums all sends (rank order) into its scratch before any rank overwrites its
  // send (in-place reductions), then copies the sum out
  ST(ensure_scratch(s, n * sizeof(float)));
  ST(sim_publish(s, send));
  RankPtrs src{};
  for (int i = 0; i < s->opt.world; ++i) src.p[i] = static_cast<const float*>(s->sim->slot[i]);
  CU(launch_sum_ranks_f32(src, s->opt.world, static_cast<float*>(s->sim_scratch), n, st));
  ST(sim_barrier(s));
  CU(cudaMemcpyAsync(recv, s->sim_scratch, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  return DFLOW_OK;
}

dflow_status comm_broadcast_f32(dflow_session* s, float* buf, size_t n, int root, cudaStream_t st) {
  if (!s->sim) {
    NC(ncclBroadcast(buf, buf, n, ncclFloat32, root, s->nccl, st));
    return DFLOW_OK;
  }
  ST(sim_publish(s, buf));
  if (s->opt.rank != root)
    CU(cudaMemcpyAsync(buf, s->sim->slot[root], n * sizeof(float), cudaMemcpyDeviceToDevice, st));
  return sim_barrier(s);
}

// Simulated point-to-point: the sender posts its buffer and waits until the receiver has
// enqueued the copy out of it (it may not overwrite the buffer before that — the blocking
// rendezvous of a device-side ncclSend/ncclRecv pair, moved to the host).
dflow_status comm_send(dflow_session* s, const void* buf, size_t bytes, int peer, cudaStream_t st) {
  if (!s->sim) {
    NC(ncclSend(buf, bytes, ncclUint8, peer, s->nccl, st));
    return DFLOW_OK;
  }
  dflow_sim_world* w = s->sim;
  std::unique_lock<std::mutex> lk(w->mu);
  dflow_sim_world::Box& b = w->box[s->opt.rank][peer];
  b.ptr = buf;
  b.bytes = bytes;
  b.state = 1;
  w->cv.notify_all();
  if (!w->cv.wait_for(lk, std::chrono::milliseconds(w->timeout_ms), [&] { return b.state == 2 || w->broken; }) ||
      b.state != 2) {
    w->broken = true;
    w->cv.notify_all();
    s->poisoned = true;
    return fail(DFLOW_NCCL, "simulated send %d -> %d timed out", s->opt.rank, peer);
  }
  b.state = 0;
  w->cv.notify_all();
  return DFLOW_OK;
}

dflow_status comm_recv(dflow_session* s, void* buf, size_t bytes, int peer, cudaStream_t st) {
  if (!s->sim) {
    NC(ncclRecv(buf, bytes, ncclUint8, peer, s->nccl, st));
    return DFLOW_OK;
  }
  dflow_sim_world* w = s->sim;
  std::unique_lock<std::mutex> lk(w->mu);
  dflow_sim_world::Box& b = w->box[peer][s->opt.rank];
  if (!w->cv.wait_for(lk, std::chrono::milliseconds(w->timeout_ms), [&] { return b.state == 1 || w->broken; }) ||
      b.state != 1) {
    w->broken = true;
    w->cv.notify_all();
    s->poisoned = true;
    return fail(DFLOW_NCCL, "simulated recv %d <- %d timed out", s->opt.rank, peer);
  }
  if (b.bytes != bytes) {
    w->broken = true;
    w->cv.notify_all();
    s->poisoned = true;
    return fail(DFLOW_NCCL, "simulated recv size mismatch (%zu sent, %zu expected)", b.bytes, bytes);
  }
  const cudaError_t e = cudaMemcpyAsync(buf, b.ptr, bytes, cudaMemcpyDeviceToDevice, st);
  b.state = 2;
  w->cv.notify_all();
  CU(e);
  return DFLOW_OK;
}

dflow_status comm_share_ptrs(dflow_session* s, void* const* mine, int count, std::vector<void*>* all,
                             std::vector<void*>* opened) {
  const int N = s->opt.world, R = s->opt.rank;
  all->assign(static_cast<size_t>(N) * count, nullptr);
  if (s->sim) {
    ST(sim_publish(s, mine));
    for (int j = 0; j < N; ++j) {
      void* const* theirs = static_cast<void* const*>(s->sim->slot[j]);
      for (int k = 0; k < count; ++k) (*all)[j * count + k] = theirs[k];
    }
    return sim_barrier(s);
  }
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  std::vector<cudaIpcMemHandle_t> h(count);
  for (int k = 0; k < count; ++k) CU(cudaIpcGetMemHandle(&h[k], mine[k]));
  uint8_t* dev = nullptr;
  CU(cudaMalloc(&dev, 64 * count * (N + 1)));
  // (stream-ordered copies: a plain cudaMemcpy from pageable memory may return before the
  // data has landed, and runs on the legacy stream the non-blocking comm stream ignores)
  CU(cudaMemcpyAsync(dev, h.data(), 64 * count, cudaMemcpyHostToDevice, s->comm));
  NC(ncclAllGather(dev, dev + 64 * count, 64 * count, ncclUint8, s->nccl, s->comm));
  std::vector<cudaIpcMemHandle_t> allh(static_cast<size_t>(N) * count);
  CU(cudaMemcpyAsync(allh.data(), dev + 64 * count, 64 * count * N, cudaMemcpyDeviceToHost, s->comm));
  CU(cudaStreamSynchronize(s->comm));
  cudaFree(dev);
  for (int j = 0; j < N; ++j) {
    for (int k = 0; k < count; ++k) {
      if (j == R) {
        (*all)[j * count + k] = mine[k];
      } else {
        void* p = nullptr;
        CU(cudaIpcOpenMemHandle(&p, allh[j * count + k], cudaIpcMemLazyEnablePeerAccess));
        (*all)[j * count + k] = p;
        opened->push_back(p);
      }
    }
  }
  return DFLOW_OK;
}

struct SymRegion {
  void* base = nullptr;
  ncclWindow_t win = nullptr;
  ncclDevComm dc{};
  bool dc_ok = false;
};

namespace {
__global__ void k_multimem_ptr(ncclWindow_t win, ncclDevComm dc, void** out) {
  *out = ncclGetLsaMultimemPointer(win, 0, dc);
}
}  // namespace

dflow_status comm_symmetric_alloc(dflow_session* s, size_t bytes, void** local, void** mc, SymRegion** out) {
  *local = *mc = nullptr;
  *out = nullptr;
  if (s->sim || !s->nccl) return fail(DFLOW_UNIMPLEMENTED, "symmetric memory needs an NCCL communicator");
  SymRegion* r = new SymRegion();
  ncclResult_t e = ncclMemAlloc(&r->base, bytes);
  if (e == ncclSuccess) e = ncclCommWindowRegister(s->nccl, r->base, bytes, &r->win, NCCL_WIN_COLL_SYMMETRIC);
  if (e == ncclSuccess) {
    ncclDevCommRequirements req{};
    req.lsaMultimem = true;
    e = ncclDevCommCreate(s->nccl, &req, &r->dc);
    r->dc_ok = e == ncclSuccess;
  }
  if (e != ncclSuccess) {
    comm_symmetric_free(s, r);
    return fail(DFLOW_NCCL, "symmetric window: %s", ncclGetErrorString(e));
  }
  void** d = nullptr;
  void* h = nullptr;
  if (cudaMalloc(&d, sizeof(void*)) == cudaSuccess) {
    k_multimem_ptr<<<1, 1, 0, s->comm>>>(r->win, r->dc, d);
    if (cudaMemcpyAsync(&h, d, sizeof(void*), cudaMemcpyDeviceToHost, s->comm) != cudaSuccess ||
        cudaStreamSynchronize(s->comm) != cudaSuccess)
      h = nullptr;
    cudaFree(d);
  }
  cudaGetLastError();
  *local = r->base;
  *mc = h;
  *out = r;
  return DFLOW_OK;
}

void comm_symmetric_free(dflow_session* s, SymRegion* r) {
  if (!r) return;
  if (r->dc_ok) ncclDevCommDestroy(s->nccl, &r->dc);
  if (r->win) ncclCommWindowDeregister(s->nccl, r->win);
  if (r->base) ncclMemFree(r->base);
  delete r;
}

dflow_status sim_run(dflow_sim_world* w, const std::function<dflow_status(int)>& fn) {
  const int N = w->world;
  std::vector<dflow_status> st(N, DFLOW_OK);
  std::vector<std::string> msg(N);
  std::vector<std::thread> th;
  th.reserve(N);
  for (int r = 0; r < N; ++r) {
    th.emplace_back([&, r] {
      if (cudaSetDevice(w->device) != cudaSuccess) {
        st[r] = DFLOW_CUDA;
        msg[r] = "cudaSetDevice failed";
        return;
      }
      st[r] = fn(r);
      if (st[r] != DFLOW_OK) msg[r] = dflow_last_error();
    });
  }
  for (auto& t : th) t.join();
  cudaSetDevice(w->device);
  const cudaError_t e = cudaStreamSynchronize(w->stream);
  for (int r = 0; r < N; ++r)
    if (st[r] != DFLOW_OK) return fail(st[r], "rank %d: %s", r, msg[r].c_str());
  if (e != cudaSuccess) return fail(DFLOW_CUDA, "simulated world stream: %s", cudaGetErrorString(e));
  return DFLOW_OK;
}

}  // namespace dflow
