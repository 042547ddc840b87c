// ensemble.cu - ensemble hook and the library's communicators ("One or multiple models
// can be added to the Moses log-linear model as different instances of the same feature ... similar
// to ensemble translation"; north_star: members on separate GPUs, per-word probabilities combined
// over NVLink).
//
// A communicator (nmt_ensemble) has one of two transports:
//  * NCCL: one member per process/GPU (nmt_ensemble_init; NCCL is dlopen'ed at run time, the same
//    libnccl.so.2 torch uses, so the library has no link-time NCCL dependency);
//  * local: all members in ONE process, one host thread per member, any devices (nmt_ensemble_init_local);
//    the exchange goes through a device buffer of the group, ordered by CUDA events and a host
//    barrier.  It runs several members (or vocab-parallel ranks) on one GPU, e.g. a 4-model
//    ensemble on fewer GPUs than members, and lets a single GPU execute every multi-rank code path.
// Both transports expose the same collective: an all-gather of `count` floats per rank.
//
// nmt_ensemble_combine = all-gather of each member's [log p (n floats) | weight] row, then ONE
// deterministic kernel on the root combines the members in member order (identical arithmetic for
// both transports):
//   mode 0 (log-linear, the paper's weighted features):  out = sum_m w_m log p_m
//   mode 1 (linear interpolation):                       out = mx + log sum_m w_m exp(log p_m - mx),
//                                                          mx = max_m log p_m  (cannot underflow)
#include <dlfcn.h>

#include <chrono>
#include <condition_variable>
#include <atomic>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "internal.h"

namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat32 = 7;

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  std::mutex mu;
  bool load() {
    std::lock_guard<std::mutex> lk(mu);
    if (h) return true;
    // The NCCL that torch itself links comes first (its path is passed by the Python binding in
    // NMT_NCCL_LIB): the first libnccl.so.2 loaded in the process is the one every later user binds
    // to by soname, so loading an older system copy before torch would break torch's own import.
    const char* env = getenv("NMT_NCCL_LIB");
    const char* cands[] = {env ? env : "", "libnccl.so.2", "libnccl.so"};
    for (const char* c : cands)
      if (*c && (h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return false;
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
    allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
    return getUniqueId && commInitRank && commDestroy && allGather && getErrorString;
  }
};
Nccl g_nccl;

// row m of `g` (stride floats) = [log p_m (n floats) | w_m | pad]; out[i] = combine over m in order
__global__ void k_ens_stage(const float* in, float* row, int n, float w) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) row[i] = in[i];
  if (i == 0) row[n] = w;
}
__global__ void k_ens_combine(const float* g, int world, size_t stride, int n, int mode, float* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (mode == 0) {
    double acc = 0.0;
    for (int m = 0; m < world; ++m) acc += (double)g[m * stride + n] * (double)g[m * stride + i];
    out[i] = (float)acc;
  } else {
    float mx = g[i];
    for (int m = 1; m < world; ++m) mx = fmaxf(mx, g[m * stride + i]);
    double s = 0.0;
    for (int m = 0; m < world; ++m) s += (double)g[m * stride + n] * exp((double)g[m * stride + i] - (double)mx);
    out[i] = (float)((double)mx + log(s));
  }
}

// one process, one host thread per member: a device buffer [world][count] + events + host barrier
struct LocalGroup {
  int world;
  std::vector<int> device;     // device of each rank
  std::mutex mu;
  std::condition_variable cv;
  int arrived = 0;
  long gen = 0;
  float* buf = nullptr;        // on device[0]; peers read/write it (same device, or P2P/UVA copies)
  size_t cap = 0;              // floats
  std::vector<cudaEvent_t> dep, done;
  std::atomic<bool> has_done{false};
  int refs = 0;
  explicit LocalGroup(int w) : world(w), device(w, 0), dep(w, nullptr), done(w, nullptr) {}
  // all `world` threads must arrive; a missing member (e.g. all members driven from one thread) is
  // reported instead of hanging
  void barrier() {
    std::unique_lock<std::mutex> lk(mu);
    const long g = gen;
    if (++arrived == world) {
      arrived = 0;
      ++gen;
      cv.notify_all();
      return;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(120), [&] { return gen != g; })) {
      --arrived;
      throw nmt::NmtError(NMT_ERR_INVALID_ARG,
                          "local communicator: not every member joined the collective within 120 s "
                          "(drive each member from its own host thread)");
    }
  }
};
}  // namespace

struct nmt_ensemble {
  int n, rank, device;
  ncclComm_t comm = nullptr;          // NCCL transport
  LocalGroup* local = nullptr;        // local transport (shared by the group's handles)
  float* gbuf = nullptr;              // combine: gathered rows [n][stride]
  size_t gcap = 0;
};

extern "C" const char* nmt_last_error(void);
namespace nmt {
nmt_status set_error(nmt_status c, const std::string& m);

int ens_world(const nmt_ensemble* e) { return e->n; }
int ens_rank(const nmt_ensemble* e) { return e->rank; }

// all-gather of `count` floats per rank: recv[q * count + i] = send_q[i] (recv may alias send's slot)
void ens_allgather(nmt_ensemble* e, const float* send, float* recv, size_t count, cudaStream_t st) {
  if (e->comm) {
    const ncclResult_t r = g_nccl.allGather(send, recv, count, kNcclFloat32, e->comm, st);
    if (r) throw NmtError(NMT_ERR_NCCL, std::string("ncclAllGather: ") + g_nccl.getErrorString(r));
    return;
  }
  LocalGroup* L = e->local;
  const int W = L->world, me = e->rank;
  L->barrier();  // everyone's previous copy-out is enqueued and its `done` event recorded
  if (me == 0 && L->cap < (size_t)W * count) {
    // (rare: first use or a larger message) every stream may still read the old buffer
    for (int q = 0; q < W; ++q) {
      CK(cudaSetDevice(L->device[q]));
      CK(cudaDeviceSynchronize());
    }
    CK(cudaSetDevice(L->device[0]));
    if (L->buf) CK(cudaFree(L->buf));
    L->buf = nullptr;
    CK(cudaMalloc(&L->buf, (size_t)W * count * sizeof(float)));
    L->cap = (size_t)W * count;
    CK(cudaSetDevice(e->device));
  }
  L->barrier();
  if (L->has_done)  // do not overwrite the buffer while a peer still copies the previous result out
    for (int q = 0; q < W; ++q) CK(cudaStreamWaitEvent(st, L->done[q], 0));
  CK(cudaMemcpyAsync(L->buf + (size_t)me * count, send, count * sizeof(float), cudaMemcpyDefault, st));
  CK(cudaEventRecord(L->dep[me], st));
  L->barrier();
  for (int q = 0; q < W; ++q)
    if (q != me) CK(cudaStreamWaitEvent(st, L->dep[q], 0));
  CK(cudaMemcpyAsync(recv, L->buf, (size_t)W * count * sizeof(float), cudaMemcpyDefault, st));
  CK(cudaEventRecord(L->done[me], st));
  L->barrier();  // every `done` is recorded before anyone waits on it in the next collective
  if (me == 0) L->has_done = true;
}
}  // namespace nmt

namespace {
nmt_status guard_ens(const std::function<void()>& f) {
  try {
    f();
    return NMT_OK;
  } catch (const nmt::NmtError& e) {
    return nmt::set_error(e.code, e.msg);
  } catch (const std::exception& e) {
    return nmt::set_error(NMT_ERR_INVALID_ARG, e.what());
  }
}
}  // namespace

extern "C" {

nmt_status nmt_ensemble_get_unique_id(void* out128) {
  if (!out128) return nmt::set_error(NMT_ERR_INVALID_ARG, "out is NULL");
  if (!g_nccl.load()) return nmt::set_error(NMT_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId id;
  ncclResult_t r = g_nccl.getUniqueId(&id);
  if (r) return nmt::set_error(NMT_ERR_NCCL, std::string("ncclGetUniqueId: ") + g_nccl.getErrorString(r));
  memcpy(out128, &id, sizeof(id));
  return NMT_OK;
}

nmt_status nmt_ensemble_init(int32_t n, int32_t rank, const void* uid, int32_t device, nmt_ensemble** out) {
  if (!uid || !out || n <= 0 || rank < 0 || rank >= n) return nmt::set_error(NMT_ERR_INVALID_ARG, "bad argument");
  if (!g_nccl.load()) return nmt::set_error(NMT_ERR_NCCL, "libnccl.so.2 not found");
  if (cudaSetDevice(device) != cudaSuccess) return nmt::set_error(NMT_ERR_CUDA, "cudaSetDevice failed");
  std::unique_ptr<nmt_ensemble> e(new nmt_ensemble());
  e->n = n;
  e->rank = rank;
  e->device = device;
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclResult_t r = g_nccl.commInitRank(&e->comm, n, id, rank);
  if (r) return nmt::set_error(NMT_ERR_NCCL, std::string("ncclCommInitRank: ") + g_nccl.getErrorString(r));
  *out = e.release();
  return NMT_OK;
}

nmt_status nmt_ensemble_init_local(int32_t n, const int32_t* devices, nmt_ensemble** out) {
  if (!out || n <= 0) return nmt::set_error(NMT_ERR_INVALID_ARG, "bad argument");
  return guard_ens([&] {
    LocalGroup* L = new LocalGroup(n);
    std::vector<std::unique_ptr<nmt_ensemble>> hs;
    try {
      for (int q = 0; q < n; ++q) {
        L->device[q] = devices ? devices[q] : 0;
        CK(cudaSetDevice(L->device[q]));
        CK(cudaEventCreateWithFlags(&L->dep[q], cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&L->done[q], cudaEventDisableTiming));
        hs.emplace_back(new nmt_ensemble());
        hs.back()->n = n;
        hs.back()->rank = q;
        hs.back()->device = L->device[q];
        hs.back()->local = L;
      }
    } catch (...) {
      for (int q = 0; q < n; ++q) {
        if (L->dep[q]) cudaEventDestroy(L->dep[q]);
        if (L->done[q]) cudaEventDestroy(L->done[q]);
      }
      delete L;
      throw;
    }
    L->refs = n;
    for (int q = 0; q < n; ++q) out[q] = hs[q].release();
  });
}

nmt_status nmt_ensemble_combine(nmt_ensemble* e, const float* in, int32_t n, float weight, int32_t mode, int32_t root,
                                float* out, void* stream) {
  if (!e || n < 0 || (n > 0 && !in) || (mode != 0 && mode != 1) || root < 0 || root >= e->n)
    return nmt::set_error(NMT_ERR_INVALID_ARG, "bad argument");
  if (n == 0) return NMT_OK;
  if (e->rank == root && !out) return nmt::set_error(NMT_ERR_INVALID_ARG, "out is NULL on the root");
  if (mode == 1 && !(weight >= 0.f)) return nmt::set_error(NMT_ERR_INVALID_ARG, "mode 1 needs a weight >= 0");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return guard_ens([&] {
    CK(cudaSetDevice(e->device));
    const size_t stride = ((size_t)n + 1 + 3) / 4 * 4;
    const size_t need = stride * (e->n + 1);  // slot `rank` is staged, then all rows are gathered
    if (need > e->gcap) {
      CK(cudaStreamSynchronize(st));
      if (e->gbuf) CK(cudaFree(e->gbuf));
      e->gbuf = nullptr;
      CK(cudaMalloc(&e->gbuf, need * sizeof(float)));
      e->gcap = need;
    }
    float* staged = e->gbuf + stride * e->n;
    nmt::note_launch();
    k_ens_stage<<<(n + 255) / 256, 256, 0, st>>>(in, staged, n, weight);
    CK(cudaGetLastError());
    nmt::ens_allgather(e, staged, e->gbuf, stride, st);
    if (e->rank == root) {
      nmt::note_launch();
      k_ens_combine<<<(n + 255) / 256, 256, 0, st>>>(e->gbuf, e->n, stride, n, mode, out);
      CK(cudaGetLastError());
    }
  });
}

void nmt_ensemble_free(nmt_ensemble* e) {
  if (!e) return;
  cudaSetDevice(e->device);
  if (e->comm) g_nccl.commDestroy(e->comm);
  if (e->gbuf) cudaFree(e->gbuf);
  if (LocalGroup* L = e->local) {
    bool last;
    {
      std::lock_guard<std::mutex> lk(L->mu);
      last = --L->refs == 0;
    }
    if (last) {
      for (int q = 0; q < L->world; ++q) {
        cudaSetDevice(L->device[q]);
        cudaDeviceSynchronize();
        cudaEventDestroy(L->dep[q]);
        cudaEventDestroy(L->done[q]);
      }
      if (L->buf) cudaFree(L->buf);
      delete L;
    }
  }
  delete e;
}

}  // extern "C"
