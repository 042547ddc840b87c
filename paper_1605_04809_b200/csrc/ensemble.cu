// ensemble.cu - ensemble hook: one member model per GPU/process; per-word log-probs of the members
// are combined with an NCCL reduce over NVLink ("One or multiple models can be added
// to the Moses log-linear model as different instances of the same feature ... similar to
// ensemble translation"; north_star: "per-word probabilities are combined with an NCCL reduce").
//   mode 0 (log-linear, the paper's weighted features):  out = sum_m w_m log p_m
//   mode 1 (linear interpolation):                       out = log sum_m w_m p_m
// NCCL is resolved at run time (dlopen of the libnccl.so.2 that torch also uses) so that the
// library has no link-time NCCL dependency.
#include <dlfcn.h>

#include <string>

#include "internal.h"

namespace {
typedef struct ncclComm* ncclComm_t;
typedef struct {
  char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
constexpr int kNcclFloat32 = 7;
constexpr int kNcclSum = 0;

struct Nccl {
  void* h = nullptr;
  ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*reduce)(const void*, void*, size_t, int, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*allGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*getErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    // The NCCL that torch itself links (nvidia/nccl/lib in the Python environment) comes first: the
    // first libnccl.so.2 loaded in the process is the one every later user binds to by soname, so
    // loading an older system copy before torch would break torch's own import.
    const char* env = getenv("NMT_NCCL_LIB");  // set by the Python binding to torch's copy
    const char* cands[] = {env ? env : "", "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2",
                           "libnccl.so.2", "libnccl.so"};
    for (const char* c : cands)
      if (*c && (h = dlopen(c, RTLD_NOW | RTLD_LOCAL))) break;
    if (!h) return false;
    getUniqueId = (decltype(getUniqueId))dlsym(h, "ncclGetUniqueId");
    commInitRank = (decltype(commInitRank))dlsym(h, "ncclCommInitRank");
    reduce = (decltype(reduce))dlsym(h, "ncclReduce");
    commDestroy = (decltype(commDestroy))dlsym(h, "ncclCommDestroy");
    getErrorString = (decltype(getErrorString))dlsym(h, "ncclGetErrorString");
    allGather = (decltype(allGather))dlsym(h, "ncclAllGather");
    return getUniqueId && commInitRank && reduce && commDestroy;
  }
};
Nccl g_nccl;


__global__ void k_scale(const float* in, float* out, int n, float w, int mode) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = mode == 0 ? w * in[i] : w * expf(in[i]);
}
__global__ void k_log(float* x, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) x[i] = logf(x[i]);
}
}  // namespace

struct nmt_ensemble {
  int n, rank, device;
  ncclComm_t comm = nullptr;
  float* tmp = nullptr;
  int cap = 0;
};

extern "C" const char* nmt_last_error(void);
namespace nmt {
nmt_status set_error(nmt_status c, const std::string& m);

// vocab-parallel exchange (api.cu): all-gather of `count` floats per rank on the communicator
int ens_world(const nmt_ensemble* e) { return e->n; }
int ens_rank(const nmt_ensemble* e) { return e->rank; }
void ens_allgather(nmt_ensemble* e, const float* send, float* recv, size_t count, cudaStream_t st) {
  if (!g_nccl.allGather) throw NmtError(NMT_ERR_NCCL, "ncclAllGather not found");
  const ncclResult_t r = g_nccl.allGather(send, recv, count, kNcclFloat32, e->comm, st);
  if (r) throw NmtError(NMT_ERR_NCCL, std::string("ncclAllGather: ") + g_nccl.getErrorString(r));
}
}

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
  nmt_ensemble* e = new nmt_ensemble();
  e->n = n;
  e->rank = rank;
  e->device = device;
  ncclUniqueId id;
  memcpy(&id, uid, sizeof(id));
  ncclResult_t r = g_nccl.commInitRank(&e->comm, n, id, rank);
  if (r) {
    delete e;
    return nmt::set_error(NMT_ERR_NCCL, std::string("ncclCommInitRank: ") + g_nccl.getErrorString(r));
  }
  *out = e;
  return NMT_OK;
}

nmt_status nmt_ensemble_combine(nmt_ensemble* e, const float* in, int32_t n, float weight, int32_t mode, int32_t root,
                                float* out, void* stream) {
  if (!e || n < 0 || (n > 0 && !in) || (mode != 0 && mode != 1) || root < 0 || root >= e->n)
    return nmt::set_error(NMT_ERR_INVALID_ARG, "bad argument");
  if (n == 0) return NMT_OK;
  if (e->rank == root && !out) return nmt::set_error(NMT_ERR_INVALID_ARG, "out is NULL on the root");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (n > e->cap) {
    if (e->tmp) cudaFree(e->tmp);
    if (cudaMalloc(&e->tmp, (size_t)n * 4) != cudaSuccess) return nmt::set_error(NMT_ERR_OOM, "cudaMalloc");
    e->cap = n;
  }
  k_scale<<<(n + 255) / 256, 256, 0, st>>>(in, e->tmp, n, weight, mode);
  ncclResult_t r = g_nccl.reduce(e->tmp, e->rank == root ? out : e->tmp, (size_t)n, kNcclFloat32, kNcclSum, root,
                                 e->comm, st);
  if (r) return nmt::set_error(NMT_ERR_NCCL, std::string("ncclReduce: ") + g_nccl.getErrorString(r));
  if (mode == 1 && e->rank == root) k_log<<<(n + 255) / 256, 256, 0, st>>>(out, n);
  if (cudaGetLastError() != cudaSuccess) return nmt::set_error(NMT_ERR_CUDA, "ensemble kernel launch failed");
  return NMT_OK;
}

void nmt_ensemble_free(nmt_ensemble* e) {
  if (!e) return;
  if (e->comm) g_nccl.commDestroy(e->comm);
  if (e->tmp) cudaFree(e->tmp);
  delete e;
}

}  // extern "C"
