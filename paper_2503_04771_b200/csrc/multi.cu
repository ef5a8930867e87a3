// Multi-device entry points of the C ABI:
//   bgx_contract_sharded  one process drives an M- (or batch-) sharded
//                         contraction over several devices: one descriptor per
//                         slab, each launched on its own device and stream
//                         (asynchronous, so the devices overlap);
//   bgx_nccl_*            a communicator for the library's own collective,
//                         NCCL loaded at run time (dlopen: the copy torch
//                         already loaded, else the system libnccl.so.2);
//   bgx_ksplit_reduce     the K-split exchange: f32 partial sums of every rank
//                         reduced with ncclReduceScatter (row slab per rank) or
//                         ncclAllReduce over NVLink, then c0 added and cast
//                         (SURVEY §8e "NCCL ReduceScatter, fp32 ncclSum");
//   bgx_shutdown          drops the library's per-process state.
// Replaces nothing in the reference (bridgegen is single-threaded, one
// process, interp.py:407-420); this is the seam a multi-GPU bridgegen
// backend would bind next to interp.py:351-352.
#include "common.cuh"

#include <dlfcn.h>
#include <mutex>
#include <nccl.h>
#include <string.h>

namespace {

using namespace bgx;

// ---- NCCL, resolved at run time -------------------------------------------
struct Nccl {
  void *handle = nullptr;
  decltype(&ncclGetUniqueId) get_unique_id = nullptr;
  decltype(&ncclCommInitRank) comm_init_rank = nullptr;
  decltype(&ncclCommDestroy) comm_destroy = nullptr;
  decltype(&ncclReduceScatter) reduce_scatter = nullptr;
  decltype(&ncclAllReduce) all_reduce = nullptr;
  decltype(&ncclGetErrorString) error_string = nullptr;
  decltype(&ncclCommCount) comm_count = nullptr;
  decltype(&ncclCommUserRank) comm_user_rank = nullptr;
};

std::mutex g_nccl_mu;
Nccl g_nccl;
int g_live_comms = 0;

// Loads libnccl.so.2 once: RTLD_NOLOAD first, so a process that already has
// NCCL (torch's) keeps one copy; else the system library.
const Nccl *nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.handle) return &g_nccl;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    set_error("NCCL unavailable: %s", dlerror());
    return nullptr;
  }
  Nccl n;
  n.handle = h;
#define BGX_NCCL_SYM(field, name)                                       \
  n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, name));        \
  if (!n.field) {                                                       \
    set_error("NCCL symbol %s missing", name);                          \
    dlclose(h);                                                         \
    return nullptr;                                                     \
  }
  BGX_NCCL_SYM(get_unique_id, "ncclGetUniqueId")
  BGX_NCCL_SYM(comm_init_rank, "ncclCommInitRank")
  BGX_NCCL_SYM(comm_destroy, "ncclCommDestroy")
  BGX_NCCL_SYM(reduce_scatter, "ncclReduceScatter")
  BGX_NCCL_SYM(all_reduce, "ncclAllReduce")
  BGX_NCCL_SYM(error_string, "ncclGetErrorString")
  BGX_NCCL_SYM(comm_count, "ncclCommCount")
  BGX_NCCL_SYM(comm_user_rank, "ncclCommUserRank")
#undef BGX_NCCL_SYM
  g_nccl = n;
  return &g_nccl;
}

int nccl_fail(const Nccl *n, ncclResult_t r, const char *what) {
  set_error("%s failed: %s", what, n->error_string ? n->error_string(r) : "?");
  return BGX_ERR_CUDA;
}

// Restores the caller's current device on scope exit.
struct DeviceScope {
  int prev = -1;
  DeviceScope() { cudaGetDevice(&prev); }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

extern "C" {

int bgx_contract_sharded(const bgx_contract_desc *descs, const int32_t *devices,
                         void *const *streams, int32_t n) {
  BGX_CHECK_ARG(descs != nullptr && devices != nullptr && n >= 0,
                "bgx_contract_sharded: null descriptors or devices");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev <= 0) {
    set_error("bgx_contract_sharded: no CUDA device");
    return BGX_ERR_NO_DEVICE;
  }
  for (int32_t i = 0; i < n; ++i)
    if (devices[i] < 0 || devices[i] >= ndev) {
      set_error("bgx_contract_sharded: shard %d names device %d of %d", i, devices[i], ndev);
      return BGX_ERR_INVALID;
    }
  DeviceScope keep;
  for (int32_t i = 0; i < n; ++i) {
    if (cudaSetDevice(devices[i]) != cudaSuccess) {
      set_error("bgx_contract_sharded: cudaSetDevice(%d) failed", devices[i]);
      return BGX_ERR_CUDA;
    }
    const int rc = bgx_contract(&descs[i], streams ? streams[i] : nullptr);
    if (rc != BGX_OK) return rc;   // bgx_last_error() already says why
  }
  return BGX_OK;
}

int bgx_nccl_unique_id(void *id_out) {
  BGX_CHECK_ARG(id_out != nullptr, "bgx_nccl_unique_id: null output");
  const Nccl *n = nccl();
  if (!n) return BGX_ERR_UNSUPPORTED;
  ncclUniqueId id;
  const ncclResult_t r = n->get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail(n, r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof(id));
  return BGX_OK;
}

int bgx_nccl_comm_init(void **comm, int32_t world, int32_t rank, const void *id) {
  BGX_CHECK_ARG(comm != nullptr && id != nullptr && world >= 1 && rank >= 0 && rank < world,
                "bgx_nccl_comm_init: bad arguments");
  const Nccl *n = nccl();
  if (!n) return BGX_ERR_UNSUPPORTED;
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = n->comm_init_rank(&c, world, uid, rank);
  if (r != ncclSuccess) return nccl_fail(n, r, "ncclCommInitRank");
  *comm = c;
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  ++g_live_comms;
  return BGX_OK;
}

int bgx_nccl_comm_destroy(void *comm) {
  if (!comm) return BGX_OK;
  const Nccl *n = nccl();
  if (!n) return BGX_ERR_UNSUPPORTED;
  const ncclResult_t r = n->comm_destroy(static_cast<ncclComm_t>(comm));
  if (r != ncclSuccess) return nccl_fail(n, r, "ncclCommDestroy");
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  --g_live_comms;
  return BGX_OK;
}

int bgx_ksplit_reduce(const float *partial, void *out, const void *c0, int32_t out_dtype,
                      int64_t rows, int64_t cols, int32_t scatter, float *ws, void *comm,
                      void *stream) {
  BGX_CHECK_ARG(partial != nullptr && out != nullptr && comm != nullptr && rows >= 0 &&
                    cols >= 0,
                "bgx_ksplit_reduce: bad arguments");
  BGX_CHECK_ARG(out_dtype == BGX_F32 || out_dtype == BGX_BF16 || out_dtype == BGX_F16,
                "bgx_ksplit_reduce: out dtype must be f32/bf16/f16");
  const Nccl *n = nccl();
  if (!n) return BGX_ERR_UNSUPPORTED;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  int world = 1;
  ncclResult_t r = n->comm_count(c, &world);
  if (r != ncclSuccess) return nccl_fail(n, r, "ncclCommCount");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t total = rows * cols;
  if (scatter) {
    BGX_CHECK_ARG(rows % world == 0, "bgx_ksplit_reduce: rows %lld not divisible by world %d",
                  (long long)rows, world);
    const int64_t mine = total / world;
    // the reduced slab: straight into `out` when it is f32 without c0, else
    // into the caller's f32 workspace (mine elements) and cast from there
    const bool direct = out_dtype == BGX_F32 && c0 == nullptr;
    BGX_CHECK_ARG(direct || ws != nullptr, "bgx_ksplit_reduce: workspace needed for the cast");
    float *dst = direct ? static_cast<float *>(out) : ws;
    r = n->reduce_scatter(partial, dst, (size_t)mine, ncclFloat32, ncclSum, c, s);
    if (r != ncclSuccess) return nccl_fail(n, r, "ncclReduceScatter");
    return direct ? BGX_OK : bgx_cast_f32(dst, c0, out, out_dtype, mine, stream);
  }
  const bool direct = out_dtype == BGX_F32 && c0 == nullptr;
  BGX_CHECK_ARG(direct || ws != nullptr, "bgx_ksplit_reduce: workspace needed for the cast");
  float *dst = direct ? static_cast<float *>(out) : ws;
  r = n->all_reduce(partial, dst, (size_t)total, ncclFloat32, ncclSum, c, s);
  if (r != ncclSuccess) return nccl_fail(n, r, "ncclAllReduce");
  return direct ? BGX_OK : bgx_cast_f32(dst, c0, out, out_dtype, total, stream);
}

int bgx_shutdown(void) {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_live_comms > 0) {
    set_error("bgx_shutdown: %d NCCL communicator(s) still alive", g_live_comms);
    return BGX_ERR_INVALID;
  }
  if (g_nccl.handle) {
    dlclose(g_nccl.handle);
    g_nccl = Nccl{};
  }
  return BGX_OK;
}

}  // extern "C"
