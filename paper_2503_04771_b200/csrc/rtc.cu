// Runtime compilation for the GPU case study: CUDA C
// generated from bridgegen FIR/IR kernels (paper_2503_04771_b200/fir_gpu.py)
// is compiled here with NVRTC for sm_100a and launched for real, replacing
// the reference's sequential simulated thread grid (interp.py:434-461).
//
// NVRTC is loaded with dlopen so libbgx.so has no link-time dependency on it;
// the cubin is loaded with the context-independent library API
// (cudaLibraryLoadData / cudaLibraryGetKernel) and launched with
// cudaLaunchKernel.
#include "common.cuh"

#include <dlfcn.h>
#include <mutex>
#include <nvrtc.h>
#include <string.h>
#include <vector>

namespace bgx {
namespace {

struct Nvrtc {
  decltype(&nvrtcCreateProgram) create = nullptr;
  decltype(&nvrtcCompileProgram) compile = nullptr;
  decltype(&nvrtcGetProgramLogSize) log_size = nullptr;
  decltype(&nvrtcGetProgramLog) log = nullptr;
  decltype(&nvrtcGetCUBINSize) cubin_size = nullptr;
  decltype(&nvrtcGetCUBIN) cubin = nullptr;
  decltype(&nvrtcDestroyProgram) destroy = nullptr;
  decltype(&nvrtcGetErrorString) error = nullptr;
  bool ok = false;
};

const Nvrtc &nvrtc() {
  static Nvrtc n;
  static std::once_flag once;
  std::call_once(once, [] {
    const char *names[] = {"libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so.12", "libnvrtc.so"};
    void *h = nullptr;
    for (const char *nm : names)
      if ((h = dlopen(nm, RTLD_NOW | RTLD_LOCAL)) != nullptr) break;
    if (!h) return;
#define BGX_SYM(field, sym) n.field = reinterpret_cast<decltype(n.field)>(dlsym(h, #sym))
    BGX_SYM(create, nvrtcCreateProgram);
    BGX_SYM(compile, nvrtcCompileProgram);
    BGX_SYM(log_size, nvrtcGetProgramLogSize);
    BGX_SYM(log, nvrtcGetProgramLog);
    BGX_SYM(cubin_size, nvrtcGetCUBINSize);
    BGX_SYM(cubin, nvrtcGetCUBIN);
    BGX_SYM(destroy, nvrtcDestroyProgram);
    BGX_SYM(error, nvrtcGetErrorString);
#undef BGX_SYM
    n.ok = n.create && n.compile && n.log_size && n.log && n.cubin_size && n.cubin && n.destroy &&
           n.error;
  });
  return n;
}

struct RtcKernel {
  cudaLibrary_t lib;
  cudaKernel_t kern;
};

}  // namespace
}  // namespace bgx

using namespace bgx;

extern "C" int bgx_rtc_compile(const char *src, const char *name, void **handle, char *log,
                               int64_t log_len) {
  BGX_CHECK_ARG(src && name && handle, "bgx_rtc_compile: null argument");
  const Nvrtc &n = nvrtc();
  if (!n.ok) {
    set_error("bgx_rtc_compile: NVRTC (libnvrtc.so.12) not available");
    return BGX_ERR_UNSUPPORTED;
  }
  nvrtcProgram prog;
  if (n.create(&prog, src, "bgx_fir.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) {
    set_error("bgx_rtc_compile: nvrtcCreateProgram failed");
    return BGX_ERR_INVALID;
  }
  // exact IEEE arithmetic: no FMA contraction, no flush-to-zero, IEEE div/sqrt
  const char *opts[] = {"-arch=sm_100a", "--fmad=false", "-ftz=false", "-prec-div=true",
                        "-prec-sqrt=true", "-std=c++17", "-default-device"};
  nvrtcResult rc = n.compile(prog, (int)(sizeof(opts) / sizeof(opts[0])), opts);
  size_t lsz = 0;
  n.log_size(prog, &lsz);
  std::vector<char> lbuf(lsz + 1, 0);
  if (lsz) n.log(prog, lbuf.data());
  if (log && log_len > 0) {
    strncpy(log, lbuf.data(), (size_t)log_len - 1);
    log[log_len - 1] = 0;
  }
  if (rc != NVRTC_SUCCESS) {
    set_error("bgx_rtc_compile: %s: %.400s", n.error(rc), lbuf.data());
    n.destroy(&prog);
    return BGX_ERR_INVALID;
  }
  size_t csz = 0;
  n.cubin_size(prog, &csz);
  std::vector<char> cubin(csz);
  n.cubin(prog, cubin.data());
  n.destroy(&prog);
  RtcKernel *k = new RtcKernel();
  cudaError_t e = cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr,
                                      nullptr, 0);
  if (e != cudaSuccess) {
    set_error("bgx_rtc_compile: cudaLibraryLoadData: %s", cudaGetErrorString(e));
    delete k;
    return BGX_ERR_CUDA;
  }
  e = cudaLibraryGetKernel(&k->kern, k->lib, name);
  if (e != cudaSuccess) {
    set_error("bgx_rtc_compile: cudaLibraryGetKernel(%s): %s", name, cudaGetErrorString(e));
    cudaLibraryUnload(k->lib);
    delete k;
    return BGX_ERR_CUDA;
  }
  *handle = k;
  return BGX_OK;
}

extern "C" int bgx_rtc_launch(void *handle, uint64_t grid, uint32_t block, void **args,
                              void *stream) {
  BGX_CHECK_ARG(handle != nullptr, "bgx_rtc_launch: null handle");
  BGX_CHECK_ARG(block >= 1 && block <= 1024, "bgx_rtc_launch: block %u", block);
  BGX_CHECK_ARG(grid >= 1 && grid < 0x7fffffffULL, "bgx_rtc_launch: grid %llu",
                (unsigned long long)grid);
  RtcKernel *k = static_cast<RtcKernel *>(handle);
  BGX_CUDA_TRY(cudaLaunchKernel((const void *)k->kern, dim3((unsigned)grid), dim3(block), args, 0,
                                (cudaStream_t)stream));
  return BGX_OK;
}

extern "C" int bgx_rtc_free(void *handle) {
  if (!handle) return BGX_OK;
  RtcKernel *k = static_cast<RtcKernel *>(handle);
  cudaLibraryUnload(k->lib);
  delete k;
  return BGX_OK;
}
