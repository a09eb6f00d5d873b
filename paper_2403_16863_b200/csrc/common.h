// common.h -- context, error plumbing and device-table structs shared by the
// libsip translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/sip.h"

struct sip_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  std::string err;
  int sm_count = 0;
  // L2 flush scratch (allocated on first use)
  void* flush_buf = nullptr;
  size_t flush_bytes = 0;
  // driver entry points resolved through cudaGetDriverEntryPoint (no -lcuda)
  CUresult (*cuModuleLoadData)(CUmodule*, const void*) = nullptr;
  CUresult (*cuModuleUnload)(CUmodule) = nullptr;
  CUresult (*cuModuleGetFunction)(CUfunction*, CUmodule, const char*) = nullptr;
  CUresult (*cuFuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  CUresult (*cuLaunchKernelEx)(const CUlaunchConfig*, CUfunction, void**, void**) = nullptr;
  CUresult (*cuGetErrorString)(CUresult, const char**) = nullptr;
  CUresult (*cuTensorMapEncodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                     const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                     const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                     CUtensorMapL2promotion, CUtensorMapFloatOOBfill) = nullptr;
  CUresult (*cuCtxGetCurrent)(CUcontext*) = nullptr;
  CUresult (*cuCtxSetCurrent)(CUcontext) = nullptr;
};

namespace sip {

int fail(sip_ctx* ctx, int code, const std::string& msg);

#define SIP_CUDA(ctx, expr)                                                               \
  do {                                                                                    \
    cudaError_t e_ = (expr);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return ::sip::fail((ctx), SIP_E_CUDA,                                               \
                         std::string(#expr) + ": " + cudaGetErrorString(e_));             \
  } while (0)

#define SIP_CHECK_LAUNCH(ctx) SIP_CUDA(ctx, cudaGetLastError())

// device copy of one listing's tables
struct KernelDev {
  int n = 0, words = 0, k = 0, nw32 = 0;
  uint2* meta = nullptr;        // (ctrl, lat) per identity
  uint8_t* klass = nullptr;
  uint64_t* reads = nullptr;
  uint64_t* writes = nullptr;
  sip_memref* refs = nullptr;
  uint8_t* nrefs = nullptr;
  uint8_t* cut = nullptr;       // [n+1]
  uint8_t* pin = nullptr;       // [n]
  uint64_t* guard = nullptr;    // [(n+1)*words] sm100 scoreboard-guard footprints, or null
  int32_t* cum = nullptr;       // [n] issue-cycle prefix sums of the listing (nvcc) order
  int16_t* gid = nullptr;       // identity -> global index (-1 = not a candidate)
  int32_t* gids = nullptr;      // global index -> identity
  uint32_t* e_after = nullptr;  // [k][nw32]  bit x = E(g, x)
  uint32_t* e_before = nullptr; // [k][nw32]  bit x = E(x, g)
};

}  // namespace sip

struct sip_kernel {
  sip_ctx* ctx = nullptr;
  sip::KernelDev d;
  int64_t baseline = 0;         // identity-schedule scoreboard total
  struct sip_chains* ws = nullptr;  // reusable chain workspace of sip_anneal_ex
  uint32_t* d_base = nullptr;   // MT19937 init_genrand(19650218) state
  void* d_epoch = nullptr;      // sip_epoch_result of the last sip_anneal_epoch
  struct sip_chains* spare = nullptr;  // a released result workspace kept for reuse
};
