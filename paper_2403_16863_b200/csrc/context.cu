// context.cu -- sip_open / sip_close.  Driver-API entry points (module
// loading, cluster launches, tensor maps) are resolved at run time through
// cudaGetDriverEntryPoint, so libsip.so links only the static CUDA runtime and
// loads on machines without a driver (CPU test tier checks its exports).
#include "common.h"

namespace {

template <typename F>
bool resolve(const char* name, F** fn) {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || p == nullptr)
    return false;
  *fn = reinterpret_cast<F*>(p);
  return true;
}

}  // namespace

extern "C" {

int sip_open(int device, sip_ctx** out) {
  if (!out) return SIP_E_ARG;
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) return SIP_E_CUDA;
  if (device < 0 || device >= count) return SIP_E_ARG;
  if (cudaSetDevice(device) != cudaSuccess) return SIP_E_CUDA;
  cudaFree(nullptr);  // make the primary context current
  auto* ctx = new sip_ctx();
  ctx->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major < 10) {
    delete ctx;
    return SIP_E_CUDA;  // sm_100a only: no other architecture is supported
  }
  ctx->sm_count = prop.multiProcessorCount;
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess) {
    delete ctx;
    return SIP_E_CUDA;
  }
  bool ok = resolve("cuModuleLoadData", &ctx->cuModuleLoadData) &&
            resolve("cuModuleUnload", &ctx->cuModuleUnload) &&
            resolve("cuModuleGetFunction", &ctx->cuModuleGetFunction) &&
            resolve("cuFuncSetAttribute", &ctx->cuFuncSetAttribute) &&
            resolve("cuLaunchKernelEx", &ctx->cuLaunchKernelEx) &&
            resolve("cuGetErrorString", &ctx->cuGetErrorString) &&
            resolve("cuTensorMapEncodeTiled", &ctx->cuTensorMapEncodeTiled) &&
            resolve("cuCtxGetCurrent", &ctx->cuCtxGetCurrent) &&
            resolve("cuCtxSetCurrent", &ctx->cuCtxSetCurrent);
  if (!ok) {
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return SIP_E_CUDA;
  }
  *out = ctx;
  return SIP_OK;
}

int sip_close(sip_ctx* ctx) {
  if (!ctx) return SIP_OK;
  cudaSetDevice(ctx->device);
  if (ctx->flush_buf) cudaFree(ctx->flush_buf);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  delete ctx;
  return SIP_OK;
}

}  // extern "C"
