// verify.cu -- G5 seeded input generation and G6 output comparison.
//
// Reference: difftest.sample_inputs (difftest.py:124-141) and the bit-exact
// ret_ptr compare of difftest.run_tests (difftest.py:158-204).  The paper
// verifies each accepted schedule over 10M random samples.
//
// * sip_sample_inputs: the reference's own stream -- random.Random(f"{seed}:{s}")
//   seeded through SHA-512 -- one device thread per sample.
// * sip_fill_normal: Philox4x32-10 + Box-Muller (16-bit uniforms) N(0, sigma^2) fp16/bf16 inputs for
//   the tcgen05 targets (the reference has no float path; extension).
// * sip_compare: HBM-bound compare of candidate vs baseline outputs: 16-byte
//   vector loads, grid-stride, warp-shuffle reductions, one atomic per warp.
#include <cuda_bf16.h>
#include <cuda_fp16.h>

#include <cstring>
#include <string>
#include <vector>

#include "common.h"
#include "rng.cuh"

namespace {

// ---- Philox4x32-10 -----------------------------------------------------
__device__ __forceinline__ uint4 philox(uint4 ctr, uint2 key) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    uint32_t hi0 = __umulhi(0xD2511F53u, ctr.x), lo0 = 0xD2511F53u * ctr.x;
    uint32_t hi1 = __umulhi(0xCD9E8D57u, ctr.z), lo1 = 0xCD9E8D57u * ctr.z;
    ctr = make_uint4(hi1 ^ ctr.y ^ key.x, lo1, hi0 ^ ctr.w ^ key.y, lo0);
    key.x += 0x9E3779B9u;
    key.y += 0xBB67AE85u;
  }
  return ctr;
}


// Box-Muller on one 32-bit word: high 16 bits -> u1 in (0, 1], low 16 bits -> angle
__device__ __forceinline__ float2 box_muller16(uint32_t w) {
  float u1 = ((w >> 16) + 1.0f) * (1.0f / 65536.0f);
  float u2 = (w & 0xFFFFu) * (1.0f / 65536.0f);
  float r = sqrtf(-2.0f * __logf(u1));
  float s, c;
  __sincosf(6.283185307179586f * u2, &s, &c);
  return make_float2(r * c, r * s);
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float a, float b);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&h);
}

template <typename T>
__global__ void fill_normal_kernel(T* out, size_t count, uint64_t seed, uint64_t stream, float sigma) {
  // One Philox4x32-10 block per 8 outputs: its 128 bits are eight 16-bit uniforms, i.e.
  // four Box-Muller pairs (u1 in (0, 1] from 16 bits bounds |x| <= 4.7 sigma, ample for
  // verification inputs).  One block per 16-byte store keeps the fill near HBM speed.
  size_t groups = (count + 7) / 8;  // 8 elements (16 bytes) per group
  uint2 key = make_uint2((uint32_t)seed, (uint32_t)(seed >> 32));
  for (size_t g = blockIdx.x * (size_t)blockDim.x + threadIdx.x; g < groups;
       g += (size_t)gridDim.x * blockDim.x) {
    uint4 r = philox(make_uint4((uint32_t)g, (uint32_t)(g >> 32), (uint32_t)stream,
                                (uint32_t)(stream >> 32)), key);
    float2 a = box_muller16(r.x), b = box_muller16(r.y), c = box_muller16(r.z), d = box_muller16(r.w);
    uint4 v = make_uint4(pack2<T>(a.x * sigma, a.y * sigma), pack2<T>(b.x * sigma, b.y * sigma),
                         pack2<T>(c.x * sigma, c.y * sigma), pack2<T>(d.x * sigma, d.y * sigma));
    size_t e = g * 8;
    if (e + 8 <= count) {
      *reinterpret_cast<uint4*>(out + e) = v;
    } else {
      const T* vv = reinterpret_cast<const T*>(&v);
      for (size_t i = 0; e + i < count; ++i) out[e + i] = vv[i];
    }
  }
}

// ---- compare -------------------------------------------------------------
struct CmpAcc {
  unsigned long long checked, mismatched, bitdiff, first;  // first = min failing element
  unsigned int max_err_bits;
};

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<__half>(__half v) { return __half2float(v); }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T>
__device__ __forceinline__ void cmp_elem(T a, T b, float atol, float rtol, size_t idx, int& mis,
                                         int& bits, float& err, unsigned long long& first,
                                         uint8_t* flags, int64_t eps, unsigned long long elem_base) {
  unsigned short ua = *reinterpret_cast<unsigned short*>(&a), ub = *reinterpret_cast<unsigned short*>(&b);
  if (ua == ub) return;
  ++bits;
  float fa = to_f(a), fb = to_f(b);
  bool an = fa != fa, bn = fb != fb;
  bool bad;
  if (an || bn) {
    bad = !(an && bn);
  } else {
    float d = fabsf(fa - fb);
    err = fmaxf(err, d);
    bad = !(d <= atol + rtol * fabsf(fa));
  }
  if (bad) {
    ++mis;
    if (idx + elem_base < first) first = idx + elem_base;
    flags[idx / eps] = 1;
  }
}

__device__ __forceinline__ unsigned long long warp_sum(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ unsigned long long warp_min(unsigned long long v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

template <typename T>
__global__ void __launch_bounds__(256) compare_kernel(const T* __restrict__ ref, const T* __restrict__ cand,
                                                      size_t count, float atol, float rtol, int64_t eps,
                                                      uint8_t* flags, CmpAcc* acc,
                                                      unsigned long long elem_base) {
  constexpr int kVec = 8;     // elements per 16-byte load
  constexpr int kUnroll = 4;  // independent 16-byte loads in flight per operand
  int mis = 0, bits = 0;
  float err = 0.f;
  unsigned long long first = ~0ull;
  size_t nvec = count / kVec;
  const uint4* r4 = reinterpret_cast<const uint4*>(ref);
  const uint4* c4 = reinterpret_cast<const uint4*>(cand);
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t tid = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (size_t base = tid; base < nvec; base += stride * kUnroll) {
    uint4 ra[kUnroll], ca[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t v = base + u * stride;
      if (v < nvec) {
        ra[u] = __ldcs(r4 + v);
        ca[u] = __ldcs(c4 + v);
      }
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      size_t v = base + u * stride;
      if (v >= nvec) continue;
      if (ra[u].x == ca[u].x && ra[u].y == ca[u].y && ra[u].z == ca[u].z && ra[u].w == ca[u].w) continue;
      const T* a = reinterpret_cast<const T*>(&ra[u]);
      const T* b = reinterpret_cast<const T*>(&ca[u]);
#pragma unroll
      for (int i = 0; i < kVec; ++i) cmp_elem(a[i], b[i], atol, rtol, v * kVec + i, mis, bits, err, first, flags, eps,
                                     elem_base);
    }
  }
  for (size_t e = nvec * kVec + tid; e < count; e += stride)  // tail
    cmp_elem(ref[e], cand[e], atol, rtol, e, mis, bits, err, first, flags, eps, elem_base);
  unsigned long long m = warp_sum((unsigned long long)mis), b = warp_sum((unsigned long long)bits);
  unsigned long long f = warp_min(first);
  float me = warp_max(err);
  if ((threadIdx.x & 31) == 0) {
    if (m) atomicAdd(&acc->mismatched, m);
    if (b) atomicAdd(&acc->bitdiff, b);
    if (f != ~0ull) atomicMin(&acc->first, f);
    if (me > 0.f) atomicMax(&acc->max_err_bits, __float_as_uint(me));
  }
}

__global__ void count_flags_kernel(const uint8_t* flags, size_t n, unsigned long long* out) {
  unsigned long long c = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    c += flags[i];
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

// ---- reference sample stream ------------------------------------------------
__device__ int fmt_i64(int64_t v, char* out) {
  char tmp[24];
  int n = 0, len = 0;
  uint64_t u = v < 0 ? (uint64_t)0 - (uint64_t)v : (uint64_t)v;
  do {
    tmp[n++] = (char)('0' + u % 10);
    u /= 10;
  } while (u);
  if (v < 0) out[len++] = '-';
  while (n) out[len++] = tmp[--n];
  return len;
}

__global__ void sample_inputs_kernel(const uint32_t* base, int64_t seed, int64_t first, int count, int nbuf,
                                     const int32_t* nbytes, const int32_t* cell, const int32_t* dist,
                                     int64_t stride, uint8_t* out) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  char str[48];
  int len = fmt_i64(seed, str);
  str[len++] = ':';
  len += fmt_i64(first + s, str + len);
  uint8_t buf[48 + 64];
  uint32_t key[32];
  int klen = sip::mt_key_from_bytes(reinterpret_cast<const uint8_t*>(str), len, buf, key);
  uint32_t state[sip::MT_N];
  sip::MtRef m{state, 1, 0};
  sip::mt_init_by_array(m, base, key, klen);
  uint8_t* dst = out + (size_t)s * stride;
  for (int k = 0; k < nbuf; ++k) {
    int nb = nbytes[k], c = cell[k];
    if (dist[k] == 2) {
      for (int i = 0; i < nb; ++i) dst[i] = 0;
    } else {
      int len_bytes = dist[k] == 1 ? nb / c : nb;  // "small": one byte per element
      int64_t bitsleft = 8 * (int64_t)len_bytes;
      for (int w = 0; bitsleft > 0; ++w, bitsleft -= 32) {
        uint32_t r = sip::mt_next(m);
        if (bitsleft < 32) r >>= (32 - bitsleft);
        for (int q = 0; q < 4; ++q) {
          int idx = 4 * w + q;
          if (idx >= len_bytes) break;
          uint8_t byte = (uint8_t)(r >> (8 * q));
          if (dist[k] == 1) {
            for (int z = 0; z < c; ++z) dst[idx * c + z] = 0;
            dst[idx * c] = byte & 0x0f;
          } else {
            dst[idx] = byte;
          }
        }
      }
    }
    dst += nb;
  }
}

}  // namespace

extern "C" {

int sip_fill_normal(sip_ctx* ctx, void* dev, size_t count, int32_t dtype, uint64_t seed,
                    uint64_t stream, float sigma) {
  if (!ctx || !dev) return SIP_E_ARG;
  if (count == 0) return SIP_OK;
  int blocks = ctx->sm_count * 8;
  if (dtype == 0)
    fill_normal_kernel<__half><<<blocks, 256, 0, ctx->stream>>>((__half*)dev, count, seed, stream, sigma);
  else if (dtype == 1)
    fill_normal_kernel<__nv_bfloat16><<<blocks, 256, 0, ctx->stream>>>((__nv_bfloat16*)dev, count, seed,
                                                                      stream, sigma);
  else
    return sip::fail(ctx, SIP_E_ARG, "dtype must be 0 (fp16) or 1 (bf16)");
  SIP_CHECK_LAUNCH(ctx);
  return SIP_OK;
}

int sip_compare(sip_ctx* ctx, const void* ref, const void* cand, size_t count, int32_t dtype,
                double atol, double rtol, int64_t elems_per_sample, int64_t first_sample,
                sip_cmp_result* out) {
  if (!ctx || !ref || !cand || !out || elems_per_sample < 1) return SIP_E_ARG;
  if ((reinterpret_cast<uintptr_t>(ref) | reinterpret_cast<uintptr_t>(cand)) & 15)
    return sip::fail(ctx, SIP_E_ARG, "buffers must be 16-byte aligned");
  size_t nsamples = (count + elems_per_sample - 1) / elems_per_sample;
  CmpAcc* acc = nullptr;
  uint8_t* flags = nullptr;
  unsigned long long* nfail = nullptr;
  SIP_CUDA(ctx, cudaMallocAsync(&acc, sizeof(CmpAcc), ctx->stream));
  SIP_CUDA(ctx, cudaMallocAsync(&flags, nsamples ? nsamples : 1, ctx->stream));
  SIP_CUDA(ctx, cudaMallocAsync(&nfail, sizeof(unsigned long long), ctx->stream));
  CmpAcc init{0, 0, 0, ~0ull, 0};
  SIP_CUDA(ctx, cudaMemcpyAsync(acc, &init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
  SIP_CUDA(ctx, cudaMemsetAsync(flags, 0, nsamples ? nsamples : 1, ctx->stream));
  SIP_CUDA(ctx, cudaMemsetAsync(nfail, 0, sizeof(unsigned long long), ctx->stream));
  int blocks = ctx->sm_count * 8;
  if (dtype == 0)
    compare_kernel<__half><<<blocks, 256, 0, ctx->stream>>>((const __half*)ref, (const __half*)cand, count,
                                                            (float)atol, (float)rtol, elems_per_sample, flags, acc,
                                                            0ull);
  else
    compare_kernel<__nv_bfloat16><<<blocks, 256, 0, ctx->stream>>>(
        (const __nv_bfloat16*)ref, (const __nv_bfloat16*)cand, count, (float)atol, (float)rtol,
        elems_per_sample, flags, acc, 0ull);
  SIP_CHECK_LAUNCH(ctx);
  count_flags_kernel<<<ctx->sm_count, 256, 0, ctx->stream>>>(flags, nsamples, nfail);
  SIP_CHECK_LAUNCH(ctx);
  CmpAcc h;
  unsigned long long nf = 0;
  SIP_CUDA(ctx, cudaMemcpyAsync(&h, acc, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  SIP_CUDA(ctx, cudaMemcpyAsync(&nf, nfail, sizeof nf, cudaMemcpyDeviceToHost, ctx->stream));
  cudaFreeAsync(acc, ctx->stream);
  cudaFreeAsync(flags, ctx->stream);
  cudaFreeAsync(nfail, ctx->stream);
  SIP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  out->checked_elems = (int64_t)count;
  out->mismatched_elems = (int64_t)h.mismatched;
  out->bitdiff_elems = (int64_t)h.bitdiff;
  out->failed_samples = (int64_t)nf;
  if (h.first != ~0ull) {
    out->first_fail_sample = first_sample + (int64_t)(h.first / elems_per_sample);
    out->first_fail_elem = (int64_t)(h.first % elems_per_sample);
  } else {
    out->first_fail_sample = -1;
    out->first_fail_elem = -1;
  }
  float me;
  std::memcpy(&me, &h.max_err_bits, sizeof me);
  out->max_abs_err = (double)me;
  return SIP_OK;
}

// ---- accumulating verification (no host synchronisation per batch) ----------
// One accumulator per verification run: every batch's compare adds into the same
// device counters, marks failing samples in a flag array indexed by the run's own
// sample counter, and tracks the first failure as a global element index
// (sample * elems_per_sample + element), so rank-strided batches merge by min.
}  // extern "C"

struct sip_verify_acc {
  sip_ctx* ctx;
  CmpAcc* acc;
  uint8_t* flags;
  unsigned long long* nfail;
  int64_t max_samples, eps, used;
};

extern "C" {

int sip_verify_open(sip_ctx* ctx, int64_t max_samples, int64_t elems_per_sample, sip_verify_acc** out) {
  if (!ctx || !out || max_samples < 1 || elems_per_sample < 1) return SIP_E_ARG;
  auto* a = new sip_verify_acc{ctx, nullptr, nullptr, nullptr, max_samples, elems_per_sample, 0};
  cudaError_t e = cudaMalloc(&a->acc, sizeof(CmpAcc));
  if (e == cudaSuccess) e = cudaMalloc(&a->flags, (size_t)max_samples);
  if (e == cudaSuccess) e = cudaMalloc(&a->nfail, sizeof(unsigned long long));
  if (e != cudaSuccess) {
    cudaFree(a->acc);
    cudaFree(a->flags);
    delete a;
    return sip::fail(ctx, SIP_E_CUDA, std::string("verify accumulator: ") + cudaGetErrorString(e));
  }
  CmpAcc init{0, 0, 0, ~0ull, 0};
  SIP_CUDA(ctx, cudaMemcpyAsync(a->acc, &init, sizeof init, cudaMemcpyHostToDevice, ctx->stream));
  SIP_CUDA(ctx, cudaMemsetAsync(a->flags, 0, (size_t)max_samples, ctx->stream));
  SIP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  *out = a;
  return SIP_OK;
}

int sip_verify_compare(sip_verify_acc* a, const void* ref, const void* cand, size_t count, int32_t dtype,
                       double atol, double rtol, int64_t first_sample) {
  if (!a || !ref || !cand || first_sample < 0) return SIP_E_ARG;
  sip_ctx* ctx = a->ctx;
  if ((reinterpret_cast<uintptr_t>(ref) | reinterpret_cast<uintptr_t>(cand)) & 15)
    return sip::fail(ctx, SIP_E_ARG, "buffers must be 16-byte aligned");
  const int64_t ns = (int64_t)((count + a->eps - 1) / a->eps);
  if (a->used + ns > a->max_samples) return sip::fail(ctx, SIP_E_ARG, "verify accumulator is full");
  const unsigned long long base = (unsigned long long)first_sample * (unsigned long long)a->eps;
  int blocks = ctx->sm_count * 8;
  if (dtype == 0)
    compare_kernel<__half><<<blocks, 256, 0, ctx->stream>>>((const __half*)ref, (const __half*)cand, count,
                                                            (float)atol, (float)rtol, a->eps,
                                                            a->flags + a->used, a->acc, base);
  else
    compare_kernel<__nv_bfloat16><<<blocks, 256, 0, ctx->stream>>>(
        (const __nv_bfloat16*)ref, (const __nv_bfloat16*)cand, count, (float)atol, (float)rtol, a->eps,
        a->flags + a->used, a->acc, base);
  SIP_CHECK_LAUNCH(ctx);
  a->used += ns;
  return SIP_OK;
}

int sip_verify_result(sip_verify_acc* a, sip_cmp_result* out) {
  if (!a || !out) return SIP_E_ARG;
  sip_ctx* ctx = a->ctx;
  SIP_CUDA(ctx, cudaMemsetAsync(a->nfail, 0, sizeof(unsigned long long), ctx->stream));
  if (a->used > 0) {
    count_flags_kernel<<<ctx->sm_count, 256, 0, ctx->stream>>>(a->flags, (size_t)a->used, a->nfail);
    SIP_CHECK_LAUNCH(ctx);
  }
  CmpAcc h;
  unsigned long long nf = 0;
  SIP_CUDA(ctx, cudaMemcpyAsync(&h, a->acc, sizeof h, cudaMemcpyDeviceToHost, ctx->stream));
  SIP_CUDA(ctx, cudaMemcpyAsync(&nf, a->nfail, sizeof nf, cudaMemcpyDeviceToHost, ctx->stream));
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess)
    return sip::fail(ctx, SIP_E_MEASURE, std::string("verification batch: ") + cudaGetErrorString(e));
  out->checked_elems = a->used * a->eps;
  out->mismatched_elems = (int64_t)h.mismatched;
  out->bitdiff_elems = (int64_t)h.bitdiff;
  out->failed_samples = (int64_t)nf;
  if (h.first != ~0ull) {
    out->first_fail_sample = (int64_t)(h.first / (unsigned long long)a->eps);
    out->first_fail_elem = (int64_t)(h.first % (unsigned long long)a->eps);
  } else {
    out->first_fail_sample = -1;
    out->first_fail_elem = -1;
  }
  float me;
  std::memcpy(&me, &h.max_err_bits, sizeof me);
  out->max_abs_err = (double)me;
  return SIP_OK;
}

int sip_verify_close(sip_verify_acc* a) {
  if (!a) return SIP_OK;
  cudaStreamSynchronize(a->ctx->stream);
  cudaFree(a->acc);
  cudaFree(a->flags);
  cudaFree(a->nfail);
  delete a;
  return SIP_OK;
}

static int sample_inputs_impl(sip_ctx* ctx, int64_t seed, int64_t first, int32_t count, int32_t nbuf,
                              const int32_t* nbytes, const int32_t* cell, const int32_t* dist, uint8_t* d_out,
                              int64_t* stride_out) {
  int64_t stride = 0;
  for (int k = 0; k < nbuf; ++k) {
    if (nbytes[k] < 0 || cell[k] < 1 || dist[k] < 0 || dist[k] > 2 || nbytes[k] % cell[k])
      return sip::fail(ctx, SIP_E_ARG, "bad buffer spec");
    stride += nbytes[k];
  }
  *stride_out = stride;
  if (count == 0) return SIP_OK;
  std::vector<uint32_t> base(sip::MT_N);
  sip::MtRef b{base.data(), 1, 0};
  sip::mt_init_genrand(b, 19650218u);
  uint32_t* d_base = nullptr;
  int32_t* d_spec = nullptr;
  SIP_CUDA(ctx, cudaMallocAsync(&d_base, sizeof(uint32_t) * sip::MT_N, ctx->stream));
  SIP_CUDA(ctx, cudaMallocAsync(&d_spec, sizeof(int32_t) * 3 * (nbuf ? nbuf : 1), ctx->stream));
  SIP_CUDA(ctx, cudaMemcpyAsync(d_base, base.data(), sizeof(uint32_t) * sip::MT_N, cudaMemcpyHostToDevice, ctx->stream));
  if (nbuf) {
    SIP_CUDA(ctx, cudaMemcpyAsync(d_spec, nbytes, sizeof(int32_t) * nbuf, cudaMemcpyHostToDevice, ctx->stream));
    SIP_CUDA(ctx, cudaMemcpyAsync(d_spec + nbuf, cell, sizeof(int32_t) * nbuf, cudaMemcpyHostToDevice, ctx->stream));
    SIP_CUDA(ctx, cudaMemcpyAsync(d_spec + 2 * nbuf, dist, sizeof(int32_t) * nbuf, cudaMemcpyHostToDevice, ctx->stream));
  }
  sample_inputs_kernel<<<(count + 63) / 64, 64, 0, ctx->stream>>>(d_base, seed, first, count, nbuf, d_spec,
                                                                 d_spec + nbuf, d_spec + 2 * nbuf, stride, d_out);
  SIP_CHECK_LAUNCH(ctx);
  cudaFreeAsync(d_base, ctx->stream);
  cudaFreeAsync(d_spec, ctx->stream);
  return SIP_OK;
}

int sip_sample_inputs(sip_ctx* ctx, int64_t seed, int64_t first, int32_t count, int32_t nbuf,
                      const int32_t* nbytes, const int32_t* cell, const int32_t* dist, uint8_t* out) {
  if (!ctx || count < 0 || nbuf < 0 || (nbuf && (!nbytes || !cell || !dist)) || (count && !out))
    return SIP_E_ARG;
  int64_t stride = 0;
  for (int k = 0; k < nbuf; ++k) stride += nbytes[k] > 0 ? nbytes[k] : 0;
  if (count == 0) return SIP_OK;
  uint8_t* d_out = nullptr;
  SIP_CUDA(ctx, cudaMallocAsync(&d_out, (size_t)count * (size_t)(stride ? stride : 1), ctx->stream));
  int rc = sample_inputs_impl(ctx, seed, first, count, nbuf, nbytes, cell, dist, d_out, &stride);
  if (rc == SIP_OK && stride)
    SIP_CUDA(ctx, cudaMemcpyAsync(out, d_out, (size_t)count * stride, cudaMemcpyDeviceToHost, ctx->stream));
  cudaFreeAsync(d_out, ctx->stream);
  SIP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return rc;
}

int sip_sample_inputs_device(sip_ctx* ctx, int64_t seed, int64_t first, int32_t count, int32_t nbuf,
                             const int32_t* nbytes, const int32_t* cell, const int32_t* dist, void* dev_out) {
  if (!ctx || count < 0 || nbuf < 0 || (nbuf && (!nbytes || !cell || !dist)) || (count && !dev_out))
    return SIP_E_ARG;
  int64_t stride = 0;
  int rc = sample_inputs_impl(ctx, seed, first, count, nbuf, nbytes, cell, dist, static_cast<uint8_t*>(dev_out),
                              &stride);
  if (rc != SIP_OK) return rc;
  SIP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

}  // extern "C"
