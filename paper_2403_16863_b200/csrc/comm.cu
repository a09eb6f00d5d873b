// comm.cu -- the per-epoch global-best exchange over NCCL (G9).
//
// Chains are independent (reference driver.py:73-79), so the only
// data-path collective is one per epoch: every rank contributes its champion
// (energy, seed) -- 24 bytes -- to an ncclAllGather, all ranks pick the same
// winner under the reference's ranking key (driver.py:81-85: best time, then
// seed; rank breaks exact duplicates) and the owner ncclBroadcasts the winning
// schedule (n u16) so every rank restarts its chains from it.
//
// NCCL is opened with dlopen("libnccl.so.2") at communicator creation: inside a
// process that already mapped torch's NCCL this resolves to that same copy
// (same soname), elsewhere to the system library.  libsip.so therefore has no
// link-time NCCL dependency and still loads on the CPU test tier.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "common.h"

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

template <typename F>
bool sym(void* h, const char* name, F** fn) {
  *fn = reinterpret_cast<F*>(dlsym(h, name));
  return *fn != nullptr;
}

NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("cannot open libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    api.ok = sym(h, "ncclGetUniqueId", &api.GetUniqueId) && sym(h, "ncclCommInitRank", &api.CommInitRank) &&
             sym(h, "ncclCommDestroy", &api.CommDestroy) && sym(h, "ncclAllGather", &api.AllGather) &&
             sym(h, "ncclBroadcast", &api.Broadcast) && sym(h, "ncclAllReduce", &api.AllReduce) &&
             sym(h, "ncclGetErrorString", &api.GetErrorString);
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

}  // namespace

struct sip_comm {
  sip_ctx* ctx = nullptr;
  ncclComm_t comm = nullptr;
  int nranks = 0, rank = 0;
  sip_best* d_rec = nullptr;  // [nranks] gathered records
  uint16_t* d_sched = nullptr;
  int sched_cap = 0;
  double* d_red = nullptr;
  int red_cap = 0;
};

#define SIP_NCCL(c, expr)                                                                   \
  do {                                                                                      \
    ncclResult_t r_ = (expr);                                                               \
    if (r_ != ncclSuccess)                                                                  \
      return ::sip::fail((c)->ctx, SIP_E_CUDA, std::string(#expr) + ": " + nccl().GetErrorString(r_)); \
  } while (0)

extern "C" {

int sip_comm_unique_id(uint8_t id[128]) {
  if (!id) return SIP_E_ARG;
  NcclApi& a = nccl();
  if (!a.ok) return SIP_E_CUDA;
  ncclUniqueId u;
  if (a.GetUniqueId(&u) != ncclSuccess) return SIP_E_CUDA;
  static_assert(sizeof(u) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return SIP_OK;
}

int sip_comm_create(sip_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank, sip_comm** out) {
  if (!ctx || !id || !out || nranks < 1 || rank < 0 || rank >= nranks) return SIP_E_ARG;
  *out = nullptr;
  NcclApi& a = nccl();
  if (!a.ok) return sip::fail(ctx, SIP_E_CUDA, a.why);
  SIP_CUDA(ctx, cudaSetDevice(ctx->device));
  auto* c = new sip_comm();
  c->ctx = ctx;
  c->nranks = nranks;
  c->rank = rank;
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  ncclResult_t r = a.CommInitRank(&c->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    delete c;
    return sip::fail(ctx, SIP_E_CUDA, std::string("ncclCommInitRank: ") + a.GetErrorString(r));
  }
  if (cudaMalloc(&c->d_rec, sizeof(sip_best) * (nranks + 1)) != cudaSuccess) {
    a.CommDestroy(c->comm);
    delete c;
    return sip::fail(ctx, SIP_E_CUDA, "cudaMalloc (exchange records)");
  }
  *out = c;
  return SIP_OK;
}

int sip_comm_destroy(sip_comm* c) {
  if (!c) return SIP_OK;
  cudaSetDevice(c->ctx->device);
  cudaStreamSynchronize(c->ctx->stream);
  if (c->comm) nccl().CommDestroy(c->comm);
  cudaFree(c->d_rec);
  cudaFree(c->d_sched);
  cudaFree(c->d_red);
  delete c;
  return SIP_OK;
}

int sip_nccl_exchange(sip_comm* c, const sip_best* mine, const uint16_t* sched_mine, int32_t n,
                      sip_best* all, sip_best* winner, uint16_t* sched_out) {
  if (!c || !mine || !winner || n < 0 || (n > 0 && (!sched_mine || !sched_out))) return SIP_E_ARG;
  sip_ctx* ctx = c->ctx;
  NcclApi& a = nccl();
  cudaStream_t st = ctx->stream;
  SIP_CUDA(ctx, cudaSetDevice(ctx->device));
  sip_best rec = *mine;
  rec.rank = c->rank;
  rec.pad = 0;
  sip_best* d_mine = c->d_rec + c->nranks;  // the send slot follows the gathered ones
  SIP_CUDA(ctx, cudaMemcpyAsync(d_mine, &rec, sizeof rec, cudaMemcpyHostToDevice, st));
  SIP_NCCL(c, a.AllGather(d_mine, c->d_rec, sizeof(sip_best), ncclUint8, c->comm, st));
  std::vector<sip_best> got(c->nranks);
  SIP_CUDA(ctx, cudaMemcpyAsync(got.data(), c->d_rec, sizeof(sip_best) * c->nranks, cudaMemcpyDeviceToHost, st));
  SIP_CUDA(ctx, cudaStreamSynchronize(st));
  // every rank applies the same key to the same records: (energy, seed, rank)
  int w = 0;
  for (int r = 1; r < c->nranks; ++r) {
    const sip_best& x = got[r];
    const sip_best& b = got[w];
    if (x.energy < b.energy || (x.energy == b.energy && (x.seed < b.seed || (x.seed == b.seed && x.rank < b.rank))))
      w = r;
  }
  *winner = got[w];
  if (all) std::memcpy(all, got.data(), sizeof(sip_best) * c->nranks);
  if (n > 0) {
    if (n > c->sched_cap) {
      cudaFree(c->d_sched);
      c->d_sched = nullptr;
      SIP_CUDA(ctx, cudaMalloc(&c->d_sched, sizeof(uint16_t) * n));
      c->sched_cap = n;
    }
    if (got[w].rank == c->rank)
      SIP_CUDA(ctx, cudaMemcpyAsync(c->d_sched, sched_mine, sizeof(uint16_t) * n, cudaMemcpyHostToDevice, st));
    SIP_NCCL(c, a.Broadcast(c->d_sched, c->d_sched, sizeof(uint16_t) * n, ncclUint8, got[w].rank, c->comm, st));
    SIP_CUDA(ctx, cudaMemcpyAsync(sched_out, c->d_sched, sizeof(uint16_t) * n, cudaMemcpyDeviceToHost, st));
    SIP_CUDA(ctx, cudaStreamSynchronize(st));
  }
  return SIP_OK;
}

int sip_comm_allreduce(sip_comm* c, double* vals, int32_t count, int32_t op) {
  if (!c || (count > 0 && !vals) || count < 0) return SIP_E_ARG;
  if (op != SIP_RED_SUM && op != SIP_RED_MAX && op != SIP_RED_MIN) return SIP_E_ARG;
  if (count == 0) return SIP_OK;
  sip_ctx* ctx = c->ctx;
  cudaStream_t st = ctx->stream;
  SIP_CUDA(ctx, cudaSetDevice(ctx->device));
  if (count > c->red_cap) {
    cudaFree(c->d_red);
    c->d_red = nullptr;
    SIP_CUDA(ctx, cudaMalloc(&c->d_red, sizeof(double) * count));
    c->red_cap = count;
  }
  const ncclRedOp_t rop = op == SIP_RED_SUM ? ncclSum : op == SIP_RED_MAX ? ncclMax : ncclMin;
  SIP_CUDA(ctx, cudaMemcpyAsync(c->d_red, vals, sizeof(double) * count, cudaMemcpyHostToDevice, st));
  SIP_NCCL(c, nccl().AllReduce(c->d_red, c->d_red, count, ncclFloat64, rop, c->comm, st));
  SIP_CUDA(ctx, cudaMemcpyAsync(vals, c->d_red, sizeof(double) * count, cudaMemcpyDeviceToHost, st));
  SIP_CUDA(ctx, cudaStreamSynchronize(st));
  return SIP_OK;
}

int sip_comm_barrier(sip_comm* c) {
  double one = 1.0;
  return sip_comm_allreduce(c, &one, 1, SIP_RED_SUM);
}

}  // extern "C"
