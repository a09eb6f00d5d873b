// targets_launch.cu -- launch descriptors (grid, smem, packed arguments with TMA
// tensor maps) for the shipped tuning-target cubins (targets/*.cu).  The
// evaluator launches whatever permutation of those cubins the search proposes
// with exactly these arguments.
#include <cstring>
#include <cstdlib>

#include "common.h"

namespace {

constexpr uint32_t kGemmOffsets[9] = {0, 128, 256, 384, 392, 396, 400, 404, 408};
constexpr uint32_t kGemmParamBytes = 412;
constexpr uint32_t kAttnOffsets[9] = {0, 128, 256, 384, 392, 396, 400, 404, 408};
constexpr uint32_t kAttnParamBytes = 412;

int encode(sip_ctx* ctx, CUtensorMap* map, const void* base, int rank, const cuuint64_t* dims,
           const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  cuuint32_t elem[5] = {1, 1, 1, 1, 1};
  CUresult r = ctx->cuTensorMapEncodeTiled(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, rank, const_cast<void*>(base),
                                           dims, strides_bytes, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return sip::fail(ctx, SIP_E_ARG, "cuTensorMapEncodeTiled failed");
  return SIP_OK;
}

}  // namespace

extern "C" {

int sip_target_gemm_launch(sip_ctx* ctx, const void* A, const void* B, void* C, int32_t M, int32_t N,
                           int32_t K, int32_t L, float slope, sip_launch* launch, void* params,
                           uint32_t params_cap) {
  if (!ctx || !A || !B || !C || !launch || !params || params_cap < kGemmParamBytes) return SIP_E_ARG;
  if (M <= 0 || N <= 0 || K <= 0 || L <= 0 || M % 256 || N % 256 || K % 64)
    return sip::fail(ctx, SIP_E_ARG, "gemm target needs M%256==0, N%256==0, K%64==0");
  uint8_t* p = static_cast<uint8_t*>(params);
  std::memset(p, 0, kGemmParamBytes);
  cuuint64_t da[3] = {(cuuint64_t)K, (cuuint64_t)M, (cuuint64_t)L};
  cuuint64_t sa[2] = {(cuuint64_t)K * 2, (cuuint64_t)M * K * 2};
  cuuint32_t ba[3] = {64, 128, 1};
  cuuint64_t db[3] = {(cuuint64_t)K, (cuuint64_t)N, (cuuint64_t)L};
  cuuint64_t sb[2] = {(cuuint64_t)K * 2, (cuuint64_t)N * K * 2};
  // each CTA of a pair stages half of the tile's B rows: 128-row boxes for 256-column
  // tiles, 64-row boxes for the 128-column tail halves
  cuuint32_t bb[3] = {64, 128, 1};
  cuuint32_t bh[3] = {64, 64, 1};
  int rc = encode(ctx, reinterpret_cast<CUtensorMap*>(p), A, 3, da, sa, ba);
  if (rc == SIP_OK) rc = encode(ctx, reinterpret_cast<CUtensorMap*>(p + 128), B, 3, db, sb, bb);
  if (rc == SIP_OK) rc = encode(ctx, reinterpret_cast<CUtensorMap*>(p + 256), B, 3, db, sb, bh);
  if (rc != SIP_OK) return rc;
  std::memcpy(p + 384, &C, 8);
  std::memcpy(p + 392, &M, 4);
  std::memcpy(p + 396, &N, 4);
  std::memcpy(p + 400, &K, 4);
  std::memcpy(p + 404, &L, 4);
  std::memcpy(p + 408, &slope, 4);
  // persistent CTA pairs (cta_group::2, one 256x256 tile each), one CTA per SM; problems
  // with at most half as many tiles as pairs run every tile as two halves (the kernel's Schedule)
  long pairs = (long)(M / 256) * (N / 256) * L;
  long cmax = ctx->sm_count / 2;
  long ncl = pairs >= cmax ? cmax : (2 * pairs <= cmax ? 2 * pairs : pairs);
  std::memset(launch, 0, sizeof *launch);
  launch->grid[0] = (uint32_t)(2 * ncl);
  launch->grid[1] = launch->grid[2] = 1;
  launch->block[0] = 192;
  launch->block[1] = launch->block[2] = 1;
  launch->cluster[0] = 2;  // CTA pairs (the kernel reads %cluster_ctarank)
  launch->cluster[1] = launch->cluster[2] = 1;
  launch->smem_bytes = 6 * (128 * 64 * 2 + 128 * 64 * 2) + 1024 + 256;  // 6 stages of 32 KB
  launch->params = params;
  launch->param_offsets = kGemmOffsets;
  launch->nparams = 9;
  launch->params_size = kGemmParamBytes;
  return SIP_OK;
}

int sip_target_attn_launch(sip_ctx* ctx, const void* Q, const void* K, const void* V, void* O, int32_t B,
                           int32_t H, int32_t S, int32_t D, float scale, sip_launch* launch, void* params,
                           uint32_t params_cap) {
  if (!ctx || !Q || !K || !V || !O || !launch || !params || params_cap < kAttnParamBytes) return SIP_E_ARG;
  if (B <= 0 || H <= 0 || S <= 0 || D != 128 || S % 256)
    return sip::fail(ctx, SIP_E_ARG, "attention target needs D == 128 and S % 256 == 0");
  uint8_t* p = static_cast<uint8_t*>(params);
  std::memset(p, 0, kAttnParamBytes);
  // [B*H][S][D]: 3-D maps, 64-column (128-byte, SWIZZLE_128B) boxes of 128 rows
  cuuint64_t dims[3] = {(cuuint64_t)D, (cuuint64_t)S, (cuuint64_t)B * H};
  cuuint64_t strides[2] = {(cuuint64_t)D * 2, (cuuint64_t)S * D * 2};
  cuuint32_t box[3] = {64, 128, 1};
  int rc = encode(ctx, reinterpret_cast<CUtensorMap*>(p), Q, 3, dims, strides, box);
  if (rc == SIP_OK) rc = encode(ctx, reinterpret_cast<CUtensorMap*>(p + 128), K, 3, dims, strides, box);
  if (rc == SIP_OK) rc = encode(ctx, reinterpret_cast<CUtensorMap*>(p + 256), V, 3, dims, strides, box);
  if (rc != SIP_OK) return rc;
  std::memcpy(p + 384, &O, 8);
  std::memcpy(p + 392, &B, 4);
  std::memcpy(p + 396, &H, 4);
  std::memcpy(p + 400, &S, 4);
  std::memcpy(p + 404, &D, 4);
  std::memcpy(p + 408, &scale, 4);
  std::memset(launch, 0, sizeof *launch);
  // persistent: one CTA per SM walks the (query-tile pair, head) items
  long items = (long)(S / 256) * B * H;
  long ctas = ctx->sm_count;
  // test hook: fewer persistent CTAs, so a small problem still runs several items per
  // CTA (carried K/V ring phases, o_free hand-offs) under compute-sanitizer
  if (const char* cap = std::getenv("SIP_ATTN_MAX_CTAS"))
    if (std::atol(cap) > 0 && std::atol(cap) < ctas) ctas = std::atol(cap);
  launch->grid[0] = (uint32_t)(items < ctas ? items : ctas);
  launch->grid[1] = 1;
  launch->grid[2] = 1;
  launch->block[0] = 512;  // TMA + MMA warps, 2 softmax warpgroups, 1 epilogue warpgroup
  launch->block[1] = launch->block[2] = 1;
  launch->cluster[0] = launch->cluster[1] = launch->cluster[2] = 1;
  // Q 2 tiles, K and V 2 stages each; 1 KB alignment slack; 256 B of mbarriers (+ the
  // TMEM slot); 1 KB of row sums handed from the softmax to the epilogue warps
  launch->smem_bytes = 6 * 128 * 128 * 2 + 1024 + 256 + 1024;
  launch->params = params;
  launch->param_offsets = kAttnOffsets;
  launch->nparams = 9;
  launch->params_size = kAttnParamBytes;
  return SIP_OK;
}

}  // extern "C"
