// attn_fwd.cu -- tuning target G8: fused attention forward, O = softmax(Q K^T * scale) V.
//
// The paper's attention workload, written by hand for
// sm_100a: fp16 [B, H, S, D=128] row-major Q/K/V/O, non-causal, fp32 softmax.
// One CTA per (128-row query tile, head); 256 threads:
//   warp 0     TMA producer: Q once, then K[t] / V[t] into 2-stage rings
//              (SWIZZLE_128B, two 64-column boxes per 128x128 tile)
//   warp 1     TMEM allocator + single-thread tcgen05.mma issuer:
//                S[t%2]  = Q K[t]^T      (M128 N128 K16 x 8, K-major A and B)
//                O      += P[t-1] V[t-1] (M128 N128 K16 x 8, V as an MN-major B)
//              S is double-buffered in TMEM so Q K[t+1]^T overlaps softmax(t)
//   warps 4-7  softmax (one TMEM lane = one query row per thread): tcgen05.ld of
//              the S row, exp2 with a lazily updated running max (O and l are
//              rescaled only when the max grows by more than 2^8), P in fp16 to a
//              swizzled shared tile for the PV MMA; epilogue O / l -> fp16 STG.
// TMEM: S0 | S1 | O = 384 of 512 columns.  Shared: Q 32 KB, K 2x32 KB, V 2x32 KB,
// P 2x32 KB.
#include "sm100.cuh"

namespace {
constexpr int BM = 128, BN = 128, HD = 128;
constexpr int TILE_BYTES = BM * HD * 2;  // 32 KB (two 16 KB SWIZZLE_128B halves)
constexpr int HALF = TILE_BYTES / 2;
constexpr int NUM_THREADS = 256;
constexpr uint32_t IDESC_QK = sm100::idesc_f16(BM, BN);
constexpr uint32_t IDESC_PV = sm100::idesc_f16(BM, HD, false, true);  // B (V) MN-major
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain: p <= 256 before a rescale

// MN-major SWIZZLE_128B B operand: 64-element rows along N (=d) per K (=kv) row;
// LBO = stride between the two 64-wide d halves, SBO = stride between 8-row kv groups
__device__ __forceinline__ uint64_t desc_v(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
#ifndef SIP_VDESC_SWAP
  d |= (uint64_t)(HALF >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
#else
  d |= (uint64_t)(1024 >> 4) << 16;
  d |= (uint64_t)(HALF >> 4) << 32;
#endif
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void sts128(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
               : "memory");
}
}  // namespace

extern "C" __global__ void __launch_bounds__(NUM_THREADS, 1)
attn_fwd_f16(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, __half* __restrict__ O, int B, int H, int S, int D,
             float scale) {
  using namespace sm100;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + TILE_BYTES;      // 2 stages
  uint8_t* sV = sK + 2 * TILE_BYTES;  // 2 stages
  uint8_t* sP = sV + 2 * TILE_BYTES;  // 2 buffers
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * TILE_BYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* k_empty = bars + 3;  // [2]
  uint64_t* v_full = bars + 5;   // [2]
  uint64_t* v_empty = bars + 7;  // [2]
  uint64_t* s_full = bars + 9;   // [2]
  uint64_t* s_empty = bars + 11; // [2]
  uint64_t* p_full = bars + 13;  // [2]
  uint64_t* p_empty = bars + 15; // [2]
  uint64_t* o_done = bars + 17;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 18);

  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const int qt = blockIdx.x, bh = blockIdx.y;
  const int T = S / BN;

  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&s_empty[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&p_empty[i], 1);
    }
    mbar_init(o_done, 1);
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t tS = tmem, tO = tmem + 2 * BN;

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      mbar_expect_tx(q_full, TILE_BYTES);
      tma_load_3d(sQ, &tmQ, q_full, 0, qt * BM, bh);
      tma_load_3d(sQ + HALF, &tmQ, q_full, 64, qt * BM, bh);
      for (int t = 0; t < T; ++t) {
        const int st = t & 1;
        const uint32_t ph = (t >> 1) & 1;
        mbar_wait(&k_empty[st], ph ^ 1);
        mbar_expect_tx(&k_full[st], TILE_BYTES);
        tma_load_3d(sK + st * TILE_BYTES, &tmK, &k_full[st], 0, t * BN, bh);
        tma_load_3d(sK + st * TILE_BYTES + HALF, &tmK, &k_full[st], 64, t * BN, bh);
        mbar_wait(&v_empty[st], ph ^ 1);
        mbar_expect_tx(&v_full[st], TILE_BYTES);
        tma_load_3d(sV + st * TILE_BYTES, &tmV, &v_full[st], 0, t * BN, bh);
        tma_load_3d(sV + st * TILE_BYTES + HALF, &tmV, &v_full[st], 64, t * BN, bh);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer ----------------
    auto pv = [&](int u) {  // O += P[u] V[u]
      const int st = u & 1;
      const uint32_t ph = (u >> 1) & 1;
      mbar_wait(&p_full[st], ph);
      mbar_wait(&v_full[st], ph);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t p0 = smem_u32(sP + st * TILE_BYTES), v0 = smem_u32(sV + st * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < BN / 16; ++kk)
          mma_f16(tO, desc_sw128(p0 + (kk >> 2) * HALF + (kk & 3) * 32), desc_v(v0 + kk * 16 * 128), IDESC_PV,
                  (u | kk) != 0);
        mma_commit(&p_empty[st]);
        mma_commit(&v_empty[st]);
        mma_commit(o_done);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    for (int t = 0; t < T; ++t) {
      const int st = t & 1;
      const uint32_t ph = (t >> 1) & 1;
      mbar_wait(&k_full[st], ph);
      mbar_wait(&s_empty[st], ph ^ 1);
      tc_fence_after();
      if (elect_one()) {
        const uint32_t q0 = smem_u32(sQ), k0 = smem_u32(sK + st * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_f16(tS + st * BN, desc_sw128(q0 + (kk >> 2) * HALF + (kk & 3) * 32),
                  desc_sw128(k0 + (kk >> 2) * HALF + (kk & 3) * 32), IDESC_QK, kk != 0);
        mma_commit(&s_full[st]);
        mma_commit(&k_empty[st]);
      }
      __syncwarp();
      if (t > 0) pv(t - 1);
    }
    pv(T - 1);
  } else if (warp >= 4) {
    // ---------------- softmax + epilogue (warps 4..7) ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * 1.4426950408889634f;
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < T; ++t) {
      const int st = t & 1;
      const uint32_t ph = (t >> 1) & 1;
      mbar_wait(&s_full[st], ph);
      tc_fence_after();
      float s[BN];
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tS + st * BN + lane_off + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(v[j]) * sl2;
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[st]);  // S buffer may be overwritten by Q K[t+2]^T
      float mx = s[0];
#pragma unroll
      for (int j = 1; j < BN; ++j) mx = fmaxf(mx, s[j]);
      float alpha = 1.f;
      const bool grow = mx > m_used + RESCALE_THRESHOLD;
      if (grow) {
        const float m_new = fmaxf(mx, m_used);
        alpha = exp2f(m_used - m_new);  // 0 on the first tile
        m_used = m_new;
      }
      float rs = 0.f;
      uint32_t pk[BN / 2];
#pragma unroll
      for (int j = 0; j < BN / 2; ++j) {
        const float a = exp2f(s[2 * j] - m_used), b = exp2f(s[2 * j + 1] - m_used);
        rs += a + b;
        pk[j] = pack_half2(a, b);
      }
      l = l * alpha + rs;
      // P[t] -> shared (swizzled K-major A operand); buffer freed by PV(t-2)
      mbar_wait(&p_empty[st], ph ^ 1);
      const uint32_t pbase = smem_u32(sP + st * TILE_BYTES);
#pragma unroll
      for (int ch = 0; ch < BN / 8; ++ch) {  // 16-byte chunk ch holds kv columns 8ch..8ch+7
        const uint32_t half = ch >> 3, c16 = ch & 7;
        const uint32_t addr = pbase + half * HALF + row * 128 + ((c16 ^ (row & 7)) << 4);
        sts128(addr, pk[4 * ch], pk[4 * ch + 1], pk[4 * ch + 2], pk[4 * ch + 3]);
      }
      fence_async_smem();
      // rescale O (rare): needs PV(t-1) complete and must precede PV(t)
      bool any = __any_sync(0xffffffffu, grow && t > 0);
      if (any) {
        mbar_wait(o_done, (t - 1) & 1);
        tc_fence_after();
        if (grow && t > 0) {
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(tO + lane_off + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
            tmem_st32(tO + lane_off + c * 32, v);
          }
        }
        tmem_st_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[st]);
    }
    // epilogue: wait for the last PV, O / l -> fp16
    mbar_wait(o_done, (T - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __half* orow = O + ((size_t)bh * S + (size_t)qt * BM + row) * HD;
#pragma unroll 1
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tO + lane_off + c * 32, v);
      tmem_ld_wait();
      uint32_t h[16];
#pragma unroll
      for (int j = 0; j < 16; ++j)
        h[j] = pack_half2(__uint_as_float(v[2 * j]) * inv, __uint_as_float(v[2 * j + 1]) * inv);
      __half* dst = orow + c * 32;
      stg128(dst, h[0], h[1], h[2], h[3]);
      stg128(dst + 8, h[4], h[5], h[6], h[7]);
      stg128(dst + 16, h[8], h[9], h[10], h[11]);
      stg128(dst + 24, h[12], h[13], h[14], h[15]);
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}
