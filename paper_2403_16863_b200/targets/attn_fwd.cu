// attn_fwd.cu -- tuning target G8: fused attention forward, O = softmax(Q K^T * scale) V.
//
// The paper's attention workload, written by hand for
// sm_100a: fp16 [B, H, S, D=128] row-major Q/K/V/O, non-causal, fp32 softmax.
// One CTA per (256 query rows = two 128-row tiles A and B, head); 384 threads:
//   warp 0      TMA producer: Q_A, Q_B once, then K[t] / V[t] into 2-stage rings
//               (SWIZZLE_128B, two 64-column boxes per 128x128 tile)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, ping-ponging
//               the two tiles so one tile's softmax overlaps the other's MMAs:
//                 S_X     = Q_X K[t]^T          (SS: Q, K from shared memory)
//                 O_X    += P_X V[t]            (TS: P from tensor memory, V MN-major)
//               tcgen05.mma executes in issue order, so S_X(t+1) may be issued
//               right after PV_X(t) even though P_X(t) aliases S_X's columns.
//   warps 4-7   softmax of tile A, warps 8-11 softmax of tile B (one TMEM lane =
//               one query row per thread): tcgen05.ld the S row, exp2 with a lazily
//               updated running max (O and l rescaled only when the max grows by
//               more than 2^8; 1/4 of the exponentials on the FMA pipe), P packed
//               to fp16 and written back into the S
//               columns with tcgen05.st; epilogue O / l -> fp16 STG.
// TMEM: S_A | S_B | O_A | O_B = 4 x 128 columns.  Shared: Q 2x32 KB, K 2x32 KB,
// V 2x32 KB.
#include "sm100.cuh"

namespace {
constexpr int BM = 128, BN = 128, HD = 128;
constexpr int TILE_BYTES = BM * HD * 2;  // 32 KB (two 16 KB SWIZZLE_128B halves)
constexpr int HALF = TILE_BYTES / 2;
constexpr int NUM_THREADS = 384;
constexpr uint32_t IDESC_QK = sm100::idesc_f16(BM, BN);
constexpr uint32_t IDESC_PV = sm100::idesc_f16(BM, HD, false, true);  // B (V) MN-major
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain: p <= 256 before a rescale

// MN-major SWIZZLE_128B B operand: 64-element rows along N (=d) per K (=kv) row;
// LBO = stride between the two 64-wide d halves, SBO = stride between 8-row kv
// groups.  (The swapped encoding was measured wrong on a B200.)
__device__ __forceinline__ uint64_t desc_v(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr & 0x3FFFF) >> 4);
  d |= (uint64_t)(HALF >> 4) << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
// 2^x on the MUFU pipe (one MUFU.EX2)
__device__ __forceinline__ float ex2_mufu(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// 2^x on the FMA/ALU pipes (FA4-style offload): x = j + f, j = round(x), f in
// [-1/2, 1/2]; 2^f by a cubic fitted for relative error (max 2.9e-4, below the
// fp16 half-ulp of P); j is added to the exponent field.
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -126.f);
  const float magic = 12582912.f;  // 1.5 * 2^23: rounds to an integer in the low mantissa bits
  const float t = x + magic;
  const float f = x - (t - magic);
  const float p = fmaf(f, fmaf(f, fmaf(f, 0.05295114f, 0.24165067f), 0.6935366f), 1.f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}
}  // namespace

extern "C" __global__ void __launch_bounds__(NUM_THREADS, 1)
attn_fwd_f16(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
             const __grid_constant__ CUtensorMap tmV, __half* __restrict__ O, int B, int H, int S, int D,
             float scale) {
  using namespace sm100;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                  // tile A, tile B
  uint8_t* sK = sQ + 2 * TILE_BYTES;   // 2 stages
  uint8_t* sV = sK + 2 * TILE_BYTES;   // 2 stages
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + 2 * TILE_BYTES);
  uint64_t* q_full = bars;            // 1
  uint64_t* k_full = bars + 1;        // [2]
  uint64_t* k_empty = bars + 3;       // [2]
  uint64_t* v_full = bars + 5;        // [2]
  uint64_t* v_empty = bars + 7;       // [2]
  uint64_t* s_full = bars + 9;        // [tile]
  uint64_t* p_full = bars + 11;       // [tile]
  uint64_t* o_done = bars + 13;       // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 15);

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
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
    }
    mbar_fence_init();
  }
  if (warp == 1) tmem_alloc<512>(tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  auto tS = [&](int x) { return tmem + x * BN; };           // S_X (P_X aliases its first 64 columns)
  auto tO = [&](int x) { return tmem + 2 * BN + x * HD; };  // O_X

  if (warp == 0) {
    // ---------------- TMA producer ----------------
    if (elect_one()) {
      mbar_expect_tx(q_full, 2 * TILE_BYTES);
      for (int x = 0; x < 2; ++x) {
        tma_load_3d(sQ + x * TILE_BYTES, &tmQ, q_full, 0, (2 * qt + x) * BM, bh);
        tma_load_3d(sQ + x * TILE_BYTES + HALF, &tmQ, q_full, 64, (2 * qt + x) * BM, bh);
      }
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
    auto qk = [&](int x, int t) {  // S_X = Q_X K[t]^T
      const uint32_t q0 = smem_u32(sQ + x * TILE_BYTES), k0 = smem_u32(sK + (t & 1) * TILE_BYTES);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        mma_f16(tS(x), desc_sw128(q0 + (kk >> 2) * HALF + (kk & 3) * 32),
                desc_sw128(k0 + (kk >> 2) * HALF + (kk & 3) * 32), IDESC_QK, kk != 0);
      mma_commit(&s_full[x]);
    };
    auto pv = [&](int x, int t) {  // O_X += P_X V[t]; P_X: fp16 pairs in S_X's columns 0..63
      const uint32_t v0 = smem_u32(sV + (t & 1) * TILE_BYTES);
#pragma unroll
      for (int kk = 0; kk < BN / 16; ++kk)
        mma_f16_ts(tO(x), tS(x) + kk * 8, desc_v(v0 + kk * 16 * 128), IDESC_PV, (t | kk) != 0);
      mma_commit(&o_done[x]);
    };
    mbar_wait(q_full, 0);
    mbar_wait(&k_full[0], 0);
    tc_fence_after();
    if (elect_one()) {
      qk(0, 0);
      qk(1, 0);
      mma_commit(&k_empty[0]);
    }
    __syncwarp();
    for (int t = 0; t < T; ++t) {
      const int st = t & 1;
      const uint32_t ph = (t >> 1) & 1;
      const bool more = t + 1 < T;
      mbar_wait(&v_full[st], ph);
      if (more) mbar_wait(&k_full[st ^ 1], ((t + 1) >> 1) & 1);
      for (int x = 0; x < 2; ++x) {
        mbar_wait(&p_full[x], t & 1);  // softmax X wrote P_X(t) (and rescaled O_X)
        tc_fence_after();
        if (elect_one()) {
          pv(x, t);
          if (more) qk(x, t + 1);  // in-order after PV_X(t): safe to overwrite S_X / P_X
          if (x == 1) {
            mma_commit(&v_empty[st]);
            if (more) mma_commit(&k_empty[st ^ 1]);
          }
        }
        __syncwarp();
      }
    }
  } else if (warp >= 4) {
    // ---------------- softmax + epilogue: warps 4-7 tile A, 8-11 tile B ----------------
    const int x = (warp - 4) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * 1.4426950408889634f;
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < T; ++t) {
      mbar_wait(&s_full[x], t & 1);
      tc_fence_after();
      float s[BN];  // raw scores; the scale is folded into the exponent FFMA
#pragma unroll
      for (int c = 0; c < BN / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tS(x) + lane_off + c * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(v[j]);
      }
      float mq[8];  // 8 independent max chains instead of one 128-long dependency chain
#pragma unroll
      for (int q = 0; q < 8; ++q) mq[q] = s[q];
#pragma unroll
      for (int j = 8; j < BN; ++j) mq[j & 7] = fmaxf(mq[j & 7], s[j]);
      const float mx = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                             fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7]))) * sl2;
      float alpha = 1.f;
      const bool grow = mx > m_used + RESCALE_THRESHOLD;
      if (grow) {
        const float m_new = fmaxf(mx, m_used);
        alpha = exp2f(m_used - m_new);  // 0 on the first tile
        m_used = m_new;
      }
      float rq[4] = {0.f, 0.f, 0.f, 0.f};  // independent partial row sums
#pragma unroll
      for (int c = 0; c < BN / 64; ++c) {  // P -> tensor memory, 32 packed columns at a time
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float za = fmaf(s[c * 64 + 2 * j], sl2, -m_used), zb = fmaf(s[c * 64 + 2 * j + 1], sl2, -m_used);
          // one pair in four goes to the FMA pipe so MUFU is not the softmax bottleneck
          const float a = (j & 3) == 3 ? ex2_poly(za) : ex2_mufu(za);
          const float b = (j & 3) == 3 ? ex2_poly(zb) : ex2_mufu(zb);
          rq[j & 3] += a + b;
          pk[j] = pack_half2(a, b);
        }
        tmem_st32(tS(x) + lane_off + c * 32, pk);
      }
      l = l * alpha + ((rq[0] + rq[1]) + (rq[2] + rq[3]));
      // rescale O_X (rare): PV_X(t-1) must be complete; PV_X(t) waits for p_full below
      if (__any_sync(0xffffffffu, grow && t > 0)) {
        mbar_wait(&o_done[x], (t - 1) & 1);
        tc_fence_after();
        if (grow && t > 0) {
#pragma unroll 1
          for (int c = 0; c < HD / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(tO(x) + lane_off + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
            tmem_st32(tO(x) + lane_off + c * 32, v);
          }
        }
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[x]);
    }
    // epilogue: wait for the last PV_X, O / l -> fp16
    mbar_wait(&o_done[x], (T - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __half* orow = O + ((size_t)bh * S + (size_t)(2 * qt + x) * BM + row) * HD;
#pragma unroll 1
    for (int c = 0; c < HD / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tO(x) + lane_off + c * 32, v);
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
