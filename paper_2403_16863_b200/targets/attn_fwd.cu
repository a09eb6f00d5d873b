// attn_fwd.cu -- tuning target G8: fused attention forward, O = softmax(Q K^T * scale) V.
//
// The paper's attention workload, written by hand for
// sm_100a: fp16 [B, H, S, D=128] row-major Q/K/V/O, non-causal, fp32 softmax.
//
// Persistent: one CTA per SM walks the work items (a pair of 128-row query tiles
// A and B of one head) with a static stride; K/V rings, mbarrier phases and TMEM
// stay live across items, so the next item's Q/K/V loads and first QK^T overlap
// the current item's last steps and its epilogue.  512 threads:
//   warp 0      TMA producer: per item K[0], Q_A and Q_B (once Q's smem is free),
//               V[0], then K[t] / V[t] through 2-stage rings (SWIZZLE_128B, two
//               64-column boxes per 128x128 tile)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer, ping-ponging
//               the two tiles so one tile's softmax overlaps the other's MMAs:
//                 S_X     = Q_X K[t]^T          (SS: Q, K from shared memory)
//                 O_X    += P_X V[t]            (TS: P from tensor memory, V MN-major),
//               issued in two 64-key halves as the softmax publishes them;
//               tcgen05.mma executes in issue order, so S_X(t+1) may be issued
//               right after PV_X(t) even though P_X(t) aliases S_X's columns.
//   warps 4-7   softmax of tile A, warps 8-11 softmax of tile B (one TMEM lane =
//               one query row per thread): tcgen05.ld the S row, exp2 with a lazily
//               updated running max (O and l rescaled only when the max grows by
//               more than 2^8; 3/8 of the exponentials on the FMA pipe; packed
//               FFMA2/FADD2 and 3-input FMNMX3), P packed to fp16 into S's columns
//               with tcgen05.st; at the end of an item the row sums go to shared memory.
//   warps 12-15 epilogue: O_X / l -> fp16 STG for both tiles, then O_X is released
//               to the next item's first PV.
// TMEM: S_A | S_B | O_A | O_B = 4 x 128 columns.  Shared: Q 2x32 KB, K 2x32 KB,
// V 2x32 KB, row sums 2 x 512 B.
#include "sm100.cuh"

namespace {
constexpr int BM = 128, BN = 128, HD = 128;
constexpr int TILE_BYTES = BM * HD * 2;  // 32 KB (two 16 KB SWIZZLE_128B halves)
constexpr int HALF = TILE_BYTES / 2;
constexpr int NUM_THREADS = 512;
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

// packed fp32x2 arithmetic (FFMA2 / FADD2) and the 3-input max (FMNMX3) of sm_100a:
// the softmax is issue- and MUFU-bound, so every element-wise op is done on pairs.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
        "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// 2^x for a pair on the FMA/ALU pipes (FA4-style offload): x = j + f, j = round(x),
// f in [-1/2, 1/2]; 2^f by a cubic fitted for relative error (max 2.9e-4, below the
// fp16 half-ulp of P); j is added to the exponent field with one IMAD per element.
__device__ __forceinline__ float2 ex2_poly2(float2 x) {
  const float magic = 12582912.f;  // 1.5 * 2^23: rounds to an integer in the low mantissa bits
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(magic, magic));
  const float2 j = fadd2(t, make_float2(-magic, -magic));
  const float2 f = ffma2(j, make_float2(-1.f, -1.f), x);
  float2 p = ffma2(f, make_float2(0.05295114f, 0.05295114f), make_float2(0.24165067f, 0.24165067f));
  p = ffma2(f, p, make_float2(0.6935366f, 0.6935366f));
  p = ffma2(f, p, make_float2(1.f, 1.f));
  return make_float2(__int_as_float(__float_as_int(t.x) * (1 << 23) + __float_as_int(p.x)),
                     __int_as_float(__float_as_int(t.y) * (1 << 23) + __float_as_int(p.y)));
}

// registers: the launch gives 512 x 128; warpgroups 0 (TMA, MMA) and 3 (epilogue) hand
// theirs to the two softmax warpgroups (128 x 56 + 128 x 72 + 256 x 192 = 64 K)
#define SIP_REGS_PRODUCER 56
#define SIP_REGS_EPILOGUE 72
#define SIP_REGS_SOFTMAX 192
#ifndef SIP_POLY8
#define SIP_POLY8 3  // pairs out of every 8 whose exponentials run on the FMA pipe
#endif
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
  uint64_t* q_full = bars;            // Q_A, Q_B of the item landed
  uint64_t* q_empty = bars + 1;       // last QK^T of the item done: Q's smem is free
  uint64_t* k_full = bars + 2;        // [2]
  uint64_t* k_empty = bars + 4;       // [2]
  uint64_t* v_full = bars + 6;        // [2]
  uint64_t* v_empty = bars + 8;       // [2]
  uint64_t* s_full = bars + 10;       // [tile]
  uint64_t* p_full = bars + 12;       // [tile][half]: P_X keys 0-63 / 64-127 in TMEM
  uint64_t* o_done = bars + 16;       // [tile] PV_X(t) complete (every step)
  uint64_t* o_full = bars + 18;       // [tile] the item's O_X is final
  uint64_t* o_free = bars + 20;       // [tile] the epilogue has read O_X out
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 24);
  float* lsum = reinterpret_cast<float*>(bars + 26);  // [tile][128]

  const int warp = warp_id();
  const int lane = threadIdx.x & 31;
  const int T = S / BN;
  const int qpairs = S / (2 * BM);
  const int items = qpairs * B * H;

  if (warp == 0 && elect_one()) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&k_full[i], 1);
      mbar_init(&k_empty[i], 1);
      mbar_init(&v_full[i], 1);
      mbar_init(&v_empty[i], 1);
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[2 * i], 4);  // the 4 softmax warps (one per lane quarter) of tile i
      mbar_init(&p_full[2 * i + 1], 4);
      mbar_init(&o_done[i], 1);
      mbar_init(&o_full[i], 1);
      mbar_init(&o_free[i], 4);      // the 4 epilogue warps
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

  if (warp < 4) {
    // setmaxnreg sits inside each role's branch so ptxas budgets each region separately
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(SIP_REGS_PRODUCER) : "memory");
    if (warp == 0) {
      // ---------------- TMA producer ----------------
      if (elect_one()) {
        int g = 0;  // global K/V step: ring stage g & 1, phase (g >> 1) & 1
        for (int w = blockIdx.x, it = 0; w < items; w += gridDim.x, ++it) {
          const int qt = w % qpairs, bh = w / qpairs;
          for (int t = 0; t < T; ++t, ++g) {
            const int st = g & 1;
            const uint32_t ph = (g >> 1) & 1;
            mbar_wait(&k_empty[st], ph ^ 1);
            mbar_expect_tx(&k_full[st], TILE_BYTES);
            tma_load_3d(sK + st * TILE_BYTES, &tmK, &k_full[st], 0, t * BN, bh);
            tma_load_3d(sK + st * TILE_BYTES + HALF, &tmK, &k_full[st], 64, t * BN, bh);
            if (t == 0) {  // Q of this item once the previous item's last QK^T is done
              if (it > 0) mbar_wait(q_empty, (it - 1) & 1);
              mbar_expect_tx(q_full, 2 * TILE_BYTES);
              for (int x = 0; x < 2; ++x) {
                tma_load_3d(sQ + x * TILE_BYTES, &tmQ, q_full, 0, (2 * qt + x) * BM, bh);
                tma_load_3d(sQ + x * TILE_BYTES + HALF, &tmQ, q_full, 64, (2 * qt + x) * BM, bh);
              }
            }
            mbar_wait(&v_empty[st], ph ^ 1);
            mbar_expect_tx(&v_full[st], TILE_BYTES);
            tma_load_3d(sV + st * TILE_BYTES, &tmV, &v_full[st], 0, t * BN, bh);
            tma_load_3d(sV + st * TILE_BYTES + HALF, &tmV, &v_full[st], 64, t * BN, bh);
          }
        }
      }
    } else if (warp == 1) {
      // ---------------- MMA issuer ----------------
      auto qk = [&](int x, int g) {  // S_X = Q_X K[g]^T
        const uint32_t q0 = smem_u32(sQ + x * TILE_BYTES), k0 = smem_u32(sK + (g & 1) * TILE_BYTES);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          mma_f16(tS(x), desc_sw128(q0 + (kk >> 2) * HALF + (kk & 3) * 32),
                  desc_sw128(k0 + (kk >> 2) * HALF + (kk & 3) * 32), IDESC_QK, kk != 0);
        mma_commit(&s_full[x]);
      };
      auto pv = [&](int x, int g, bool first, int h) {  // O_X += P_X V[g], keys 64h..64h+63
        const uint32_t v0 = smem_u32(sV + (g & 1) * TILE_BYTES);
#pragma unroll
        for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
          mma_f16_ts(tO(x), tS(x) + kk * 8, desc_v(v0 + kk * 16 * 128), IDESC_PV, !first || kk != 0);
        if (h == 1) mma_commit(&o_done[x]);
      };
      int g = 0;   // global step
      int gs = 0;  // global s_full / p_full step (same as g, kept for clarity)
      for (int w = blockIdx.x, it = 0; w < items; w += gridDim.x, ++it) {
        (void)w;
        // first QK^T of the item (S_X is free: in issue order after the previous PV_X)
        mbar_wait(q_full, it & 1);
        mbar_wait(&k_full[g & 1], (g >> 1) & 1);
        tc_fence_after();
        if (elect_one()) {
          qk(0, g);
          qk(1, g);
          mma_commit(&k_empty[g & 1]);
        }
        __syncwarp();
        for (int t = 0; t < T; ++t, ++g, ++gs) {
          const int st = g & 1;
          const uint32_t ph = (g >> 1) & 1;
          const bool more = t + 1 < T;
          mbar_wait(&v_full[st], ph);
          if (more) mbar_wait(&k_full[st ^ 1], ((g + 1) >> 1) & 1);
          for (int x = 0; x < 2; ++x) {
            if (t == 0 && it > 0) mbar_wait(&o_free[x], (it - 1) & 1);  // O_X read out
            // the first half of PV_X(t) starts while softmax X still exponentiates keys 64-127
            mbar_wait(&p_full[2 * x], gs & 1);  // keys 0-63 of P_X(t) written (O_X rescaled)
            tc_fence_after();
            if (elect_one()) pv(x, g, t == 0, 0);
            __syncwarp();
            mbar_wait(&p_full[2 * x + 1], gs & 1);
            tc_fence_after();
            if (elect_one()) {
              pv(x, g, t == 0, 1);
              if (more) {
                qk(x, g + 1);  // in-order after PV_X(t): safe to overwrite S_X / P_X
              } else {
                mma_commit(&o_full[x]);  // the item's O_X is final
                if (x == 1) mma_commit(q_empty);
              }
              if (x == 1) {
                mma_commit(&v_empty[st]);
                if (more) mma_commit(&k_empty[st ^ 1]);
              }
            }
            __syncwarp();
          }
        }
      }
    }
  } else if (warp < 12) {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SIP_REGS_SOFTMAX) : "memory");
    // ---------------- softmax: warps 4-7 tile A, 8-11 tile B ----------------
    const int x = (warp - 4) >> 2;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * 1.4426950408889634f;
    int g = 0;  // global step
    for (int w = blockIdx.x, it = 0; w < items; w += gridDim.x, ++it) {
      float m_used = -INFINITY, l = 0.f;
      for (int t = 0; t < T; ++t, ++g) {
        mbar_wait(&s_full[x], g & 1);
        tc_fence_after();
        float s[BN];  // raw scores; the scale is folded into the exponent FFMA2
        {
          uint32_t v[BN / 32][32];  // all loads in flight, one wait
#pragma unroll
          for (int c = 0; c < BN / 32; ++c) tmem_ld32(tS(x) + lane_off + c * 32, v[c]);
          tmem_ld_wait();
#pragma unroll
          for (int c = 0; c < BN / 32; ++c)
#pragma unroll
            for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(v[c][j]);
        }
        float mq[4];  // 4 independent FMNMX3 chains, two new scores per step
#pragma unroll
        for (int q = 0; q < 4; ++q) mq[q] = s[q];
#pragma unroll
        for (int j = 4; j < BN; j += 8)
#pragma unroll
          for (int q = 0; q < 4; ++q) mq[q] = max3(mq[q], s[j + 2 * q], s[j + 2 * q + 1]);
#ifdef SIP_DIAG_NOMATH  // diagnostic build (tools/upper_bound.py): no row max, no exponentials
        const float mx = 0.f;
        (void)mq;
#else
        const float mx = fmaxf(max3(mq[0], mq[1], mq[2]), mq[3]) * sl2;
#endif
        float alpha = 1.f;
        const bool grow = mx > m_used + RESCALE_THRESHOLD;
        if (grow) {
          const float m_new = fmaxf(mx, m_used);
          alpha = exp2f(m_used - m_new);  // 0 on the first step of an item
          m_used = m_new;
        }
        // rescale O_X (rare) before any P of this step is published: PV_X(t-1) must be
        // complete; the first half of PV_X(t) waits for p_full below.  tcgen05.ld/st are
        // warp-collective (.sync.aligned): every lane of a warp with a growing row runs the
        // loop, the others with alpha = 1 (x * 1 == x).  Guarding it per lane deadlocked
        // the kernel once rows grew often (inputs with sigma >= 2).
        const bool rescale = __any_sync(0xffffffffu, grow && t > 0);
        if (rescale) {
          mbar_wait(&o_done[x], (g - 1) & 1);
          tc_fence_after();
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
        const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m_used, -m_used);
        float2 rq[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};  // independent partial sums
#pragma unroll
        for (int c = 0; c < BN / 64; ++c) {  // P -> tensor memory, 32 packed columns (64 keys) at a time
          uint32_t pk[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const float2 z = ffma2(make_float2(s[c * 64 + 2 * j], s[c * 64 + 2 * j + 1]), sc2, nm2);
            float2 e;
#ifdef SIP_DIAG_NOMATH
            e = z;
#else
            if ((j & 7) < SIP_POLY8) {
              e = ex2_poly2(z);
            } else {
              e.x = ex2_mufu(z.x);
              e.y = ex2_mufu(z.y);
            }
#endif
            pk[j] = pack_half2(e.x, e.y);
            rq[j & 3] = fadd2(rq[j & 3], e);
          }
          tmem_st32(tS(x) + lane_off + c * 32, pk);
          // publish this half of P_X(t) (and, with it, any O rescale above)
          tmem_st_wait();
          // observe o_done's previous phase once per step (compute-sanitizer synccheck:
          // no unobserved phases).  S_X(t) completing implied PV_X of the previous step
          // had, tcgen05.mma running in issue order, so this returns at once; it must
          // precede the arrive that lets the next PV_X start.
          if (c == 0 && g > 0 && !rescale) mbar_wait(&o_done[x], (g - 1) & 1);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[2 * x + c]);
        }
        const float2 r2 = fadd2(fadd2(rq[0], rq[1]), fadd2(rq[2], rq[3]));
        l = l * alpha + (r2.x + r2.y);
      }
      // the item's row sums for the epilogue warps, handed over on named barrier 1 + x
      // (softmax warps arrive, epilogue warps sync: 256 threads).  The next item cannot
      // reach this point before the epilogue has synced and read them: its PV needs
      // o_free, which the epilogue sends after the read.
      lsum[x * BM + row] = l;
      asm volatile("bar.arrive %0, 256;" ::"r"(1 + x) : "memory");
    }
  } else {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(SIP_REGS_EPILOGUE) : "memory");
    // ---------------- epilogue: warps 12-15, O / l -> fp16 for both tiles ----------------
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    for (int w = blockIdx.x, it = 0; w < items; w += gridDim.x, ++it) {
      const int qt = w % qpairs, bh = w / qpairs;
      for (int x = 0; x < 2; ++x) {
        asm volatile("bar.sync %0, 256;" ::"r"(1 + x) : "memory");  // row sums of tile x
        mbar_wait(&o_full[x], it & 1);
        tc_fence_after();
        const float inv = 1.f / lsum[x * BM + row];
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
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&o_free[x]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}
