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
//               more than 2^8; 3/8 of the exponentials on the FMA pipe; packed
//               FFMA2/FADD2 and 3-input FMNMX3 for the element-wise work), P packed
//               to fp16 and written back into the S
//               columns with tcgen05.st; epilogue O / l -> fp16 STG.
// TMEM: S_A | S_B | O_A | O_B = 4 x 128 columns.  Shared: Q 2x32 KB, K 2x32 KB,
// V 2x32 KB.
#include "sm100.cuh"

namespace {
constexpr int BM = 128, BN = 128, HD = 128;
constexpr int TILE_BYTES = BM * HD * 2;  // 32 KB (two 16 KB SWIZZLE_128B halves)
constexpr int HALF = TILE_BYTES / 2;
constexpr int NUM_THREADS_FOR_SPLIT(int split) { return 128 + 2 * 128 * split; }
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

#ifndef SIP_SPLIT
// softmax warps per query row (each takes BN / SIP_SPLIT score columns).  2 (640 threads,
// partial maxima exchanged through shared memory) was measured 3-7 % slower on a B200
// than 1, so the launcher (targets_launch.cu) uses 1 warp per row / 384 threads.
#define SIP_SPLIT 1
#endif
#if SIP_SPLIT == 1
#define SIP_REGS_LOW 56    // warpgroup 0 after setmaxnreg.dec
#define SIP_REGS_HIGH 224  // softmax warpgroups: 128 x 56 + 256 x 224 = 64 K registers
#else
// setmaxnreg.inc only draws on registers this CTA released with .dec: the launch gives
// 640 x 96 = 61440, and 128 x 32 + 512 x 112 = 61440
#define SIP_REGS_LOW 32
#define SIP_REGS_HIGH 112
#endif
#ifndef SIP_POLY8
#define SIP_POLY8 3  // pairs out of every 8 whose exponentials run on the FMA pipe
#endif
constexpr int SPLIT = SIP_SPLIT;
constexpr int CW = BN / SPLIT;       // score columns per softmax thread
constexpr int OW = HD / SPLIT;       // output columns per softmax thread (rescale, epilogue)
constexpr int NUM_THREADS = NUM_THREADS_FOR_SPLIT(SPLIT);
static_assert(CW % 64 == 0 && OW % 32 == 0, "column split");
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
  uint64_t* p_full = bars + 11;       // [tile][half]: P_X keys 0-63 / 64-127 in TMEM
  uint64_t* o_done = bars + 15;       // [tile]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 17);
  float* xch = reinterpret_cast<float*>(bars + 18);  // [tile][parity][SPLIT][128] row maxima / sums

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
      mbar_init(&p_full[2 * i], 4);  // the 4 warps (one per lane quarter) owning that half
      mbar_init(&p_full[2 * i + 1], 4);
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

  // registers: warpgroup 0 (TMA, MMA, two idle warps) gives most of its budget to the
  // two softmax warpgroups, whose 128 live scores plus packed P exceed 168.  Each
  // setmaxnreg sits inside its role's branch so ptxas budgets each region separately.
  if (warp < 4) {
#ifndef SIP_NO_SETMAXNREG
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(SIP_REGS_LOW) : "memory");
#endif
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
    auto pv = [&](int x, int t, int h) {  // O_X += P_X V[t], keys 64h..64h+63 (P columns 32h..)
      const uint32_t v0 = smem_u32(sV + (t & 1) * TILE_BYTES);
#pragma unroll
      for (int kk = 4 * h; kk < 4 * h + 4; ++kk)
        mma_f16_ts(tO(x), tS(x) + kk * 8, desc_v(v0 + kk * 16 * 128), IDESC_PV, (t | kk) != 0);
      if (h == 1) mma_commit(&o_done[x]);
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
        // the first half of PV_X(t) starts while softmax X still exponentiates keys 64-127
        mbar_wait(&p_full[2 * x], t & 1);  // keys 0-63 of P_X(t) written (O_X rescaled)
        tc_fence_after();
        if (elect_one()) pv(x, t, 0);
        __syncwarp();
        mbar_wait(&p_full[2 * x + 1], t & 1);
        tc_fence_after();
        if (elect_one()) {
          pv(x, t, 1);
          if (more) qk(x, t + 1);  // in-order after PV_X(t): safe to overwrite S_X / P_X
          if (x == 1) {
            mma_commit(&v_empty[st]);
            if (more) mma_commit(&k_empty[st ^ 1]);
          }
        }
        __syncwarp();
      }
    }
  }
  } else {
#ifndef SIP_NO_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(SIP_REGS_HIGH) : "memory");
#endif
    // ---------------- softmax + epilogue ----------------
    // warps 4.. : tile x = (warp-4) / (4*SPLIT); column part hh = ((warp-4)/4) % SPLIT;
    // warp & 3 is the TMEM lane quarter (query rows 32*q .. 32*q+31).  With SPLIT = 2 the
    // two warps of a row exchange their partial maxima through shared memory so both
    // take the same (lazy) max and rescale decision.
    const int sw = warp - 4;
    const int x = sw / (4 * SPLIT);
    const int hh = (sw >> 2) % SPLIT;
    const int quarter = warp & 3;
    const int row = quarter * 32 + lane;
    const uint32_t lane_off = (uint32_t)(quarter * 32) << 16;
    const float sl2 = scale * 1.4426950408889634f;
    auto pair_sync = [&]() {  // the SPLIT warps sharing these 32 rows
      if (SPLIT > 1) asm volatile("bar.sync %0, %1;" ::"r"(1 + x * 4 + quarter), "r"(32 * SPLIT) : "memory");
    };
    float m_used = -INFINITY, l = 0.f;
    for (int t = 0; t < T; ++t) {
      mbar_wait(&s_full[x], t & 1);
      tc_fence_after();
      float s[CW];  // raw scores; the scale is folded into the exponent FFMA2
      {
        uint32_t v[CW / 32][32];  // all loads in flight, one wait
#pragma unroll
        for (int c = 0; c < CW / 32; ++c) tmem_ld32(tS(x) + lane_off + hh * CW + c * 32, v[c]);
        tmem_ld_wait();
#pragma unroll
        for (int c = 0; c < CW / 32; ++c)
#pragma unroll
          for (int j = 0; j < 32; ++j) s[c * 32 + j] = __uint_as_float(v[c][j]);
      }
      float mq[4];  // 4 independent FMNMX3 chains, two new scores per step
#pragma unroll
      for (int q = 0; q < 4; ++q) mq[q] = s[q];
#pragma unroll
      for (int j = 4; j < CW; j += 8)
#pragma unroll
        for (int q = 0; q < 4; ++q) mq[q] = max3(mq[q], s[j + 2 * q], s[j + 2 * q + 1]);
      float mx = fmaxf(max3(mq[0], mq[1], mq[2]), mq[3]);
      if (SPLIT > 1) {
        // every S column of this row is in registers (tmem_ld_wait above) before the
        // barrier, so no warp overwrites S with P while its partner still reads it
        float* slot = xch + ((x * 2 + (t & 1)) * SPLIT) * 128;
        slot[hh * 128 + row] = mx;
        pair_sync();
#pragma unroll
        for (int k = 0; k < SPLIT; ++k) mx = fmaxf(mx, slot[k * 128 + row]);
      }
      mx *= sl2;
      float alpha = 1.f;
      const bool grow = mx > m_used + RESCALE_THRESHOLD;
      if (grow) {
        const float m_new = fmaxf(mx, m_used);
        alpha = exp2f(m_used - m_new);  // 0 on the first tile
        m_used = m_new;
      }
      // rescale O_X (rare) before any P of this step is published: PV_X(t-1) must be
      // complete; the first half of PV_X(t) waits for p_full below
      // rescale O_X (rare) before any P of this step is published: PV_X(t-1) must be
      // complete; the first half of PV_X(t) waits for p_full below
      const bool rescale = __any_sync(0xffffffffu, grow && t > 0);
      if (rescale) {
        mbar_wait(&o_done[x], (t - 1) & 1);
        tc_fence_after();
        if (grow && t > 0) {
#pragma unroll 1
          for (int c = 0; c < OW / 32; ++c) {
            uint32_t v[32];
            tmem_ld32(tO(x) + lane_off + hh * OW + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __float_as_uint(__uint_as_float(v[j]) * alpha);
            tmem_st32(tO(x) + lane_off + hh * OW + c * 32, v);
          }
        }
      }
      const float2 sc2 = make_float2(sl2, sl2), nm2 = make_float2(-m_used, -m_used);
      float2 rq[4] = {{0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}, {0.f, 0.f}};  // independent partial sums
#pragma unroll
      for (int c = 0; c < CW / 64; ++c) {  // P -> tensor memory, 32 packed columns (64 keys) at a time
        uint32_t pk[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const float2 z = ffma2(make_float2(s[c * 64 + 2 * j], s[c * 64 + 2 * j + 1]), sc2, nm2);
          float2 e;
          if ((j & 7) < SIP_POLY8) {
            e = ex2_poly2(z);
          } else {
            e.x = ex2_mufu(z.x);
            e.y = ex2_mufu(z.y);
          }
          pk[j] = pack_half2(e.x, e.y);
          rq[j & 3] = fadd2(rq[j & 3], e);
        }
        tmem_st32(tS(x) + lane_off + hh * (CW / 2) + c * 32, pk);
        // publish this half of P_X(t) (and, with it, any O rescale above)
        tmem_st_wait();
        // observe o_done's phase t-1 once per step (synccheck: no unobserved phases).
        // S_X(t) completing implied PV_X(t-1) had, tcgen05.mma running in issue order,
        // so this returns at once; it must precede the arrive that lets PV_X(t) start.
        if (c == 0 && t > 0 && !rescale) mbar_wait(&o_done[x], (t - 1) & 1);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[2 * x + hh * (CW / 64) + c]);
      }
      const float2 r2 = fadd2(fadd2(rq[0], rq[1]), fadd2(rq[2], rq[3]));
      l = l * alpha + (r2.x + r2.y);  // this part's share of the row sum
    }
    if (SPLIT > 1) {  // full row sum from the parts (slot parity T&1 is free: last use was T-2)
      float* slot = xch + ((x * 2 + (T & 1)) * SPLIT) * 128;
      slot[hh * 128 + row] = l;
      pair_sync();
      l = 0.f;
#pragma unroll
      for (int k = 0; k < SPLIT; ++k) l += slot[k * 128 + row];
    }
    // epilogue: wait for the last PV_X, O / l -> fp16 (this part's OW columns)
    mbar_wait(&o_done[x], (T - 1) & 1);
    tc_fence_after();
    const float inv = 1.f / l;
    __half* orow = O + ((size_t)bh * S + (size_t)(2 * qt + x) * BM + row) * HD + hh * OW;
#pragma unroll 1
    for (int c = 0; c < OW / 32; ++c) {
      uint32_t v[32];
      tmem_ld32(tO(x) + lane_off + hh * OW + c * 32, v);
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
