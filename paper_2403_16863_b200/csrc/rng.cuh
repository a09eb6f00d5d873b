// rng.cuh -- CPython-exact random streams on the device.
//
// The reference draws every random number through CPython's random.Random:
//   * int seeds (anneal.py:145)            random.Random(cfg.seed)
//   * string seeds (difftest.py:126)       random.Random(f"{seed}:{index}")
// Seeding is init_by_array over the 32-bit words of |seed| (int) or of
// int.from_bytes(s + sha512(s), "big") (str, "version 2" seeding).  Draws:
// getrandbits(k) keeps the top k bits of each 32-bit word, least significant
// word first; randrange(n) = rejection loop on getrandbits(bit_length(n));
// random() = ((a >> 5) * 2^26 + (b >> 6)) / 2^53.
//
// MT state lives wherever the caller puts it: `st[i * stride]` lets the anneal
// engine interleave the 624 words of all chains ([624][chains], coalesced) and
// the sample generator keep one private state in local memory (stride 1).
#pragma once
#include <stdint.h>

namespace sip {

constexpr int MT_N = 624;
constexpr int MT_M = 397;

struct MtRef {
  uint32_t* st;
  int stride;
  int mti;
  __host__ __device__ uint32_t& at(int i) { return st[(long long)i * stride]; }
};

__host__ __device__ inline void mt_init_genrand(MtRef& m, uint32_t s) {
  m.at(0) = s;
  uint32_t prev = s;
  for (int i = 1; i < MT_N; ++i) {
    prev = 1812433253u * (prev ^ (prev >> 30)) + (uint32_t)i;
    m.at(i) = prev;
  }
  m.mti = MT_N;
}

// init_by_array with the 19650218 base state taken from `base` (precomputed once).
__host__ __device__ inline void mt_init_by_array(MtRef& m, const uint32_t* base, const uint32_t* key,
                                                 int klen) {
  for (int i = 0; i < MT_N; ++i) m.at(i) = base[i];
  int i = 1, j = 0;
  uint32_t prev = m.at(0);
  for (int k = (MT_N > klen ? MT_N : klen); k; --k) {
    uint32_t v = (m.at(i) ^ ((prev ^ (prev >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
    m.at(i) = v;
    prev = v;
    ++i;
    ++j;
    if (i >= MT_N) {
      m.at(0) = m.at(MT_N - 1);
      prev = m.at(0);
      i = 1;
    }
    if (j >= klen) j = 0;
  }
  // second pass: eight words per step with their loads issued first (the chain
  // through `prev` is serial, the words it mixes in are not)
  for (int k = MT_N - 1; k;) {
    if (k >= 8 && i + 8 <= MT_N) {
      uint32_t w[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) w[u] = m.at(i + u);
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        uint32_t v = (w[u] ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)(i + u);
        m.at(i + u) = v;
        prev = v;
      }
      i += 8;
      k -= 8;
    } else {
      uint32_t v = (m.at(i) ^ ((prev ^ (prev >> 30)) * 1566083941u)) - (uint32_t)i;
      m.at(i) = v;
      prev = v;
      ++i;
      --k;
    }
    if (i >= MT_N) {
      m.at(0) = m.at(MT_N - 1);
      prev = m.at(0);
      i = 1;
    }
  }
  m.at(0) = 0x80000000u;
  m.mti = MT_N;
}

// Lazy twist: word i of a new round is regenerated right before it is tempered.
// The textbook twist's step i reads slots i, i+1 (both not yet regenerated) and
// i+397 mod 624 (not yet regenerated for i < 227, already regenerated for
// i >= 227), so doing step i on demand yields exactly the same words; a chain
// that draws ~200 numbers no longer regenerates all 624.  mti == 624 after
// seeding still means "start a new round".
__host__ __device__ inline uint32_t mt_next(MtRef& m) {
  if (m.mti >= MT_N) m.mti = 0;
  {
    const int i = m.mti;
    uint32_t y = (m.at(i) & 0x80000000u) | (m.at(i + 1 < MT_N ? i + 1 : 0) & 0x7fffffffu);
    int j = i + MT_M;
    if (j >= MT_N) j -= MT_N;
    m.at(i) = m.at(j) ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
  }
  uint32_t y = m.at(m.mti++);
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

__host__ __device__ inline int bit_length_u32(uint32_t v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

// random.randrange(n) for 1 <= n < 2^32 (Random._randbelow_with_getrandbits)
__host__ __device__ inline uint32_t mt_randbelow(MtRef& m, uint32_t n) {
  int k = bit_length_u32(n);
  uint32_t r = mt_next(m) >> (32 - k);
  while (r >= n) r = mt_next(m) >> (32 - k);
  return r;
}

// random.random()
__host__ __device__ inline double mt_random(MtRef& m) {
  uint32_t a = mt_next(m) >> 5, b = mt_next(m) >> 6;
  return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

// ---------------------------------------------------------------------------
// SHA-512 (FIPS 180-4), single- or multi-block, for the string-seed path.
struct Sha512 {
  uint64_t h[8];
};

__host__ __device__ inline uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

__host__ __device__ inline void sha512_block(uint64_t* h, const uint8_t* blk) {
  const uint64_t K[80] = {
      0x428a2f98d728ae22ull, 0x7137449123ef65cdull, 0xb5c0fbcfec4d3b2full, 0xe9b5dba58189dbbcull,
      0x3956c25bf348b538ull, 0x59f111f1b605d019ull, 0x923f82a4af194f9bull, 0xab1c5ed5da6d8118ull,
      0xd807aa98a3030242ull, 0x12835b0145706fbeull, 0x243185be4ee4b28cull, 0x550c7dc3d5ffb4e2ull,
      0x72be5d74f27b896full, 0x80deb1fe3b1696b1ull, 0x9bdc06a725c71235ull, 0xc19bf174cf692694ull,
      0xe49b69c19ef14ad2ull, 0xefbe4786384f25e3ull, 0x0fc19dc68b8cd5b5ull, 0x240ca1cc77ac9c65ull,
      0x2de92c6f592b0275ull, 0x4a7484aa6ea6e483ull, 0x5cb0a9dcbd41fbd4ull, 0x76f988da831153b5ull,
      0x983e5152ee66dfabull, 0xa831c66d2db43210ull, 0xb00327c898fb213full, 0xbf597fc7beef0ee4ull,
      0xc6e00bf33da88fc2ull, 0xd5a79147930aa725ull, 0x06ca6351e003826full, 0x142929670a0e6e70ull,
      0x27b70a8546d22ffcull, 0x2e1b21385c26c926ull, 0x4d2c6dfc5ac42aedull, 0x53380d139d95b3dfull,
      0x650a73548baf63deull, 0x766a0abb3c77b2a8ull, 0x81c2c92e47edaee6ull, 0x92722c851482353bull,
      0xa2bfe8a14cf10364ull, 0xa81a664bbc423001ull, 0xc24b8b70d0f89791ull, 0xc76c51a30654be30ull,
      0xd192e819d6ef5218ull, 0xd69906245565a910ull, 0xf40e35855771202aull, 0x106aa07032bbd1b8ull,
      0x19a4c116b8d2d0c8ull, 0x1e376c085141ab53ull, 0x2748774cdf8eeb99ull, 0x34b0bcb5e19b48a8ull,
      0x391c0cb3c5c95a63ull, 0x4ed8aa4ae3418acbull, 0x5b9cca4f7763e373ull, 0x682e6ff3d6b2b8a3ull,
      0x748f82ee5defb2fcull, 0x78a5636f43172f60ull, 0x84c87814a1f0ab72ull, 0x8cc702081a6439ecull,
      0x90befffa23631e28ull, 0xa4506cebde82bde9ull, 0xbef9a3f7b2c67915ull, 0xc67178f2e372532bull,
      0xca273eceea26619cull, 0xd186b8c721c0c207ull, 0xeada7dd6cde0eb1eull, 0xf57d4f7fee6ed178ull,
      0x06f067aa72176fbaull, 0x0a637dc5a2c898a6ull, 0x113f9804bef90daeull, 0x1b710b35131c471bull,
      0x28db77f523047d84ull, 0x32caab7b40c72493ull, 0x3c9ebe0a15c9bebcull, 0x431d67c49c100d4cull,
      0x4cc5d4becb3e42b6ull, 0x597f299cfc657e2aull, 0x5fcb6fab3ad6faecull, 0x6c44198c4a475817ull};
  uint64_t w[80];
  for (int t = 0; t < 16; ++t) {
    uint64_t v = 0;
    for (int b = 0; b < 8; ++b) v = (v << 8) | blk[t * 8 + b];
    w[t] = v;
  }
  for (int t = 16; t < 80; ++t) {
    uint64_t s0 = rotr64(w[t - 15], 1) ^ rotr64(w[t - 15], 8) ^ (w[t - 15] >> 7);
    uint64_t s1 = rotr64(w[t - 2], 19) ^ rotr64(w[t - 2], 61) ^ (w[t - 2] >> 6);
    w[t] = w[t - 16] + s0 + w[t - 7] + s1;
  }
  uint64_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
  for (int t = 0; t < 80; ++t) {
    uint64_t S1 = rotr64(e, 14) ^ rotr64(e, 18) ^ rotr64(e, 41);
    uint64_t ch = (e & f) ^ (~e & g);
    uint64_t t1 = hh + S1 + ch + K[t] + w[t];
    uint64_t S0 = rotr64(a, 28) ^ rotr64(a, 34) ^ rotr64(a, 39);
    uint64_t mj = (a & b) ^ (a & c) ^ (b & c);
    uint64_t t2 = S0 + mj;
    hh = g;
    g = f;
    f = e;
    e = d + t1;
    d = c;
    c = b;
    b = a;
    a = t1 + t2;
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d;
  h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

// digest of msg[0..len) (len < 2^32), written big-endian into out[64]
__host__ __device__ inline void sha512(const uint8_t* msg, int len, uint8_t* out) {
  uint64_t h[8] = {0x6a09e667f3bcc908ull, 0xbb67ae8584caa73bull, 0x3c6ef372fe94f82bull,
                   0xa54ff53a5f1d36f1ull, 0x510e527fade682d1ull, 0x9b05688c2b3e6c1full,
                   0x1f83d9abfb41bd6bull, 0x5be0cd19137e2179ull};
  uint8_t blk[128];
  int off = 0;
  while (len - off >= 128) {
    sha512_block(h, msg + off);
    off += 128;
  }
  int rem = len - off;
  for (int i = 0; i < 128; ++i) blk[i] = 0;
  for (int i = 0; i < rem; ++i) blk[i] = msg[off + i];
  blk[rem] = 0x80;
  if (rem >= 112) {
    sha512_block(h, blk);
    for (int i = 0; i < 128; ++i) blk[i] = 0;
  }
  uint64_t bits = (uint64_t)len * 8;
  for (int b = 0; b < 8; ++b) blk[127 - b] = (uint8_t)(bits >> (8 * b));
  sha512_block(h, blk);
  for (int i = 0; i < 8; ++i)
    for (int b = 0; b < 8; ++b) out[i * 8 + b] = (uint8_t)(h[i] >> (56 - 8 * b));
}

// Key words for random.Random(int): 32-bit words of |seed|, least significant first.
__host__ __device__ inline int mt_key_from_int(int64_t seed, uint32_t* key) {
  uint64_t n = seed < 0 ? (uint64_t)(-(seed + 1)) + 1u : (uint64_t)seed;
  key[0] = (uint32_t)n;
  key[1] = (uint32_t)(n >> 32);
  return key[1] ? 2 : 1;
}

// Key words for random.Random(str): int.from_bytes(s + sha512(s), "big").
// buf must hold len+64 bytes; key must hold (len+64+3)/4 words.
__host__ __device__ inline int mt_key_from_bytes(const uint8_t* s, int len, uint8_t* buf,
                                                 uint32_t* key) {
  for (int i = 0; i < len; ++i) buf[i] = s[i];
  sha512(s, len, buf + len);
  int total = len + 64;
  int lead = 0;  // leading zero bytes do not count toward the key length
  while (lead < total && buf[lead] == 0) ++lead;
  int used = total - lead;
  int words = used == 0 ? 1 : (used + 3) / 4;
  for (int w = 0; w < words; ++w) {
    uint32_t v = 0;
    for (int b = 3; b >= 0; --b) {
      int idx = total - 1 - (w * 4 + b);
      v = (v << 8) | (idx >= 0 ? buf[idx] : 0u);
    }
    key[w] = v;
  }
  return words;
}

}  // namespace sip
