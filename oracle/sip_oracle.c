/*
 * sip_oracle.c -- CPU restatement of the reference SIP search loop.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in paper_2403_16863_b200/ links, loads or
 * calls this file; only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may use it, and only as the checker or
 * the timed CPU baseline ("kind": "port").
 *
 * It follows the reference package /root/reference/pkg/src/sasstune line by
 * line in algorithmic structure (not code):
 *   oracle_depgraph_adjacent  deps.build_depgraph     deps.py:279-349
 *   oracle_simulate           machine.simulate        machine.py:116-161
 *   oracle_anneal             anneal.anneal           anneal.py:123-213
 *                             perturb.candidates      perturb.py:48-53
 *                             perturb.sample_action   perturb.py:56-61
 *                             perturb.apply_action    perturb.py:64-90
 *                             anneal.accept_move      anneal.py:39-44
 *   oracle_sample_inputs      difftest.sample_inputs  difftest.py:124-141
 *   MT19937 / seeding         CPython Modules/_randommodule.c (random_seed,
 *                             init_by_array, genrand_uint32, getrandbits,
 *                             random_random) and Lib/random.py (_randbelow)
 * In particular the dependence graph is rebuilt from scratch after every
 * accepted move (anneal.py:198), exactly as the reference does.
 *
 * Parity is pinned: tests/test_oracle.py checks every function here against
 * tests/golden/reference.json.gz, produced by running the reference itself
 * (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/sip.h"

/* ---------------- CPython MT19937 ---------------- */
typedef struct {
  uint32_t mt[624];
  int mti;
} mt_t;

static void mt_seed_genrand(mt_t* m, uint32_t s) {
  m->mt[0] = s;
  for (int i = 1; i < 624; i++)
    m->mt[i] = 1812433253u * (m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) + (uint32_t)i;
  m->mti = 624;
}

static void mt_seed_array(mt_t* m, const uint32_t* key, int len) {
  mt_seed_genrand(m, 19650218u);
  int i = 1, j = 0, k = 624 > len ? 624 : len;
  for (; k; k--) {
    m->mt[i] = (m->mt[i] ^ ((m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) * 1664525u)) + key[j] + (uint32_t)j;
    i++;
    j++;
    if (i >= 624) {
      m->mt[0] = m->mt[623];
      i = 1;
    }
    if (j >= len) j = 0;
  }
  for (k = 623; k; k--) {
    m->mt[i] = (m->mt[i] ^ ((m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) * 1566083941u)) - (uint32_t)i;
    i++;
    if (i >= 624) {
      m->mt[0] = m->mt[623];
      i = 1;
    }
  }
  m->mt[0] = 0x80000000u;
}

static uint32_t mt_u32(mt_t* m) {
  static const uint32_t mag[2] = {0u, 0x9908b0dfu};
  uint32_t y;
  if (m->mti >= 624) {
    int kk;
    for (kk = 0; kk < 624 - 397; kk++) {
      y = (m->mt[kk] & 0x80000000u) | (m->mt[kk + 1] & 0x7fffffffu);
      m->mt[kk] = m->mt[kk + 397] ^ (y >> 1) ^ mag[y & 1u];
    }
    for (; kk < 623; kk++) {
      y = (m->mt[kk] & 0x80000000u) | (m->mt[kk + 1] & 0x7fffffffu);
      m->mt[kk] = m->mt[kk + (397 - 624)] ^ (y >> 1) ^ mag[y & 1u];
    }
    y = (m->mt[623] & 0x80000000u) | (m->mt[0] & 0x7fffffffu);
    m->mt[623] = m->mt[396] ^ (y >> 1) ^ mag[y & 1u];
    m->mti = 0;
  }
  y = m->mt[m->mti++];
  y ^= (y >> 11);
  y ^= (y << 7) & 0x9d2c5680u;
  y ^= (y << 15) & 0xefc60000u;
  y ^= (y >> 18);
  return y;
}

static void mt_seed_int(mt_t* m, int64_t seed) {
  uint64_t a = seed < 0 ? (uint64_t)0 - (uint64_t)seed : (uint64_t)seed;
  uint32_t key[2] = {(uint32_t)a, (uint32_t)(a >> 32)};
  mt_seed_array(m, key, key[1] ? 2 : 1);
}

static uint32_t mt_below(mt_t* m, uint32_t n) {
  int k = 0;
  for (uint32_t v = n; v; v >>= 1) k++;
  uint32_t r;
  do {
    r = mt_u32(m) >> (32 - k);
  } while (r >= n);
  return r;
}

static double mt_unit(mt_t* m) {
  uint32_t a = mt_u32(m) >> 5, b = mt_u32(m) >> 6;
  return (a * 67108864.0 + b) * (1.0 / 9007199254740992.0);
}

/* ---------------- SHA-512 (for string seeds) ---------------- */
static uint64_t ror(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

static const uint64_t SHA_K[80] = {
    0x428a2f98d728ae22ULL, 0x7137449123ef65cdULL, 0xb5c0fbcfec4d3b2fULL, 0xe9b5dba58189dbbcULL,
    0x3956c25bf348b538ULL, 0x59f111f1b605d019ULL, 0x923f82a4af194f9bULL, 0xab1c5ed5da6d8118ULL,
    0xd807aa98a3030242ULL, 0x12835b0145706fbeULL, 0x243185be4ee4b28cULL, 0x550c7dc3d5ffb4e2ULL,
    0x72be5d74f27b896fULL, 0x80deb1fe3b1696b1ULL, 0x9bdc06a725c71235ULL, 0xc19bf174cf692694ULL,
    0xe49b69c19ef14ad2ULL, 0xefbe4786384f25e3ULL, 0x0fc19dc68b8cd5b5ULL, 0x240ca1cc77ac9c65ULL,
    0x2de92c6f592b0275ULL, 0x4a7484aa6ea6e483ULL, 0x5cb0a9dcbd41fbd4ULL, 0x76f988da831153b5ULL,
    0x983e5152ee66dfabULL, 0xa831c66d2db43210ULL, 0xb00327c898fb213fULL, 0xbf597fc7beef0ee4ULL,
    0xc6e00bf33da88fc2ULL, 0xd5a79147930aa725ULL, 0x06ca6351e003826fULL, 0x142929670a0e6e70ULL,
    0x27b70a8546d22ffcULL, 0x2e1b21385c26c926ULL, 0x4d2c6dfc5ac42aedULL, 0x53380d139d95b3dfULL,
    0x650a73548baf63deULL, 0x766a0abb3c77b2a8ULL, 0x81c2c92e47edaee6ULL, 0x92722c851482353bULL,
    0xa2bfe8a14cf10364ULL, 0xa81a664bbc423001ULL, 0xc24b8b70d0f89791ULL, 0xc76c51a30654be30ULL,
    0xd192e819d6ef5218ULL, 0xd69906245565a910ULL, 0xf40e35855771202aULL, 0x106aa07032bbd1b8ULL,
    0x19a4c116b8d2d0c8ULL, 0x1e376c085141ab53ULL, 0x2748774cdf8eeb99ULL, 0x34b0bcb5e19b48a8ULL,
    0x391c0cb3c5c95a63ULL, 0x4ed8aa4ae3418acbULL, 0x5b9cca4f7763e373ULL, 0x682e6ff3d6b2b8a3ULL,
    0x748f82ee5defb2fcULL, 0x78a5636f43172f60ULL, 0x84c87814a1f0ab72ULL, 0x8cc702081a6439ecULL,
    0x90befffa23631e28ULL, 0xa4506cebde82bde9ULL, 0xbef9a3f7b2c67915ULL, 0xc67178f2e372532bULL,
    0xca273eceea26619cULL, 0xd186b8c721c0c207ULL, 0xeada7dd6cde0eb1eULL, 0xf57d4f7fee6ed178ULL,
    0x06f067aa72176fbaULL, 0x0a637dc5a2c898a6ULL, 0x113f9804bef90daeULL, 0x1b710b35131c471bULL,
    0x28db77f523047d84ULL, 0x32caab7b40c72493ULL, 0x3c9ebe0a15c9bebcULL, 0x431d67c49c100d4cULL,
    0x4cc5d4becb3e42b6ULL, 0x597f299cfc657e2aULL, 0x5fcb6fab3ad6faecULL, 0x6c44198c4a475817ULL};

static void sha_compress(uint64_t st[8], const uint8_t b[128]) {
  uint64_t w[80], v[8];
  for (int t = 0; t < 16; t++) {
    w[t] = 0;
    for (int i = 0; i < 8; i++) w[t] = (w[t] << 8) | b[8 * t + i];
  }
  for (int t = 16; t < 80; t++)
    w[t] = w[t - 16] + (ror(w[t - 15], 1) ^ ror(w[t - 15], 8) ^ (w[t - 15] >> 7)) + w[t - 7] +
           (ror(w[t - 2], 19) ^ ror(w[t - 2], 61) ^ (w[t - 2] >> 6));
  memcpy(v, st, sizeof v);
  for (int t = 0; t < 80; t++) {
    uint64_t t1 = v[7] + (ror(v[4], 14) ^ ror(v[4], 18) ^ ror(v[4], 41)) +
                  ((v[4] & v[5]) ^ (~v[4] & v[6])) + SHA_K[t] + w[t];
    uint64_t t2 = (ror(v[0], 28) ^ ror(v[0], 34) ^ ror(v[0], 39)) +
                  ((v[0] & v[1]) ^ (v[0] & v[2]) ^ (v[1] & v[2]));
    memmove(v + 1, v, 7 * sizeof(uint64_t));
    v[4] += t1;
    v[0] = t1 + t2;
  }
  for (int i = 0; i < 8; i++) st[i] += v[i];
}

void oracle_sha512(const uint8_t* msg, size_t len, uint8_t out[64]) {
  uint64_t st[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                    0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                    0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
  uint8_t blk[128];
  size_t off = 0;
  for (; len - off >= 128; off += 128) sha_compress(st, msg + off);
  size_t rem = len - off;
  memset(blk, 0, sizeof blk);
  memcpy(blk, msg + off, rem);
  blk[rem] = 0x80;
  if (rem >= 112) {
    sha_compress(st, blk);
    memset(blk, 0, sizeof blk);
  }
  uint64_t bits = (uint64_t)len * 8;
  for (int i = 0; i < 8; i++) blk[127 - i] = (uint8_t)(bits >> (8 * i));
  sha_compress(st, blk);
  for (int i = 0; i < 8; i++)
    for (int j = 0; j < 8; j++) out[8 * i + j] = (uint8_t)(st[i] >> (56 - 8 * j));
}

/* random.Random(str): seed = int.from_bytes(s + sha512(s).digest(), 'big') */
static void mt_seed_str(mt_t* m, const char* s) {
  size_t len = strlen(s);
  uint8_t* buf = (uint8_t*)malloc(len + 64);
  memcpy(buf, s, len);
  oracle_sha512((const uint8_t*)s, len, buf + len);
  size_t total = len + 64, lead = 0;
  while (lead < total && buf[lead] == 0) lead++;
  size_t nbytes = total - lead;
  int words = nbytes == 0 ? 1 : (int)((nbytes + 3) / 4);
  uint32_t* key = (uint32_t*)calloc((size_t)words, sizeof(uint32_t));
  for (size_t i = 0; i < total && i / 4 < (size_t)words; i++) /* least significant byte first */
    key[i / 4] |= (uint32_t)buf[total - 1 - i] << (8 * (i % 4));
  mt_seed_array(m, key, words);
  free(key);
  free(buf);
}

/* getrandbits(k) for k > 0, little-endian bytes of the result into out[(k+7)/8] */
static void mt_bits_le(mt_t* m, int64_t k, uint8_t* out) {
  int64_t nbytes = (k + 7) / 8;
  int64_t words = (k - 1) / 32 + 1;
  for (int64_t i = 0; i < words; i++, k -= 32) {
    uint32_t r = mt_u32(m);
    if (k < 32) r >>= (32 - k);
    for (int b = 0; b < 4; b++) {
      int64_t idx = i * 4 + b;
      if (idx < nbytes) out[idx] = (uint8_t)(r >> (8 * b));
    }
  }
}

/* ---------------- dependence graph (reference algorithm) ---------------- */
typedef struct {
  int n, words, nregs;
  const uint32_t* ctrl;
  const uint32_t* lat;
  const uint64_t* reads;
  const uint64_t* writes;
  const sip_memref* refs;
  const uint8_t* nrefs;
  const uint8_t* cut;
} listing_t;

typedef struct {
  int* v;
  int len, cap;
} ivec;

static void ivec_push(ivec* a, int x) {
  if (a->len == a->cap) {
    a->cap = a->cap ? 2 * a->cap : 8;
    a->v = (int*)realloc(a->v, sizeof(int) * (size_t)a->cap);
  }
  a->v[a->len++] = x;
}

static int bit_get(const uint64_t* row, int b) { return (int)((row[b >> 6] >> (b & 63)) & 1u); }

#define FENCE_BIT (1u << 21)
#define GLOBAL_BIT (1u << 22)
#define CAND_BIT (1u << 23) /* movable: GLOBAL classes (reference) or the opt-in extension */

static int alias(const sip_memref* a, const sip_memref* b) {
  if (a->space != 3 && b->space != 3 && a->space != b->space) return 0;
  if (a->base < 0 || b->base < 0 || a->base != b->base) return 1;
  return !(a->offset + a->size <= b->offset || b->offset + b->size <= a->offset);
}

static int mem_edge(const listing_t* L, int i, int j) {
  int bg = (L->ctrl[i] & GLOBAL_BIT) && (L->ctrl[j] & GLOBAL_BIT);
  for (int x = 0; x < L->nrefs[i]; x++)
    for (int y = 0; y < L->nrefs[j]; y++) {
      const sip_memref* a = &L->refs[i * SIP_MAX_REFS + x];
      const sip_memref* b = &L->refs[j * SIP_MAX_REFS + y];
      if (alias(a, b) && (a->write || b->write || bg)) return 1;
    }
  return 0;
}

/* Builds every edge of the schedule `order` (positions -> identities), as
 * deps.build_depgraph does, and reports which adjacent pairs are connected:
 * adj[p] = 1 iff an edge joins positions p and p+1.  Returns the edge count. */
long oracle_depgraph_adjacent(const listing_t* L, const uint16_t* order, uint8_t* adj) {
  int n = L->n, R = L->nregs;
  long edges = 0;
  int* last_writer = (int*)malloc(sizeof(int) * (size_t)(R ? R : 1));
  ivec* readers = (ivec*)calloc((size_t)(R ? R : 1), sizeof(ivec));
  int last_setter[6];
  ivec waiters[6];
  memset(waiters, 0, sizeof waiters);
  for (int r = 0; r < R; r++) last_writer[r] = -1;
  for (int b = 0; b < 6; b++) last_setter[b] = -1;
  memset(adj, 0, (size_t)(n > 0 ? n : 1));
#define EDGE(s, d)                        \
  do {                                    \
    int s_ = (s), d_ = (d);               \
    if (s_ != d_) {                       \
      edges++;                            \
      if (d_ == s_ + 1) adj[s_] = 1;      \
    }                                     \
  } while (0)
  for (int j = 0; j < n; j++) {
    int x = order[j];
    const uint64_t* rd = L->reads + (size_t)x * L->words;
    const uint64_t* wr = L->writes + (size_t)x * L->words;
    for (int r = 0; r < R; r++)
      if (bit_get(rd, r) && last_writer[r] >= 0) EDGE(last_writer[r], j);
    for (int r = 0; r < R; r++) {
      if (!bit_get(wr, r)) continue;
      for (int q = 0; q < readers[r].len; q++) EDGE(readers[r].v[q], j);
      if (last_writer[r] >= 0) EDGE(last_writer[r], j);
    }
    for (int r = 0; r < R; r++)
      if (bit_get(wr, r)) {
        last_writer[r] = j;
        readers[r].len = 0;
      }
    for (int r = 0; r < R; r++)
      if (bit_get(rd, r)) ivec_push(&readers[r], j);
    uint32_t c = L->ctrl[x];
    for (int b = 0; b < 6; b++)
      if ((c >> b) & 1u) {
        if (last_setter[b] >= 0) EDGE(last_setter[b], j);
        ivec_push(&waiters[b], j);
      }
    int bars[2] = {(int)((c >> 6) & 7u), (int)((c >> 9) & 7u)};
    for (int t = 0; t < 2; t++) {
      int b = bars[t];
      if (b >= 6) continue;
      for (int q = 0; q < waiters[b].len; q++) EDGE(waiters[b].v[q], j);
      waiters[b].len = 0;
      last_setter[b] = j;
    }
  }
  /* memory pass: every ordered pair of memory instructions (O(m^2)) */
  for (int i = 0; i < n; i++) {
    if (!L->nrefs[order[i]]) continue;
    for (int j = i + 1; j < n; j++)
      if (L->nrefs[order[j]] && mem_edge(L, order[i], order[j])) EDGE(i, j);
  }
  /* block fence: BARRIER / CONTROL_FLOW instructions fence their block */
  int start = 0;
  for (int i = 0; i < n; i++) {
    if (i > 0 && L->cut[i]) start = i;
    if (!(L->ctrl[order[i]] & FENCE_BIT)) continue;
    int end = i + 1;
    while (end < n && !L->cut[end]) end++;
    for (int j = start; j < end; j++) {
      if (j < i) EDGE(j, i);
      else if (j > i) EDGE(i, j);
    }
  }
#undef EDGE
  for (int r = 0; r < R; r++) free(readers[r].v);
  for (int b = 0; b < 6; b++) free(waiters[b].v);
  free(readers);
  free(last_writer);
  return edges;
}

/* machine.simulate total_cycles for positions -> identities `order` */
int64_t oracle_simulate(const listing_t* L, const uint16_t* order) {
  int64_t clear[6] = {0, 0, 0, 0, 0, 0}, ptr = 0, fin = 0;
  for (int p = 0; p < L->n; p++) {
    uint32_t c = L->ctrl[order[p]];
    int64_t issue = ptr;
    for (int b = 0; b < 6; b++)
      if (((c >> b) & 1u) && clear[b] > issue) issue = clear[b];
    int64_t done = issue + (int64_t)L->lat[order[p]];
    int rdb = (int)((c >> 6) & 7u), wrb = (int)((c >> 9) & 7u);
    if (rdb < 6) clear[rdb] = done;
    if (wrb < 6) clear[wrb] = done;
    if (done > fin) fin = done;
    ptr = issue + (int64_t)((c >> 12) & 31u);
  }
  if (L->n == 0) return 0;
  return fin > ptr ? fin : ptr;
}

static void make_listing(listing_t* L, const sip_tables* t) {
  L->n = t->n;
  L->words = t->words;
  L->nregs = t->words * 64;
  L->ctrl = t->ctrl;
  L->lat = t->lat;
  L->reads = t->reads;
  L->writes = t->writes;
  L->refs = t->refs;
  L->nrefs = t->nrefs;
  L->cut = t->cut;
}

int64_t oracle_simulate_tables(const sip_tables* t, const uint16_t* order) {
  listing_t L;
  make_listing(&L, t);
  return oracle_simulate(&L, order);
}

/* adjacency verdicts of deps.swap_legal for every slot of one schedule */
long oracle_swap_legal(const sip_tables* t, const uint16_t* order, uint8_t* legal) {
  listing_t L;
  make_listing(&L, t);
  uint8_t* adj = (uint8_t*)malloc((size_t)(t->n > 0 ? t->n : 1));
  long e = oracle_depgraph_adjacent(&L, order, adj);
  for (int p = 0; p + 1 < t->n; p++) legal[p] = (uint8_t)(!t->cut[p + 1] && !adj[p]);
  free(adj);
  return e;
}

/* One annealing chain with the simulator backend (anneal.py:123-213). */
int oracle_anneal(const sip_tables* t, const double* temps, int budget, int unsafe, int64_t seed,
                  sip_record* hist, uint16_t* best_out, uint16_t* cur_out,
                  sip_chain_summary* summary) {
  listing_t L;
  make_listing(&L, t);
  int n = t->n;
  uint16_t* x = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
  uint16_t* cand = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
  uint16_t* best = (uint16_t*)malloc(sizeof(uint16_t) * (size_t)n);
  uint8_t* adj = (uint8_t*)malloc((size_t)n);
  int* cpos = (int*)malloc(sizeof(int) * (size_t)n);
  for (int i = 0; i < n; i++) x[i] = best[i] = (uint16_t)i;
  int k = 0;
  for (int i = 0; i < n; i++)
    if (t->ctrl[i] & CAND_BIT) k++;
  if (k == 0) {
    free(x); free(cand); free(best); free(adj); free(cpos);
    return SIP_E_NOCAND;
  }
  double t0 = (double)oracle_simulate(&L, x);
  mt_t m;
  mt_seed_int(&m, seed);
  oracle_depgraph_adjacent(&L, x, adj);
  double e_x = 1.0, e_best = 1.0;
  int best_iter = -1;
  for (int it = 0; it < budget; it++) {
    int nc = 0; /* perturb.candidates: positions of global-class instructions */
    for (int p = 0; p < n; p++)
      if (t->ctrl[x[p]] & CAND_BIT) cpos[nc++] = p;
    uint32_t cell = mt_below(&m, 2u * (uint32_t)nc);
    int ci = (int)(cell >> 1), dir = (int)(cell & 1u);
    int pos = cpos[ci];
    int lo = dir == 0 ? pos - 1 : pos;
    sip_record* r = &hist[it];
    r->candidate = (uint16_t)ci;
    r->direction = (uint8_t)dir;
    r->lo = lo;
    r->time = 0.0;
    if (lo < 0 || lo + 1 >= n || t->cut[lo + 1]) {
      r->status = SIP_ST_BOUNDARY;
      continue;
    }
    if (!unsafe && adj[lo]) {
      r->status = SIP_ST_DEPENDENCY;
      continue;
    }
    memcpy(cand, x, sizeof(uint16_t) * (size_t)n);
    cand[lo] = x[lo + 1];
    cand[lo + 1] = x[lo];
    double tc = (double)oracle_simulate(&L, cand);
    double e_c = tc / t0;
    double de = e_c - e_x;
    int acc = de < 0 ? 1 : (mt_unit(&m) < exp(-de / temps[it]));
    r->time = tc;
    r->status = acc ? SIP_ST_ACCEPTED : SIP_ST_PRICED;
    if (acc) {
      memcpy(x, cand, sizeof(uint16_t) * (size_t)n);
      e_x = e_c;
      oracle_depgraph_adjacent(&L, x, adj); /* full rebuild, anneal.py:198 */
      if (de < 0 && e_c < e_best) {
        e_best = e_c;
        best_iter = it;
        memcpy(best, x, sizeof(uint16_t) * (size_t)n);
      }
    }
  }
  if (best_out) memcpy(best_out, best, sizeof(uint16_t) * (size_t)n);
  if (cur_out) memcpy(cur_out, x, sizeof(uint16_t) * (size_t)n);
  if (summary) {
    summary->t0 = t0;
    summary->best_energy = e_best;
    summary->current_energy = e_x;
    summary->best_iter = best_iter;
    summary->ambiguous = 0;
    summary->replayed = 0;
    summary->priced = 0;
    for (int it = 0; it < budget; it++) summary->priced += hist[it].status <= SIP_ST_PRICED;
    summary->pad = 0;
  }
  free(x); free(cand); free(best); free(adj); free(cpos);
  return SIP_OK;
}

/* difftest.sample_inputs for one sample index; buffers concatenated in `out`.
 * dist: 0 uniform, 1 small, 2 zero.  length = element count, cell = bytes. */
int oracle_sample_inputs(int64_t seed, int64_t index, int nbuf, const int32_t* length,
                         const int32_t* cell, const int32_t* dist, uint8_t* out) {
  char s[64];
  int len = 0;
  {
    /* f"{seed}:{index}" */
    char tmp[48];
    int64_t vals[2] = {seed, index};
    for (int v = 0; v < 2; v++) {
      int64_t a = vals[v];
      int neg = a < 0, tl = 0;
      uint64_t u = neg ? (uint64_t)0 - (uint64_t)a : (uint64_t)a;
      do {
        tmp[tl++] = (char)('0' + u % 10);
        u /= 10;
      } while (u);
      if (neg) s[len++] = '-';
      while (tl) s[len++] = tmp[--tl];
      if (v == 0) s[len++] = ':';
    }
    s[len] = 0;
  }
  mt_t m;
  mt_seed_str(&m, s);
  size_t off = 0;
  for (int b = 0; b < nbuf; b++) {
    size_t nbytes = (size_t)length[b] * (size_t)cell[b];
    if (dist[b] == 2) {
      memset(out + off, 0, nbytes);
    } else if (dist[b] == 1) {
      uint8_t* raw = (uint8_t*)malloc((size_t)length[b]);
      mt_bits_le(&m, 8 * (int64_t)length[b], raw);
      memset(out + off, 0, nbytes);
      for (int i = 0; i < length[b]; i++) out[off + (size_t)i * cell[b]] = raw[i] & 0x0f;
      free(raw);
    } else {
      mt_bits_le(&m, 8 * (int64_t)nbytes, out + off);
    }
    off += nbytes;
  }
  return SIP_OK;
}
