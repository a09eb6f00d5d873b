// interp.cu -- GPU interpreter of the reference's integer SASS subset.
//
// Reference: machine.CompiledKernel / interpret (machine.py:164-723): a
// single-thread functional model -- integer ALU, LDG/STG/LDS/STS/LDGSTS,
// predicates, constant bank -- used by difftest.run_tests (difftest.py:158-204)
// to compare a mutant schedule against the reference schedule on random inputs.
// Here the host compiles each instruction once into a 64-byte op (interp.py,
// which raises UnsupportedInstruction exactly where the reference does) and
// one device thread executes one sample: registers and predicates live in the
// thread's local memory, the sample's buffers in its own slice of a device
// region filled by the device sample stream (verify.cu), shared memory in a
// per-sample scratch slice.  Outcomes: 0 ok, 1 global OOB, 2 shared OOB,
// 3 uninitialised read (strict mode); bits 8.. = access size; fault = offending
// address (or register id).
#include <cstring>

#include "common.h"

namespace {

constexpr int NREG = 512;      // R0..R299, RZ=300, UR0..UR99 = 301.., URZ = 401
constexpr int RZ_IDX = 300, URZ_IDX = 401;
constexpr int PT_IDX = 8, UPT_IDX = 17;

enum Op : int32_t {
  OP_NOP = 0, OP_EXIT, OP_MOV, OP_ZERO, OP_LDC2, OP_IMAD, OP_IMADW, OP_IADD3, OP_LEA, OP_LOP3,
  OP_SHF, OP_SEL, OP_ISETP, OP_IMNMX, OP_IABS, OP_POPC, OP_LOAD, OP_STORE, OP_LDGSTS
};
enum SrcKind : int32_t { SK_IMM = 0, SK_REG = 1, SK_ZERO = 2 };
enum Mod : int32_t { MD_NONE = 0, MD_NEG = 1, MD_NOT = 2, MD_ABS = 3 };

struct VmOp {
  int32_t w[16];
};

struct Mem {
  uint8_t* region;         // this sample's buffers
  uint8_t* shared;         // this sample's shared scratch (may be null)
  int32_t shared_bytes;
  int nbuf;
  const int64_t* bases;    // virtual base address per buffer
  const int32_t* lens;     // bytes per buffer
  const int32_t* offs;     // byte offset of each buffer inside the region
};

struct Th {
  uint32_t R[NREG];
  uint32_t valid[NREG / 32];
  uint32_t P;
  int strict;
  int status;
  int64_t fault;
};

__device__ __forceinline__ bool reg_null(int r) { return r == RZ_IDX || r == URZ_IDX; }

__device__ __forceinline__ uint32_t rd_reg(Th& t, int r) {
  if (reg_null(r)) return 0u;
  if (t.strict && !((t.valid[r >> 5] >> (r & 31)) & 1u)) {
    if (t.status == 0) {
      t.status = 3;
      t.fault = r;
    }
    return 0u;
  }
  return t.R[r];
}
__device__ __forceinline__ void wr_reg(Th& t, int r, uint32_t v) {
  if (reg_null(r) || r < 0 || r >= NREG) return;
  t.R[r] = v;
  t.valid[r >> 5] |= 1u << (r & 31);
}
__device__ __forceinline__ bool rd_pred(const Th& t, int p, int neg) {
  bool v = (p == PT_IDX || p == UPT_IDX) ? true : ((t.P >> p) & 1u);
  return neg ? !v : v;
}
__device__ __forceinline__ void wr_pred(Th& t, int p, bool v) {
  if (p == PT_IDX || p == UPT_IDX) return;
  t.P = v ? (t.P | (1u << p)) : (t.P & ~(1u << p));
}

__device__ __forceinline__ uint32_t src(Th& t, int32_t km, int32_t val) {
  int kind = km & 15, mod = km >> 4;
  if (kind == SK_IMM) return (uint32_t)val;
  if (kind == SK_ZERO) return 0u;
  if (kind == 3) {  // unset constant-bank word read in strict mode
    if (t.status == 0) {
      t.status = 3;
      t.fault = -1;
    }
    return 0u;
  }
  uint32_t v = rd_reg(t, val);
  if (mod == MD_NEG) return (uint32_t)(-(int64_t)v);
  if (mod == MD_NOT) return ~v;
  if (mod == MD_ABS) {
    int32_t s = (int32_t)v;
    return (uint32_t)(s < 0 ? -(int64_t)s : s);
  }
  return v;
}

// 64-bit address: base register (lo | hi<<32 when paired) + signed offset
__device__ __forceinline__ int64_t addr_of(Th& t, int32_t base, int32_t pair, int32_t off_lo, int32_t off_hi) {
  int64_t off = (int64_t)(((uint64_t)(uint32_t)off_hi << 32) | (uint32_t)off_lo);
  if (base < 0) return off;
  uint64_t lo = rd_reg(t, base);
  uint64_t v = lo;
  if (pair) v |= (uint64_t)rd_reg(t, base + 1) << 32;
  return (int64_t)v + off;
}

__device__ uint8_t* locate(Th& t, const Mem& m, int space, int64_t addr, int size) {
  if (space == 1) {  // shared
    if (addr < 0 || addr + size > m.shared_bytes) {
      if (t.status == 0) {
        t.status = 2 | (size << 8);
        t.fault = addr;
      }
      return nullptr;
    }
    return m.shared + addr;
  }
  for (int b = 0; b < m.nbuf; ++b) {
    int64_t off = addr - m.bases[b];
    if (off >= 0 && off + size <= m.lens[b]) return m.region + m.offs[b] + off;
  }
  if (t.status == 0) {
    t.status = 1 | (size << 8);
    t.fault = addr;
  }
  return nullptr;
}

__device__ bool cmp_op(int c, int64_t a, int64_t b) {
  switch (c) {
    case 0: return a == b;
    case 1: return a != b;
    case 2: return a < b;
    case 3: return a <= b;
    case 4: return a > b;
    default: return a >= b;
  }
}

__device__ void exec(const VmOp* prog, int nops, Th& t, const Mem& m) {
  for (int i = 0; i < nops && t.status == 0; ++i) {
    const int32_t* w = prog[i].w;
    const int32_t g = w[1];
    if (g & (1 << 9)) {
      if (!rd_pred(t, g & 0xff, (g >> 8) & 1)) continue;
    }
    switch (w[0]) {
      case OP_NOP:
        break;
      case OP_EXIT:
        return;
      case OP_MOV:
        wr_reg(t, w[2], src(t, w[3], w[4]));
        break;
      case OP_ZERO:
        wr_reg(t, w[2], 0u);
        break;
      case OP_LDC2: {  // constants resolved on the host: lo in A, hi in B (w[9] = words)
        uint32_t lo = src(t, w[3], w[4]), hi = src(t, w[5], w[6]);
        wr_reg(t, w[2], lo);
        if (w[9] == 2) wr_reg(t, w[10], hi);
        break;
      }
      case OP_IMAD: {
        uint32_t a = src(t, w[3], w[4]), b = src(t, w[5], w[6]), c = src(t, w[7], w[8]);
        wr_reg(t, w[2], a * b + c);
        break;
      }
      case OP_IMADW: {  // w[9]=unsigned, w[10]=acc kind (0 reg pair, 1 imm), w[11..12] acc
        uint32_t a = src(t, w[3], w[4]), b = src(t, w[5], w[6]);
        uint64_t c64;
        if (w[10] == 0) {
          int ar = w[11];
          uint64_t lo = rd_reg(t, ar);
          uint64_t hi = reg_null(ar) ? 0u : rd_reg(t, ar + 1);
          c64 = lo | (hi << 32);
        } else {
          c64 = ((uint64_t)(uint32_t)w[12] << 32) | (uint32_t)w[11];
        }
        uint64_t prod = w[9] ? (uint64_t)a * (uint64_t)b : (uint64_t)((int64_t)(int32_t)a * (int64_t)(int32_t)b);
        uint64_t tot = prod + c64;
        wr_reg(t, w[2], (uint32_t)tot);
        if (!reg_null(w[2])) wr_reg(t, w[2] + 1, (uint32_t)(tot >> 32));
        break;
      }
      case OP_IADD3:
        wr_reg(t, w[2], src(t, w[3], w[4]) + src(t, w[5], w[6]) + src(t, w[7], w[8]));
        break;
      case OP_LEA: {
        uint32_t a = src(t, w[3], w[4]), b = src(t, w[5], w[6]);
        wr_reg(t, w[2], b + (a << (w[9] & 31)));
        break;
      }
      case OP_LOP3: {
        uint32_t a = src(t, w[3], w[4]), b = src(t, w[5], w[6]), c = src(t, w[7], w[8]);
        uint32_t lut = (uint32_t)w[9], out = 0;
        for (int mt = 0; mt < 8; ++mt) {
          if (!((lut >> mt) & 1u)) continue;
          uint32_t term = (mt & 4) ? a : ~a;
          term &= (mt & 2) ? b : ~b;
          term &= (mt & 1) ? c : ~c;
          out |= term;
        }
        wr_reg(t, w[2], out);
        break;
      }
      case OP_SHF: {  // w[9] bit0 left, bit1 arithmetic, bit2 hi
        uint32_t lo = src(t, w[3], w[4]), sh = src(t, w[5], w[6]) & 63u, hi = src(t, w[7], w[8]);
        uint64_t cat = ((uint64_t)hi << 32) | lo;
        uint64_t r;
        if (w[9] & 1) r = cat << sh;
        else if (w[9] & 2) r = (uint64_t)((int64_t)cat >> sh);
        else r = cat >> sh;
        wr_reg(t, w[2], (uint32_t)((w[9] & 4) ? (r >> 32) : r));
        break;
      }
      case OP_SEL: {  // w[9] pred, w[10] negate
        uint32_t a = src(t, w[3], w[4]), b = src(t, w[5], w[6]);
        wr_reg(t, w[2], rd_pred(t, w[9], w[10]) ? a : b);
        break;
      }
      case OP_ISETP: {  // w[2] pd, w[9] cmp, w[10] comb (0 and 1 or 2 xor), w[11] unsigned, w[12] pin, w[13] neg
        uint32_t a = src(t, w[3], w[4]), b = src(t, w[5], w[6]);
        int64_t x = w[11] ? (int64_t)a : (int64_t)(int32_t)a;
        int64_t y = w[11] ? (int64_t)b : (int64_t)(int32_t)b;
        bool c = cmp_op(w[9], x, y), p = rd_pred(t, w[12], w[13]);
        bool r = w[10] == 0 ? (c && p) : (w[10] == 1 ? (c || p) : (c != p));
        wr_pred(t, w[2], r);
        break;
      }
      case OP_IMNMX: {  // w[9] pred, w[10] negate, w[11] unsigned
        uint32_t a = src(t, w[3], w[4]), b = src(t, w[5], w[6]);
        int64_t x = w[11] ? (int64_t)a : (int64_t)(int32_t)a;
        int64_t y = w[11] ? (int64_t)b : (int64_t)(int32_t)b;
        bool take_min = rd_pred(t, w[9], w[10]);
        wr_reg(t, w[2], take_min ? (x <= y ? a : b) : (x >= y ? a : b));
        break;
      }
      case OP_IABS: {
        int32_t s = (int32_t)src(t, w[3], w[4]);
        wr_reg(t, w[2], (uint32_t)(s < 0 ? -(int64_t)s : s));
        break;
      }
      case OP_POPC:
        wr_reg(t, w[2], (uint32_t)__popc(src(t, w[3], w[4])));
        break;
      case OP_LOAD: {  // w[9] space, w[10] base, w[11] pair, w[12..13] offset, w[14] size, w[15] signed
        int64_t ad = addr_of(t, w[10], w[11], w[12], w[13]);
        int size = w[14];
        uint8_t* p = locate(t, m, w[9], ad, size);
        if (!p) return;
        if (size >= 4) {
          for (int k = 0; k < size / 4; ++k) {
            uint32_t v;
            memcpy(&v, p + 4 * k, 4);
            if (!reg_null(w[2])) wr_reg(t, w[2] + k, v);
          }
        } else {
          uint32_t v = size == 1 ? p[0] : (uint32_t)p[0] | ((uint32_t)p[1] << 8);
          if (w[15]) v = size == 1 ? (uint32_t)(int32_t)(int8_t)v : (uint32_t)(int32_t)(int16_t)v;
          wr_reg(t, w[2], v);
        }
        break;
      }
      case OP_STORE: {  // w[2] data reg, w[9] space, w[10] base, w[11] pair, w[12..13] off, w[14] size
        int size = w[14];
        uint32_t data[4];
        int nr = size >= 4 ? size / 4 : 1;
        for (int k = 0; k < nr; ++k) data[k] = rd_reg(t, reg_null(w[2]) ? w[2] : w[2] + k);
        int64_t ad = addr_of(t, w[10], w[11], w[12], w[13]);
        uint8_t* p = locate(t, m, w[9], ad, size);
        if (!p) return;
        if (size >= 4) {
          memcpy(p, data, size);
        } else {
          p[0] = (uint8_t)data[0];
          if (size == 2) p[1] = (uint8_t)(data[0] >> 8);
        }
        break;
      }
      case OP_LDGSTS: {  // dst shared: w[2] base, w[3] pair, w[4..5] off; src global: w[10] base, w[11] pair, w[12..13]
        int size = w[14];
        int64_t src_ad = addr_of(t, w[10], w[11], w[12], w[13]);
        int64_t dst_ad = addr_of(t, w[2], w[3], w[4], w[5]);
        uint8_t* s = locate(t, m, 0, src_ad, size);
        if (!s) return;
        uint8_t* d = locate(t, m, 1, dst_ad, size);
        if (!d) return;
        memcpy(d, s, size);
        break;
      }
      default:
        t.status = 4;
        return;
    }
  }
}

__global__ void vm_kernel(const VmOp* prog, int nops, int nbuf, const int64_t* bases, const int32_t* lens,
                          const int32_t* offs, uint8_t* region, int64_t stride, uint8_t* shared_region,
                          int32_t shared_bytes, int count, int strict, int32_t* status, int64_t* fault) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  Th t;
  for (int i = 0; i < NREG / 32; ++i) t.valid[i] = 0u;
  for (int i = 0; i < NREG; ++i) t.R[i] = 0u;
  t.P = 0u;
  t.strict = strict;
  t.status = 0;
  t.fault = 0;
  Mem m;
  m.region = region + (size_t)s * stride;
  m.shared = shared_region ? shared_region + (size_t)s * shared_bytes : nullptr;
  if (m.shared)
    for (int i = 0; i < shared_bytes; ++i) m.shared[i] = 0;
  m.shared_bytes = shared_region ? shared_bytes : 0;
  m.nbuf = nbuf;
  m.bases = bases;
  m.lens = lens;
  m.offs = offs;
  exec(prog, nops, t, m);
  status[s] = t.status;
  fault[s] = t.fault;
}

// first differing cell of the ret buffer per sample (-1 = identical)
__global__ void cell_diff_kernel(const uint8_t* a, const uint8_t* b, int64_t stride, int32_t off, int32_t nbytes,
                                 int32_t cell, int count, int32_t* first) {
  int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= count) return;
  const uint8_t* x = a + (size_t)s * stride + off;
  const uint8_t* y = b + (size_t)s * stride + off;
  int f = -1;
  for (int i = 0; i < nbytes; ++i)
    if (x[i] != y[i]) {
      f = i / cell;
      break;
    }
  first[s] = f;
}

}  // namespace

extern "C" {

int sip_vm_exec(sip_ctx* ctx, const void* prog, int32_t nops, int32_t nbuf, const int64_t* bases,
                const int32_t* lens, const int32_t* offs, void* region, int64_t stride, int32_t count,
                int32_t shared_bytes, int32_t strict, int32_t* status, int64_t* fault) {
  if (!ctx || (!prog && nops) || nops < 0 || count < 0 || nbuf < 0 || !region || !status || !fault)
    return SIP_E_ARG;
  if (count == 0) return SIP_OK;
  VmOp* d_prog = nullptr;
  int64_t* d_bases = nullptr;
  int32_t *d_lens = nullptr, *d_offs = nullptr, *d_status = nullptr;
  int64_t* d_fault = nullptr;
  uint8_t* d_shared = nullptr;
  cudaStream_t st = ctx->stream;
  SIP_CUDA(ctx, cudaMallocAsync(&d_prog, sizeof(VmOp) * (nops ? nops : 1), st));
  SIP_CUDA(ctx, cudaMallocAsync(&d_bases, sizeof(int64_t) * (nbuf ? nbuf : 1), st));
  SIP_CUDA(ctx, cudaMallocAsync(&d_lens, sizeof(int32_t) * (nbuf ? nbuf : 1), st));
  SIP_CUDA(ctx, cudaMallocAsync(&d_offs, sizeof(int32_t) * (nbuf ? nbuf : 1), st));
  SIP_CUDA(ctx, cudaMallocAsync(&d_status, sizeof(int32_t) * count, st));
  SIP_CUDA(ctx, cudaMallocAsync(&d_fault, sizeof(int64_t) * count, st));
  if (shared_bytes > 0) SIP_CUDA(ctx, cudaMallocAsync(&d_shared, (size_t)shared_bytes * count, st));
  if (nops) SIP_CUDA(ctx, cudaMemcpyAsync(d_prog, prog, sizeof(VmOp) * nops, cudaMemcpyHostToDevice, st));
  if (nbuf) {
    SIP_CUDA(ctx, cudaMemcpyAsync(d_bases, bases, sizeof(int64_t) * nbuf, cudaMemcpyHostToDevice, st));
    SIP_CUDA(ctx, cudaMemcpyAsync(d_lens, lens, sizeof(int32_t) * nbuf, cudaMemcpyHostToDevice, st));
    SIP_CUDA(ctx, cudaMemcpyAsync(d_offs, offs, sizeof(int32_t) * nbuf, cudaMemcpyHostToDevice, st));
  }
  vm_kernel<<<(count + 63) / 64, 64, 0, st>>>(d_prog, nops, nbuf, d_bases, d_lens, d_offs,
                                              static_cast<uint8_t*>(region), stride, d_shared, shared_bytes,
                                              count, strict, d_status, d_fault);
  SIP_CHECK_LAUNCH(ctx);
  SIP_CUDA(ctx, cudaMemcpyAsync(status, d_status, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, st));
  SIP_CUDA(ctx, cudaMemcpyAsync(fault, d_fault, sizeof(int64_t) * count, cudaMemcpyDeviceToHost, st));
  void* ptrs[] = {d_prog, d_bases, d_lens, d_offs, d_status, d_fault, d_shared};
  for (void* p : ptrs)
    if (p) cudaFreeAsync(p, st);
  SIP_CUDA(ctx, cudaStreamSynchronize(st));
  return SIP_OK;
}

int sip_vm_cell_diff(sip_ctx* ctx, const void* a, const void* b, int64_t stride, int32_t off, int32_t nbytes,
                     int32_t cell, int32_t count, int32_t* first_cell) {
  if (!ctx || !a || !b || !first_cell || count < 0 || cell < 1) return SIP_E_ARG;
  if (count == 0) return SIP_OK;
  int32_t* d = nullptr;
  SIP_CUDA(ctx, cudaMallocAsync(&d, sizeof(int32_t) * count, ctx->stream));
  cell_diff_kernel<<<(count + 127) / 128, 128, 0, ctx->stream>>>(static_cast<const uint8_t*>(a),
                                                                 static_cast<const uint8_t*>(b), stride, off,
                                                                 nbytes, cell, count, d);
  SIP_CHECK_LAUNCH(ctx);
  SIP_CUDA(ctx, cudaMemcpyAsync(first_cell, d, sizeof(int32_t) * count, cudaMemcpyDeviceToHost, ctx->stream));
  cudaFreeAsync(d, ctx->stream);
  SIP_CUDA(ctx, cudaStreamSynchronize(ctx->stream));
  return SIP_OK;
}

}  // extern "C"
