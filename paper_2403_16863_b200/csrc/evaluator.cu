// evaluator.cu -- G3 cubin frontend / re-encoder and G4 candidate evaluator.
//
// Replaces the reference's measurement path: backends.ExternalCommandBackend
// (backends.py:66-116) spawning an adapter process per repetition
// (frontend/src/measure.ts:66-85).  Here a candidate schedule is a
// permutation of the kernel's 128-bit instruction words: the re-encoder
// gathers the words of .text.<func> in schedule order, the driver loads the
// patched image with cuModuleLoadData, and warmup + reps launches are
// replayed from one CUDA graph with an event pair around every timed launch.
//
// Offset-bearing metadata: instructions named by EIATTR offset
// lists in .nv.info.<func> and by relocations against .text.<func> are
// reported as pinned (sip_module_pins) so the search never moves them;
// branch targets are block cuts in the listing, so block starts never move.
#include <elf.h>

#include <algorithm>
#include <atomic>
#include <memory>
#include <cstring>
#include <list>
#include <string>
#include <chrono>
#include <thread>
#include <unordered_map>
#include <vector>

#include "common.h"

namespace {

struct Sec {
  std::string name;
  uint32_t type;
  uint64_t off, size;
  uint32_t link, info;
  uint64_t entsize;
  size_t hdr_off;  // offset of the section header in the image
};

bool parse_sections(const std::vector<uint8_t>& img, std::vector<Sec>& out, std::string& err) {
  if (img.size() < sizeof(Elf64_Ehdr) || std::memcmp(img.data(), ELFMAG, SELFMAG) != 0) {
    err = "not an ELF image";
    return false;
  }
  Elf64_Ehdr eh;
  std::memcpy(&eh, img.data(), sizeof eh);
  if (eh.e_ident[EI_CLASS] != ELFCLASS64 || eh.e_shentsize != sizeof(Elf64_Shdr)) {
    err = "not an ELF64 cubin";
    return false;
  }
  if (eh.e_shoff + (uint64_t)eh.e_shnum * sizeof(Elf64_Shdr) > img.size()) {
    err = "section table out of range";
    return false;
  }
  std::vector<Elf64_Shdr> sh(eh.e_shnum);
  std::memcpy(sh.data(), img.data() + eh.e_shoff, sizeof(Elf64_Shdr) * eh.e_shnum);
  if (eh.e_shstrndx >= eh.e_shnum) {
    err = "bad shstrndx";
    return false;
  }
  const Elf64_Shdr& ss = sh[eh.e_shstrndx];
  for (size_t i = 0; i < sh.size(); ++i) {
    Sec s;
    uint64_t no = ss.sh_offset + sh[i].sh_name;
    if (no >= img.size()) {
      err = "section name out of range";
      return false;
    }
    s.name = std::string(reinterpret_cast<const char*>(img.data() + no));
    s.type = sh[i].sh_type;
    s.off = sh[i].sh_offset;
    s.size = sh[i].sh_size;
    s.link = sh[i].sh_link;
    s.info = sh[i].sh_info;
    s.entsize = sh[i].sh_entsize;
    s.hdr_off = eh.e_shoff + i * sizeof(Elf64_Shdr);
    if (s.type != SHT_NOBITS && s.off + s.size > img.size()) {
      err = "section " + s.name + " out of range";
      return false;
    }
    out.push_back(s);
  }
  return true;
}

// EIATTR attributes whose SVAL payload is a list of u32 instruction offsets.
bool is_offset_list(uint8_t attr) {
  switch (attr) {
    case 0x14:  // BINDLESS_IMAGE_OFFSETS
    case 0x1c:  // EXIT_INSTR_OFFSETS
    case 0x1d:  // S2RCTAID_INSTR_OFFSETS
    case 0x25:  // LD_CACHEMOD_INSTR_OFFSETS
    case 0x27:  // ATOM_SYS_INSTR_OFFSETS
    case 0x28:  // COOP_GROUP_INSTR_OFFSETS
    case 0x2d:  // ATOMF16_EMUL_INSTR_OFFSETS
    case 0x31:  // INT_WARP_WIDE_INSTR_OFFSETS
    case 0x34:  // INDIRECT_BRANCH_TARGETS
    case 0x39:  // MBARRIER_INSTR_OFFSETS
    case 0x3a:  // COROUTINE_RESUME_ID_OFFSETS
      return true;
    default:
      return false;
  }
}

struct CachedMod {
  std::vector<uint16_t> perm;
  CUmodule mod = nullptr;
  CUfunction fn = nullptr;
  uint32_t smem_set = 0;
  uint64_t stamp = 0;
  bool pinned = false;  // in use by the batch being measured: never evicted
};

}  // namespace

struct sip_module {
  sip_ctx* ctx = nullptr;
  std::vector<uint8_t> image;       // the cubin as given (sip_module_patch emits from it)
  std::vector<uint8_t> load_image;  // the same without debug-section data: what is loaded
  uint64_t load_text_off = 0;       // .text offset inside load_image
  std::string func;
  uint64_t text_off = 0, text_size = 0;
  int n = 0;
  std::vector<uint8_t> pin;
  std::vector<uint8_t> patched;
  // loaded schedules in least-recently-used order (front = oldest); std::list keeps
  // addresses stable (callers hold CachedMod* across loads) and splice is O(1).
  // `index` maps a hash of the schedule to its entries, so a lookup is O(1) rather than
  // a scan of every loaded schedule (which made 16 k-candidate rounds lookup-bound).
  std::list<CachedMod> cache;
  std::unordered_multimap<uint64_t, std::list<CachedMod>::iterator> index;
  size_t cache_cap = 4;  // modules kept loaded (raised for a batch)
  uint64_t clock = 0;
  std::vector<cudaEvent_t> events;
};

namespace {

int neutralize_merc(sip_module* m, std::vector<uint8_t>& img) {
  // Rename .nv.capmerc.* / .nv.merc.* so that a loader keyed on those names sees only the
  // (patched) SASS.  The driver runs the patched .text either way (the canary test passes in
  // both modes), but without them cuModuleLoadData is ~27 % faster (a 35-candidate GEMM
  // round: 6.3 -> 4.6 ms of loading).  SIP_MERC_MODE=0 keeps the sections.
  const char* mode = getenv("SIP_MERC_MODE");
  if (mode && mode[0] == '0') return SIP_OK;
  std::vector<Sec> secs;
  std::string err;
  if (!parse_sections(img, secs, err)) return sip::fail(m->ctx, SIP_E_ELF, err);
  Elf64_Ehdr eh;
  std::memcpy(&eh, img.data(), sizeof eh);
  Elf64_Shdr ss;
  std::memcpy(&ss, img.data() + eh.e_shoff + eh.e_shstrndx * sizeof(Elf64_Shdr), sizeof ss);
  for (auto& s : secs) {
    if (s.name.rfind(".nv.capmerc", 0) == 0 || s.name.rfind(".nv.merc", 0) == 0) {
      Elf64_Shdr h;
      std::memcpy(&h, img.data() + s.hdr_off, sizeof h);
      char* nm = reinterpret_cast<char*>(img.data() + ss.sh_offset + h.sh_name);
      nm[4] = 'x';  // ".nv.xapmerc..." / ".nv.xerc..."
    }
  }
  return SIP_OK;
}

// Debug sections (-lineinfo: DWARF line tables, SASS/PTX line maps, the embedded PTX text
// and their .nv.merc copies) do not change the code, but the driver's cuModuleLoadData
// cost grows with the modules a process has loaded, far faster for images that carry
// them.  Candidates are loaded from a copy rebuilt without their data:
// the kept sections' byte ranges are repacked (each keeps its offset modulo 1024, so every
// alignment holds), section and program headers are remapped, and the debug sections
// stay in the header table with size 0 so section indices do not change.
bool is_debug_section(const std::string& name) {
  static const char* const prefixes[] = {".debug_", ".nv_debug_", ".rela.debug_", ".rela.nv_debug_",
                                         ".nv.merc.debug_", ".nv.merc.nv_debug_", ".nv.merc.rela.debug_",
                                         ".nv.merc.rela.nv_debug_"};
  for (const char* p : prefixes)
    if (name.rfind(p, 0) == 0) return true;
  return false;
}

bool strip_debug(const std::vector<uint8_t>& img, const std::vector<Sec>& secs, std::vector<uint8_t>& out) {
  Elf64_Ehdr eh;
  std::memcpy(&eh, img.data(), sizeof eh);
  if (eh.e_phentsize != sizeof(Elf64_Phdr) && eh.e_phnum) return false;
  if (eh.e_phoff + (uint64_t)eh.e_phnum * sizeof(Elf64_Phdr) > img.size()) return false;
  bool any = false;
  std::vector<std::pair<uint64_t, uint64_t>> ranges;  // kept file data [begin, end)
  for (const auto& x : secs) {
    if (is_debug_section(x.name)) {
      any = true;
      continue;
    }
    if (x.type == SHT_NOBITS || x.type == SHT_NULL || x.size == 0) continue;
    if (x.off + x.size > img.size()) return false;
    ranges.push_back({x.off, x.off + x.size});
  }
  if (!any) return false;
  std::sort(ranges.begin(), ranges.end());
  std::vector<std::pair<uint64_t, uint64_t>> merged;
  for (auto& r : ranges)
    if (!merged.empty() && r.first <= merged.back().second)
      merged.back().second = std::max(merged.back().second, r.second);
    else
      merged.push_back(r);
  std::vector<uint64_t> new_start(merged.size());
  uint64_t cur = sizeof(Elf64_Ehdr);
  for (size_t i = 0; i < merged.size(); ++i) {
    uint64_t want = merged[i].first % 1024;
    uint64_t base = cur - cur % 1024 + want;
    if (base < cur) base += 1024;
    new_start[i] = base;
    cur = base + (merged[i].second - merged[i].first);
  }
  auto map_off = [&](uint64_t off, bool& ok) -> uint64_t {
    for (size_t i = 0; i < merged.size(); ++i)
      if (off >= merged[i].first && off <= merged[i].second) return new_start[i] + (off - merged[i].first);
    ok = false;
    return 0;
  };
  const uint64_t phoff = (cur + 7) & ~7ull;
  const uint64_t shoff = (phoff + (uint64_t)eh.e_phnum * sizeof(Elf64_Phdr) + 7) & ~7ull;
  out.assign(shoff + (uint64_t)eh.e_shnum * sizeof(Elf64_Shdr), 0);
  for (size_t i = 0; i < merged.size(); ++i)
    std::memcpy(out.data() + new_start[i], img.data() + merged[i].first, merged[i].second - merged[i].first);
  bool ok = true;
  for (int i = 0; i < eh.e_phnum; ++i) {
    Elf64_Phdr ph;
    std::memcpy(&ph, img.data() + eh.e_phoff + i * sizeof ph, sizeof ph);
    if (ph.p_offset == eh.e_phoff) {
      ph.p_offset = phoff;  // the program header table itself (PT_PHDR and its PT_LOAD)
    } else if (ph.p_filesz > 0 || ph.p_offset != 0) {
      bool hit = true;
      const uint64_t o = map_off(ph.p_offset, hit);
      if (hit) ph.p_offset = o;
      else if (ph.p_filesz > 0) ok = false;
    }
    std::memcpy(out.data() + phoff + i * sizeof ph, &ph, sizeof ph);
  }
  for (int i = 0; i < eh.e_shnum; ++i) {
    Elf64_Shdr sh;
    std::memcpy(&sh, img.data() + eh.e_shoff + i * sizeof sh, sizeof sh);
    if (i < (int)secs.size() && is_debug_section(secs[i].name)) {
      sh.sh_offset = 0;
      sh.sh_size = 0;
    } else if (sh.sh_type != SHT_NULL) {
      bool hit = true;
      const uint64_t o = map_off(sh.sh_offset, hit);
      if (hit) sh.sh_offset = o;
      else if (sh.sh_type != SHT_NOBITS && sh.sh_size > 0) ok = false;
      else sh.sh_offset = 0;  // an empty section between removed ranges
    }
    std::memcpy(out.data() + shoff + i * sizeof sh, &sh, sizeof sh);
  }
  eh.e_phoff = eh.e_phnum ? phoff : 0;
  eh.e_shoff = shoff;
  std::memcpy(out.data(), &eh, sizeof eh);
  return ok;
}

bool is_permutation(const sip_module* m, const uint16_t* perm) {
  std::vector<uint8_t> seen(m->n, 0);
  for (int i = 0; i < m->n; ++i) {
    const int p = perm[i];
    if (p >= m->n || seen[p]) return false;
    seen[p] = 1;
  }
  return true;
}

// the image for schedule `perm` (a permutation the caller has checked): the template's
// .text words gathered in schedule order.  Touches no shared state, so the evaluator's
// worker threads build their candidates' images themselves.
void gather_image(const sip_module* m, const uint16_t* perm, std::vector<uint8_t>& out, bool for_load) {
  out = for_load ? m->load_image : m->image;
  if (!perm) return;
  const uint8_t* src = m->image.data() + m->text_off;
  uint8_t* dst = out.data() + (for_load ? m->load_text_off : m->text_off);
  for (int i = 0; i < m->n; ++i) std::memcpy(dst + 16 * (size_t)i, src + 16 * (size_t)perm[i], 16);
}

int build_image(sip_module* m, const uint16_t* perm, std::vector<uint8_t>& out, bool for_load = true) {
  if (perm && !is_permutation(m, perm)) return sip::fail(m->ctx, SIP_E_ARG, "perm is not a permutation");
  // the load image already had its merc sections renamed at sip_module_open; a patched
  // cubin written out keeps them
  gather_image(m, perm, out, for_load);
  return SIP_OK;
}

int cu_fail(sip_ctx* ctx, int code, const char* what, CUresult r) {
  const char* s = nullptr;
  if (ctx->cuGetErrorString) ctx->cuGetErrorString(r, &s);
  return sip::fail(ctx, code, std::string(what) + ": " + (s ? s : "CUDA driver error"));
}

uint64_t perm_hash(const std::vector<uint16_t>& key) {
  uint64_t h = 1469598103934665603ull;  // FNV-1a over the 16-bit entries
  for (uint16_t v : key) h = (h ^ v) * 1099511628211ull;
  return h ^ key.size();
}

// the loaded module for schedule `key` (moved to the most-recently-used end), or null
CachedMod* find_module(sip_module* m, const std::vector<uint16_t>& key) {
  auto range = m->index.equal_range(perm_hash(key));
  for (auto it = range.first; it != range.second; ++it)
    if (it->second->perm == key) {
      m->cache.splice(m->cache.end(), m->cache, it->second);
      it->second->stamp = ++m->clock;
      return &*it->second;
    }
  return nullptr;
}

CachedMod* insert_module(sip_module* m, CachedMod&& cm) {
  m->cache.push_back(std::move(cm));
  auto it = std::prev(m->cache.end());
  m->index.emplace(perm_hash(it->perm), it);
  return &*it;
}

// unload the least recently used module that no batch in flight is holding
void evict_one(sip_module* m) {
  auto victim = m->cache.begin();
  while (victim != m->cache.end() && victim->pinned) ++victim;  // pinned entries are recent
  if (victim == m->cache.end()) return;
  auto range = m->index.equal_range(perm_hash(victim->perm));
  for (auto it = range.first; it != range.second; ++it)
    if (it->second == victim) {
      m->index.erase(it);
      break;
    }
  m->ctx->cuModuleUnload(victim->mod);
  m->cache.erase(victim);
}

int get_module(sip_module* m, const uint16_t* perm, CachedMod** out) {
  std::vector<uint16_t> key;
  if (perm) key.assign(perm, perm + m->n);
  if (CachedMod* hit = find_module(m, key)) {
    *out = hit;
    return SIP_OK;
  }
  std::vector<uint8_t> img;
  int rc = build_image(m, perm, img);
  if (rc != SIP_OK) return rc;
  sip_ctx* ctx = m->ctx;
  CachedMod cm;
  cm.perm = key;
  CUresult r = ctx->cuModuleLoadData(&cm.mod, img.data());
  if (r != CUDA_SUCCESS) return cu_fail(ctx, SIP_E_MEASURE, "cuModuleLoadData", r);
  r = ctx->cuModuleGetFunction(&cm.fn, cm.mod, m->func.c_str());
  if (r != CUDA_SUCCESS) {
    ctx->cuModuleUnload(cm.mod);
    return cu_fail(ctx, SIP_E_MEASURE, "cuModuleGetFunction", r);
  }
  cm.stamp = ++m->clock;
  if (m->cache.size() >= m->cache_cap) evict_one(m);
  *out = insert_module(m, std::move(cm));
  return SIP_OK;
}

int launch(sip_module* m, CachedMod* cm, const sip_launch* L) {
  sip_ctx* ctx = m->ctx;
  if (L->smem_bytes > 48 * 1024 && cm->smem_set < L->smem_bytes) {
    CUresult r = ctx->cuFuncSetAttribute(cm->fn, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                         (int)L->smem_bytes);
    if (r != CUDA_SUCCESS) return cu_fail(ctx, SIP_E_MEASURE, "cuFuncSetAttribute", r);
    cm->smem_set = L->smem_bytes;
  }
  std::vector<void*> args(L->nparams);
  for (uint32_t i = 0; i < L->nparams; ++i)
    args[i] = const_cast<uint8_t*>(static_cast<const uint8_t*>(L->params) + L->param_offsets[i]);
  CUlaunchConfig cfg;
  std::memset(&cfg, 0, sizeof cfg);
  cfg.gridDimX = L->grid[0];
  cfg.gridDimY = std::max(1u, L->grid[1]);
  cfg.gridDimZ = std::max(1u, L->grid[2]);
  cfg.blockDimX = L->block[0];
  cfg.blockDimY = std::max(1u, L->block[1]);
  cfg.blockDimZ = std::max(1u, L->block[2]);
  cfg.sharedMemBytes = L->smem_bytes;
  cfg.hStream = (CUstream)ctx->stream;
  CUlaunchAttribute attr[1];
  uint32_t cx = std::max(1u, L->cluster[0]), cy = std::max(1u, L->cluster[1]), cz = std::max(1u, L->cluster[2]);
  if (cx * cy * cz > 1) {
    attr[0].id = CU_LAUNCH_ATTRIBUTE_CLUSTER_DIMENSION;
    attr[0].value.clusterDim.x = cx;
    attr[0].value.clusterDim.y = cy;
    attr[0].value.clusterDim.z = cz;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
  }
  CUresult r = ctx->cuLaunchKernelEx(&cfg, cm->fn, args.data(), nullptr);
  if (r != CUDA_SUCCESS) return cu_fail(ctx, SIP_E_MEASURE, "cuLaunchKernelEx", r);
  return SIP_OK;
}

int ensure_flush(sip_ctx* ctx) {
  if (ctx->flush_buf) return SIP_OK;
  ctx->flush_bytes = 256ull << 20;  // 2x the 126 MB L2
  SIP_CUDA(ctx, cudaMalloc(&ctx->flush_buf, ctx->flush_bytes));
  return SIP_OK;
}

}  // namespace

extern "C" {

int sip_module_open(sip_ctx* ctx, const void* cubin, size_t size, const char* func,
                    sip_module** out) {
  // ctx may be NULL: parse-only use (listing frontend, pins, patching) on a host without a GPU
  if (!cubin || !func || !out || size == 0) return SIP_E_ARG;
  auto* m = new sip_module();
  m->ctx = ctx;
  m->func = func;
  m->image.assign(static_cast<const uint8_t*>(cubin), static_cast<const uint8_t*>(cubin) + size);
  std::vector<Sec> secs;
  std::string err;
  if (!parse_sections(m->image, secs, err)) {
    delete m;
    return sip::fail(ctx, SIP_E_ELF, err);
  }
  const std::string tname = ".text." + m->func, iname = ".nv.info." + m->func;
  int tidx = -1;
  for (size_t i = 0; i < secs.size(); ++i)
    if (secs[i].name == tname) tidx = (int)i;
  if (tidx < 0) {
    delete m;
    return sip::fail(ctx, SIP_E_ELF, "no section " + tname);
  }
  m->text_off = secs[tidx].off;
  m->text_size = secs[tidx].size;
  if (m->text_size % 16 != 0 || m->text_size / 16 > 65535) {
    delete m;
    return sip::fail(ctx, SIP_E_ELF, tname + " size is not a multiple of 16 or too large");
  }
  m->n = (int)(m->text_size / 16);
  m->pin.assign(m->n, 0);
  auto pin_off = [&](uint64_t off) {
    if (off < m->text_size) m->pin[off / 16] = 1;
  };
  for (auto& s : secs) {
    if (s.name == iname) {  // EIATTR records: u8 format, u8 attribute, payload
      const uint8_t* b = m->image.data() + s.off;
      size_t i = 0;
      while (i + 2 <= s.size) {
        uint8_t fmt = b[i], attr = b[i + 1];
        if (fmt == 0x04) {
          if (i + 4 > s.size) break;
          uint16_t len;
          std::memcpy(&len, b + i + 2, 2);
          if (is_offset_list(attr))
            for (size_t k = 0; k + 4 <= len && i + 4 + k + 4 <= s.size; k += 4) {
              uint32_t v;
              std::memcpy(&v, b + i + 4 + k, 4);
              pin_off(v);
            }
          i += 4 + len;
        } else if (fmt == 0x01) {
          i += 2;
        } else {
          i += 4;  // BVAL / HVAL: 2-byte header + 2-byte value
        }
      }
    }
    if ((s.type == SHT_RELA || s.type == SHT_REL) && s.info == (uint32_t)tidx) {
      size_t ent = s.type == SHT_RELA ? sizeof(Elf64_Rela) : sizeof(Elf64_Rel);
      for (size_t o = 0; o + ent <= s.size; o += ent) {
        uint64_t roff;
        std::memcpy(&roff, m->image.data() + s.off + o, 8);
        pin_off(roff);
      }
    }
  }
  m->load_image = m->image;
  m->load_text_off = m->text_off;
  std::vector<uint8_t> stripped;
  if (!getenv("SIP_KEEP_DEBUG") && strip_debug(m->image, secs, stripped)) {
    std::vector<Sec> s2;
    std::string e2;
    if (parse_sections(stripped, s2, e2) && (size_t)tidx < s2.size() && s2[tidx].size == m->text_size &&
        std::memcmp(stripped.data() + s2[tidx].off, m->image.data() + m->text_off, m->text_size) == 0) {
      m->load_image.swap(stripped);
      m->load_text_off = s2[tidx].off;
    }
  }
  // images the driver loads drop the merc sections (renamed once here, not per candidate)
  if (int rc = neutralize_merc(m, m->load_image); rc != SIP_OK) {
    delete m;
    return rc;
  }
  *out = m;
  return SIP_OK;
}

int sip_module_close(sip_module* m) {
  if (!m) return SIP_OK;
  for (auto& c : m->cache)
    if (c.mod && m->ctx) m->ctx->cuModuleUnload(c.mod);
  for (auto e : m->events) cudaEventDestroy(e);
  delete m;
  return SIP_OK;
}

int sip_module_info(sip_module* m, int32_t* n_instr, uint64_t* text_offset) {
  if (!m) return SIP_E_ARG;
  if (n_instr) *n_instr = m->n;
  if (text_offset) *text_offset = m->text_off;
  return SIP_OK;
}

int sip_module_words(sip_module* m, uint64_t* words) {
  if (!m || !words) return SIP_E_ARG;
  std::memcpy(words, m->image.data() + m->text_off, m->text_size);
  return SIP_OK;
}

int sip_module_pins(sip_module* m, uint8_t* pin) {
  if (!m || !pin) return SIP_E_ARG;
  std::memcpy(pin, m->pin.data(), m->n);
  return SIP_OK;
}

int sip_module_patch(sip_module* m, const uint16_t* perm, void* out, size_t* size) {
  if (!m || !size) return SIP_E_ARG;
  std::vector<uint8_t> img;
  // SIP_PATCH_LOAD_IMAGE=1 emits the image the evaluator loads (debug data removed; tests)
  int rc = build_image(m, perm, img, /*for_load=*/getenv("SIP_PATCH_LOAD_IMAGE") != nullptr);
  if (rc != SIP_OK) return rc;
  if (!out) {
    *size = img.size();
    return SIP_OK;
  }
  if (*size < img.size()) return sip::fail(m->ctx, SIP_E_ARG, "output buffer too small");
  std::memcpy(out, img.data(), img.size());
  *size = img.size();
  return SIP_OK;
}

int sip_run(sip_module* m, const uint16_t* perm, const sip_launch* L) {
  if (!m || !L || !m->ctx) return SIP_E_ARG;
  sip_ctx* ctx = m->ctx;
  CachedMod* cm = nullptr;
  int rc = get_module(m, perm, &cm);
  if (rc != SIP_OK) return rc;
  rc = launch(m, cm, L);
  if (rc != SIP_OK) return rc;
  cudaError_t e = cudaStreamSynchronize(ctx->stream);
  if (e != cudaSuccess)
    return sip::fail(ctx, SIP_E_MEASURE, std::string("candidate execution: ") + cudaGetErrorString(e));
  return SIP_OK;
}

int sip_run_async(sip_module* m, const uint16_t* perm, const sip_launch* L) {
  if (!m || !L || !m->ctx) return SIP_E_ARG;
  CachedMod* cm = nullptr;
  int rc = get_module(m, perm, &cm);
  if (rc != SIP_OK) return rc;
  return launch(m, cm, L);
}

// warmup launches of every module, then `reps` rounds; round r launches the
// modules in rotated order (ABAB.. / BABA..), each bracketed by an event pair
// and preceded by an optional L2 flush.  Everything runs from one CUDA graph.
static int run_timed(sip_module* m, CachedMod** mods, int nm, const sip_launch* L, int warmup, int reps,
                     int flush_l2, std::vector<std::vector<double>>& times) {
  sip_ctx* ctx = m->ctx;
  int rc = SIP_OK;
  if (flush_l2 && (rc = ensure_flush(ctx)) != SIP_OK) return rc;
  const int nev = 2 * reps * nm;
  while ((int)m->events.size() < nev) {
    cudaEvent_t e;
    SIP_CUDA(ctx, cudaEventCreate(&e));
    m->events.push_back(e);
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  SIP_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  for (int w = 0; w < warmup && rc == SIP_OK; ++w)
    for (int i = 0; i < nm && rc == SIP_OK; ++i) rc = launch(m, mods[i], L);
  for (int r = 0; r < reps && rc == SIP_OK; ++r)
    for (int q = 0; q < nm && rc == SIP_OK; ++q) {
      const int i = (q + r) % nm;
      const int e = 2 * (r * nm + i);
      if (flush_l2) cudaMemsetAsync(ctx->flush_buf, (r * nm + q) & 0xff, ctx->flush_bytes, ctx->stream);
      cudaEventRecordWithFlags(m->events[e], ctx->stream, cudaEventRecordExternal);
      rc = launch(m, mods[i], L);
      cudaEventRecordWithFlags(m->events[e + 1], ctx->stream, cudaEventRecordExternal);
    }
  cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc != SIP_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ce != cudaSuccess) return sip::fail(ctx, SIP_E_MEASURE, std::string("capture: ") + cudaGetErrorString(ce));
  ce = cudaGraphInstantiate(&exec, graph, 0);
  if (ce == cudaSuccess) ce = cudaGraphLaunch(exec, ctx->stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
  times.assign(nm, std::vector<double>(reps, 0.0));
  for (int r = 0; r < reps && ce == cudaSuccess; ++r)
    for (int i = 0; i < nm && ce == cudaSuccess; ++i) {
      float ms = 0.f;
      const int e = 2 * (r * nm + i);
      ce = cudaEventElapsedTime(&ms, m->events[e], m->events[e + 1]);
      times[i][r] = ms;
    }
  if (exec) cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess)
    return sip::fail(ctx, SIP_E_MEASURE, std::string("timed launches: ") + cudaGetErrorString(ce));
  return SIP_OK;
}

static double median_of(std::vector<double> v) {
  std::sort(v.begin(), v.end());
  size_t k = v.size();
  return k % 2 ? v[k / 2] : 0.5 * (v[k / 2 - 1] + v[k / 2]);
}

int sip_measure(sip_module* m, const uint16_t* perm, const sip_launch* L, int32_t warmup,
                int32_t reps, int32_t flush_l2, double* median_ms, double* raw_ms) {
  if (!m || !L || !m->ctx || !median_ms || reps < 1 || warmup < 0) return SIP_E_ARG;
  CachedMod* cm = nullptr;
  int rc = get_module(m, perm, &cm);
  if (rc != SIP_OK) return rc;
  std::vector<std::vector<double>> t;
  rc = run_timed(m, &cm, 1, L, warmup, reps, flush_l2, t);
  if (rc != SIP_OK) return rc;
  if (raw_ms) std::copy(t[0].begin(), t[0].end(), raw_ms);
  *median_ms = median_of(t[0]);
  return SIP_OK;
}

int sip_measure_paired(sip_module* m, const uint16_t* perm_ref, const uint16_t* perm_cand,
                       const sip_launch* L, int32_t warmup, int32_t reps, int32_t flush_l2,
                       double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                       double* raw_ratio) {
  if (!m || !L || !m->ctx || !ratio_median || reps < 1 || warmup < 0) return SIP_E_ARG;
  CachedMod* mods[2] = {nullptr, nullptr};
  int rc = get_module(m, perm_ref, &mods[0]);
  if (rc == SIP_OK) rc = get_module(m, perm_cand, &mods[1]);
  if (rc != SIP_OK) return rc;
  std::vector<std::vector<double>> t;
  rc = run_timed(m, mods, 2, L, warmup, reps, flush_l2, t);
  if (rc != SIP_OK) return rc;
  std::vector<double> ratio(reps);
  for (int r = 0; r < reps; ++r) ratio[r] = t[1][r] / t[0][r];
  if (raw_ratio) std::copy(ratio.begin(), ratio.end(), raw_ratio);
  *ratio_median = median_of(ratio);
  if (ref_median_ms) *ref_median_ms = median_of(t[0]);
  if (cand_median_ms) *cand_median_ms = median_of(t[1]);
  return SIP_OK;
}

// Batched paired timing (the hardware search prices one candidate per live chain per
// round): the candidates' cubins are patched and loaded on a few host threads, then
// every candidate's (warmup + reps) interleaved pairs with the baseline run from ONE
// CUDA graph, so the GPU does not idle between candidates for loads, graph builds and
// host round trips.  status[i] = SIP_OK or SIP_E_MEASURE (that candidate is skipped).
static int measure_batch_impl(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                              const sip_launch* L, int32_t warmup, int32_t reps, int32_t flush_l2,
                              double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                              double* raw_ratio, int32_t* status);
static int measure_round_impl(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                              const sip_launch* L, int32_t nL, int32_t warmup, int32_t reps, int32_t flush_l2,
                              double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                              double* raw_ratio, int32_t* status);
static int measure_round_streamed(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                                  const sip_launch* L, int32_t nL, int32_t warmup, int32_t reps,
                                  int32_t flush_l2, double* ratio_median, double* ref_median_ms,
                                  double* cand_median_ms, double* raw_ratio, int32_t* status);

int sip_measure_round(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                      const sip_launch* L, int32_t nL, int32_t warmup, int32_t reps, int32_t flush_l2,
                      double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                      double* raw_ratio, int32_t* status) {
  if (!m || !L || nL < 1 || !m->ctx || !perms || k < 1 || !ratio_median || !status || reps < 1 || warmup < 0)
    return SIP_E_ARG;
  static const bool graph = getenv("SIP_ROUND_GRAPH") != nullptr;  // the captured-graph round (A/B)
  const int rc = graph ? measure_round_impl(m, perm_ref, perms, k, L, nL, warmup, reps, flush_l2, ratio_median,
                                            ref_median_ms, cand_median_ms, raw_ratio, status)
                       : measure_round_streamed(m, perm_ref, perms, k, L, nL, warmup, reps, flush_l2,
                                                ratio_median, ref_median_ms, cand_median_ms, raw_ratio, status);
  for (auto& c : m->cache) c.pinned = false;
  // the round is done, so unloading no longer stalls it: keep the most recent modules only
  // (a driver holding thousands of modules loads new ones more slowly; SIP_MODULE_KEEP)
  static const size_t keep = getenv("SIP_MODULE_KEEP") ? (size_t)atol(getenv("SIP_MODULE_KEEP")) : 64;
  m->cache_cap = std::max<size_t>(keep, 4);
  while (m->cache.size() > m->cache_cap) {
    const size_t before = m->cache.size();
    evict_one(m);
    if (m->cache.size() == before) break;
  }
  return rc;
}

int sip_measure_paired_batch(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                             const sip_launch* L, int32_t warmup, int32_t reps, int32_t flush_l2,
                             double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                             double* raw_ratio, int32_t* status) {
  if (!m || !L || !m->ctx || !perms || k < 1 || !ratio_median || !status || reps < 1 || warmup < 0)
    return SIP_E_ARG;
  const int rc = measure_batch_impl(m, perm_ref, perms, k, L, warmup, reps, flush_l2, ratio_median,
                                    ref_median_ms, cand_median_ms, raw_ratio, status);
  for (auto& c : m->cache) c.pinned = false;  // the batch's modules may be evicted again
  return rc;
}

}  // extern "C"

// the reference module and every candidate's module of a batch, loaded (cache misses in
// parallel, SIP_LOAD_THREADS host threads) and pinned in the cache for the batch
static int load_batch(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                      CachedMod** ref_out, std::vector<CachedMod*>& mods, int32_t* status) {
  sip_ctx* ctx = m->ctx;
  if (m->cache_cap < (size_t)k + 1) m->cache_cap = (size_t)k + 1;
  CachedMod* ref = nullptr;
  int rc = get_module(m, perm_ref, &ref);
  if (rc != SIP_OK) return rc;
  ref->pinned = true;  // held by every pair of this batch
  *ref_out = ref;
  // images + parallel cuModuleLoadData for the candidates not loaded yet
  mods.assign(k, nullptr);
  std::vector<int> todo;
  for (int i = 0; i < k; ++i) {
    const uint16_t* p = perms + (size_t)i * m->n;
    std::vector<uint16_t> key(p, p + m->n);
    if (CachedMod* hit = find_module(m, key)) {
      hit->pinned = true;
      mods[i] = hit;
    }
    status[i] = SIP_OK;
    if (!mods[i]) todo.push_back(i);
  }
  std::vector<std::vector<uint8_t>> imgs(todo.size());
  std::vector<CUmodule> loaded(todo.size(), nullptr);
  std::vector<CUresult> lres(todo.size(), CUDA_SUCCESS);
  for (size_t t = 0; t < todo.size(); ++t)
    if (!is_permutation(m, perms + (size_t)todo[t] * m->n)) lres[t] = CUDA_ERROR_INVALID_IMAGE;
  // the loads run in this thread's CUDA context (made current in each worker), so the
  // modules belong to the context the launches below use
  CUcontext cur = nullptr;
  if (ctx->cuCtxGetCurrent(&cur) != CUDA_SUCCESS || cur == nullptr) {
    SIP_CUDA(ctx, cudaFree(nullptr));  // bind this device's primary context
    ctx->cuCtxGetCurrent(&cur);
  }
  const char* lt = getenv("SIP_LOAD_THREADS");
  const int want = lt ? std::max(1, atoi(lt)) : 8;
  const int nthreads = (int)std::min<size_t>(todo.size(), (size_t)want);
  std::vector<std::thread> pool;
  for (int w = 0; w < nthreads; ++w)
    pool.emplace_back([&, w]() {
      const bool ctx_ok = ctx->cuCtxSetCurrent(cur) == CUDA_SUCCESS;
      for (size_t t = w; t < todo.size(); t += nthreads)
        if (lres[t] == CUDA_SUCCESS) {  // each worker gathers its own images (gather_image)
          gather_image(m, perms + (size_t)todo[t] * m->n, imgs[t], /*for_load=*/true);
          lres[t] = ctx_ok ? ctx->cuModuleLoadData(&loaded[t], imgs[t].data()) : CUDA_ERROR_INVALID_CONTEXT;
        }
    });
  for (auto& th : pool) th.join();
  for (size_t t = 0; t < todo.size(); ++t) {
    const int i = todo[t];
    if (lres[t] != CUDA_SUCCESS) {
      status[i] = SIP_E_MEASURE;
      continue;
    }
    CachedMod cm;
    cm.perm.assign(perms + (size_t)i * m->n, perms + (size_t)(i + 1) * m->n);
    cm.mod = loaded[t];
    if (ctx->cuModuleGetFunction(&cm.fn, cm.mod, m->func.c_str()) != CUDA_SUCCESS) {
      ctx->cuModuleUnload(cm.mod);
      status[i] = SIP_E_MEASURE;
      continue;
    }
    cm.stamp = ++m->clock;
    cm.pinned = true;
    if (m->cache.size() >= m->cache_cap) evict_one(m);  // the oldest module not in this batch
    mods[i] = insert_module(m, std::move(cm));
  }
  return SIP_OK;
}

static int measure_batch_impl(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                              const sip_launch* L, int32_t warmup, int32_t reps, int32_t flush_l2,
                              double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                              double* raw_ratio, int32_t* status) {
  sip_ctx* ctx = m->ctx;
  CachedMod* ref = nullptr;
  std::vector<CachedMod*> mods;
  int rc = load_batch(m, perm_ref, perms, k, &ref, mods, status);
  if (rc != SIP_OK) return rc;
  if (flush_l2 && (rc = ensure_flush(ctx)) != SIP_OK) return rc;
  const int nev = 4 * reps * k;
  while ((int)m->events.size() < nev) {
    cudaEvent_t e;
    SIP_CUDA(ctx, cudaEventCreate(&e));
    m->events.push_back(e);
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  SIP_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < k && rc == SIP_OK; ++i) {
    if (status[i] != SIP_OK) continue;
    CachedMod* pair[2] = {ref, mods[i]};
    for (int w = 0; w < warmup && rc == SIP_OK; ++w)
      for (int q = 0; q < 2 && rc == SIP_OK; ++q) rc = launch(m, pair[q], L);
    for (int r = 0; r < reps && rc == SIP_OK; ++r)
      for (int q = 0; q < 2 && rc == SIP_OK; ++q) {
        const int j = (q + r) % 2;  // rotate the order every rep
        const int e = 4 * (i * reps + r) + 2 * j;
        if (flush_l2) cudaMemsetAsync(ctx->flush_buf, (r * 2 + q) & 0xff, ctx->flush_bytes, ctx->stream);
        cudaEventRecordWithFlags(m->events[e], ctx->stream, cudaEventRecordExternal);
        rc = launch(m, pair[j], L);
        cudaEventRecordWithFlags(m->events[e + 1], ctx->stream, cudaEventRecordExternal);
      }
  }
  cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc != SIP_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ce != cudaSuccess) return sip::fail(ctx, SIP_E_MEASURE, std::string("capture: ") + cudaGetErrorString(ce));
  ce = cudaGraphInstantiate(&exec, graph, 0);
  if (ce == cudaSuccess) ce = cudaGraphLaunch(exec, ctx->stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
  for (int i = 0; i < k && ce == cudaSuccess; ++i) {
    if (status[i] != SIP_OK) continue;
    std::vector<double> tr(reps), tc(reps), ratio(reps);
    for (int r = 0; r < reps && ce == cudaSuccess; ++r) {
      float a = 0.f, b = 0.f;
      const int e = 4 * (i * reps + r);
      ce = cudaEventElapsedTime(&a, m->events[e], m->events[e + 1]);
      if (ce == cudaSuccess) ce = cudaEventElapsedTime(&b, m->events[e + 2], m->events[e + 3]);
      tr[r] = a;
      tc[r] = b;
      ratio[r] = b / a;
    }
    ratio_median[i] = median_of(ratio);
    if (ref_median_ms) ref_median_ms[i] = median_of(tr);
    if (cand_median_ms) cand_median_ms[i] = median_of(tc);
    if (raw_ratio) std::copy(ratio.begin(), ratio.end(), raw_ratio + (size_t)i * reps);
  }
  if (exec) cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess)
    return sip::fail(ctx, SIP_E_MEASURE, std::string("timed launches: ") + cudaGetErrorString(ce));
  return SIP_OK;
}

// One nvcc reference per round: the k candidates and the reference
// are warmed up once each, then every rep launches all k+1 modules once in an order
// rotated by one slot per rep, each launch bracketed by an event pair.  Launch slot q of
// the graph uses parameter set L[q % nL]: with nL >= 3 buffer sets larger than L2 in
// rotation, no launch finds its inputs in L2 and no flush is needed (flush_l2 = 0); with
// flush_l2 the 256 MB memset precedes every timed launch as before.  A candidate's energy
// is the median over reps of its time / the reference's time in the same rep.
static int measure_round_impl(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                              const sip_launch* L, int32_t nL, int32_t warmup, int32_t reps, int32_t flush_l2,
                              double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                              double* raw_ratio, int32_t* status) {
  sip_ctx* ctx = m->ctx;
  CachedMod* ref = nullptr;
  std::vector<CachedMod*> mods;
  static const bool timing = getenv("SIP_EVAL_TIMING") != nullptr;
  const auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t_begin = now();
  int rc = load_batch(m, perm_ref, perms, k, &ref, mods, status);
  if (rc != SIP_OK) return rc;
  const auto t_loaded = now();
  if (flush_l2 && (rc = ensure_flush(ctx)) != SIP_OK) return rc;
  // the round's modules: slot 0 = the reference, then the loadable candidates
  std::vector<CachedMod*> set{ref};
  std::vector<int> cand_of;  // set index -> candidate index
  cand_of.push_back(-1);
  for (int i = 0; i < k; ++i)
    if (status[i] == SIP_OK) {
      set.push_back(mods[i]);
      cand_of.push_back(i);
    }
  const int nm = (int)set.size();
  const int nev = 2 * reps * nm;
  while ((int)m->events.size() < nev) {
    cudaEvent_t e;
    SIP_CUDA(ctx, cudaEventCreate(&e));
    m->events.push_back(e);
  }
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int slot = 0;
  SIP_CUDA(ctx, cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
  for (int w = 0; w < warmup && rc == SIP_OK; ++w)
    for (int q = 0; q < nm && rc == SIP_OK; ++q) rc = launch(m, set[q], &L[slot++ % nL]);
  for (int r = 0; r < reps && rc == SIP_OK; ++r)
    for (int q = 0; q < nm && rc == SIP_OK; ++q) {
      const int j = (q + r) % nm;  // rotate the order every rep
      const int e = 2 * (r * nm + j);
      if (flush_l2) cudaMemsetAsync(ctx->flush_buf, (r * nm + q) & 0xff, ctx->flush_bytes, ctx->stream);
      cudaEventRecordWithFlags(m->events[e], ctx->stream, cudaEventRecordExternal);
      rc = launch(m, set[j], &L[slot++ % nL]);
      cudaEventRecordWithFlags(m->events[e + 1], ctx->stream, cudaEventRecordExternal);
    }
  cudaError_t ce = cudaStreamEndCapture(ctx->stream, &graph);
  if (rc != SIP_OK) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ce != cudaSuccess) return sip::fail(ctx, SIP_E_MEASURE, std::string("capture: ") + cudaGetErrorString(ce));
  const auto t_captured = now();
  ce = cudaGraphInstantiate(&exec, graph, 0);
  const auto t_inst = now();
  if (ce == cudaSuccess) ce = cudaGraphLaunch(exec, ctx->stream);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(ctx->stream);
  if (timing) {
    const auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[sip round] k=%d load %.3f capture %.3f instantiate %.3f execute %.3f ms\n", k,
            ms(t_begin, t_loaded), ms(t_loaded, t_captured), ms(t_captured, t_inst), ms(t_inst, now()));
  }
  std::vector<double> tref(reps);
  for (int r = 0; r < reps && ce == cudaSuccess; ++r) {
    float a = 0.f;
    ce = cudaEventElapsedTime(&a, m->events[2 * r * nm], m->events[2 * r * nm + 1]);
    tref[r] = a;
  }
  for (int q = 1; q < nm && ce == cudaSuccess; ++q) {
    const int i = cand_of[q];
    std::vector<double> tc(reps), ratio(reps);
    for (int r = 0; r < reps && ce == cudaSuccess; ++r) {
      float b = 0.f;
      const int e = 2 * (r * nm + q);
      ce = cudaEventElapsedTime(&b, m->events[e], m->events[e + 1]);
      tc[r] = b;
      ratio[r] = b / tref[r];
    }
    ratio_median[i] = median_of(ratio);
    if (ref_median_ms) ref_median_ms[i] = median_of(tref);
    if (cand_median_ms) cand_median_ms[i] = median_of(tc);
    if (raw_ratio) std::copy(ratio.begin(), ratio.end(), raw_ratio + (size_t)i * reps);
  }
  if (exec) cudaGraphExecDestroy(exec);
  cudaGraphDestroy(graph);
  if (ce != cudaSuccess)
    return sip::fail(ctx, SIP_E_MEASURE, std::string("timed launches: ") + cudaGetErrorString(ce));
  return SIP_OK;
}

// The streamed round (the default): the candidates' modules load on worker threads while the
// device already runs the reference's warm-up launches and those of every candidate loaded so
// far, so module loading hides behind warm-up work instead of preceding the whole round; the
// timed launches then go straight onto the stream between event pairs (the host enqueues the
// round's ~100 launches in far less time than the first one runs, so they execute back to
// back as in a captured graph, without the capture and instantiation).  Same launch order,
// input-set rotation and median-of-ratios semantics as measure_round_impl.
static int measure_round_streamed(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                                  const sip_launch* L, int32_t nL, int32_t warmup, int32_t reps,
                                  int32_t flush_l2, double* ratio_median, double* ref_median_ms,
                                  double* cand_median_ms, double* raw_ratio, int32_t* status) {
  sip_ctx* ctx = m->ctx;
  static const bool timing = getenv("SIP_EVAL_TIMING") != nullptr;
  const auto now = [] { return std::chrono::steady_clock::now(); };
  const auto t_begin = now();
  if (m->cache_cap < (size_t)k + 1) m->cache_cap = (size_t)k + 1;
  CachedMod* ref = nullptr;
  int rc = get_module(m, perm_ref, &ref);
  if (rc != SIP_OK) return rc;
  ref->pinned = true;
  std::vector<CachedMod*> mods(k, nullptr);
  std::vector<int> todo;
  for (int i = 0; i < k; ++i) {
    const uint16_t* p = perms + (size_t)i * m->n;
    std::vector<uint16_t> key(p, p + m->n);
    if (CachedMod* hit = find_module(m, key)) {
      hit->pinned = true;
      mods[i] = hit;
    }
    status[i] = SIP_OK;
    if (!mods[i]) todo.push_back(i);
  }
  const size_t nt = todo.size();
  std::vector<std::vector<uint8_t>> imgs(nt);
  std::vector<CUmodule> loaded(nt, nullptr);
  std::vector<CUfunction> fns(nt, nullptr);
  std::unique_ptr<std::atomic<int>[]> ready(new std::atomic<int>[nt > 0 ? nt : 1]);
  // only the check runs here; each worker gathers its candidates' images itself, so the
  // first module reaches the device after one image and one load, not after all k images
  for (size_t t = 0; t < nt; ++t)
    ready[t].store(is_permutation(m, perms + (size_t)todo[t] * m->n) ? 0 : -1);
  CUcontext cur = nullptr;
  if (ctx->cuCtxGetCurrent(&cur) != CUDA_SUCCESS || cur == nullptr) {
    SIP_CUDA(ctx, cudaFree(nullptr));
    ctx->cuCtxGetCurrent(&cur);
  }
  const char* lt = getenv("SIP_LOAD_THREADS");
  const int want = lt ? std::max(1, atoi(lt)) : 8;
  const int nthreads = (int)std::min<size_t>(nt, (size_t)want);
  std::vector<std::thread> pool;
  for (int w = 0; w < nthreads; ++w)
    pool.emplace_back([&, w]() {
      const bool ctx_ok = ctx->cuCtxSetCurrent(cur) == CUDA_SUCCESS;
      for (size_t t = w; t < nt; t += nthreads) {
        if (ready[t].load() != 0) continue;  // not a permutation
        gather_image(m, perms + (size_t)todo[t] * m->n, imgs[t], /*for_load=*/true);
        bool ok = ctx_ok && ctx->cuModuleLoadData(&loaded[t], imgs[t].data()) == CUDA_SUCCESS;
        std::vector<uint8_t>().swap(imgs[t]);  // the driver keeps its own copy
        if (ok && ctx->cuModuleGetFunction(&fns[t], loaded[t], m->func.c_str()) != CUDA_SUCCESS) {
          ctx->cuModuleUnload(loaded[t]);
          loaded[t] = nullptr;
          ok = false;
        }
        ready[t].store(ok ? 1 : -1, std::memory_order_release);
      }
    });
  auto join = [&]() {
    for (auto& th : pool)
      if (th.joinable()) th.join();
  };
  if (flush_l2 && (rc = ensure_flush(ctx)) != SIP_OK) {
    join();
    return rc;
  }
  int slot = 0;
  for (int w = 0; w < warmup && rc == SIP_OK; ++w) rc = launch(m, ref, &L[slot++ % nL]);
  // warm-ups in candidate order, each as soon as its module is there
  size_t t = 0;
  for (int i = 0; i < k && rc == SIP_OK; ++i) {
    if (!mods[i]) {  // the next module being loaded (todo is ascending)
      int st;
      while ((st = ready[t].load(std::memory_order_acquire)) == 0) std::this_thread::yield();
      if (st < 0) {
        status[i] = SIP_E_MEASURE;
        ++t;
        continue;
      }
      CachedMod cm;
      cm.perm.assign(perms + (size_t)i * m->n, perms + (size_t)(i + 1) * m->n);
      cm.mod = loaded[t];
      cm.fn = fns[t];
      cm.stamp = ++m->clock;
      cm.pinned = true;
      // no eviction while the device runs this round's launches: cuModuleUnload waits for
      // the context's pending work, which would stall the pipeline once per candidate; the
      // cache is trimmed after the round (sip_measure_round)
      mods[i] = insert_module(m, std::move(cm));
      ++t;
    }
    for (int w = 0; w < warmup && rc == SIP_OK; ++w) rc = launch(m, mods[i], &L[slot++ % nL]);
  }
  join();
  // modules a failed launch left unclaimed still belong to the cache-less tail: unload them
  for (size_t u = t; u < nt; ++u)
    if (ready[u].load() > 0) ctx->cuModuleUnload(loaded[u]);
  if (rc != SIP_OK) return rc;
  const auto t_warm = now();
  std::vector<CachedMod*> set{ref};
  std::vector<int> cand_of{-1};
  for (int i = 0; i < k; ++i)
    if (status[i] == SIP_OK) {
      set.push_back(mods[i]);
      cand_of.push_back(i);
    }
  const int nm = (int)set.size();
  const int nev = 2 * reps * nm;
  while ((int)m->events.size() < nev) {
    cudaEvent_t e;
    SIP_CUDA(ctx, cudaEventCreate(&e));
    m->events.push_back(e);
  }
  for (int r = 0; r < reps && rc == SIP_OK; ++r)
    for (int q = 0; q < nm && rc == SIP_OK; ++q) {
      const int j = (q + r) % nm;  // rotate the order every rep
      const int e = 2 * (r * nm + j);
      if (flush_l2) cudaMemsetAsync(ctx->flush_buf, (r * nm + q) & 0xff, ctx->flush_bytes, ctx->stream);
      cudaEventRecord(m->events[e], ctx->stream);
      rc = launch(m, set[j], &L[slot++ % nL]);
      cudaEventRecord(m->events[e + 1], ctx->stream);
    }
  if (rc != SIP_OK) return rc;
  const auto t_enq = now();
  cudaError_t ce = cudaStreamSynchronize(ctx->stream);
  if (timing)
    fprintf(stderr, "[sip round streamed] k=%d load+warmup-enqueue %.3f timed-enqueue %.3f execute %.3f ms\n", k,
            std::chrono::duration<double, std::milli>(t_warm - t_begin).count(),
            std::chrono::duration<double, std::milli>(t_enq - t_warm).count(),
            std::chrono::duration<double, std::milli>(now() - t_enq).count());
  std::vector<double> tref(reps);
  for (int r = 0; r < reps && ce == cudaSuccess; ++r) {
    float a = 0.f;
    ce = cudaEventElapsedTime(&a, m->events[2 * r * nm], m->events[2 * r * nm + 1]);
    tref[r] = a;
  }
  for (int q = 1; q < nm && ce == cudaSuccess; ++q) {
    const int i = cand_of[q];
    std::vector<double> tc(reps), ratio(reps);
    for (int r = 0; r < reps && ce == cudaSuccess; ++r) {
      float b = 0.f;
      const int e = 2 * (r * nm + q);
      ce = cudaEventElapsedTime(&b, m->events[e], m->events[e + 1]);
      tc[r] = b;
      ratio[r] = b / tref[r];
    }
    ratio_median[i] = median_of(ratio);
    if (ref_median_ms) ref_median_ms[i] = median_of(tref);
    if (cand_median_ms) cand_median_ms[i] = median_of(tc);
    if (raw_ratio) std::copy(ratio.begin(), ratio.end(), raw_ratio + (size_t)i * reps);
  }
  if (ce != cudaSuccess)
    return sip::fail(ctx, SIP_E_MEASURE, std::string("timed launches: ") + cudaGetErrorString(ce));
  return SIP_OK;
}
