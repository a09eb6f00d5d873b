/*
 * sip.h -- C ABI of the B200-native SIP search-and-evaluate layer (libsip.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in any signature.
 * Every function returns SIP_OK (0) or an SIP_E_* code; sip_last_error()
 * gives the message of the most recent failure on that context.
 *
 * Each entry point replaces one piece of the reference package
 * (/root/reference/pkg/src/sasstune, pure Python).  The citations name the
 * reference interface the entry point stands in for; INTEGRATION.md shows the
 * ctypes binding (paper_2403_16863_b200/engine.py) a maintainer would add.
 */
#ifndef SIP_H
#define SIP_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SIP_OK 0
#define SIP_E_ARG 1         /* bad argument (ValueError in the reference)            */
#define SIP_E_CUDA 2        /* CUDA runtime / driver failure                         */
#define SIP_E_MEASURE 3     /* -> backends.MeasurementFailed (backends.py:28)        */
#define SIP_E_NOCAND 4      /* -> perturb.NoCandidatesError (perturb.py:35)          */
#define SIP_E_ELF 5         /* cubin could not be parsed / patched                   */
#define SIP_E_STATE 6       /* call out of sequence                                  */

#define SIP_MAX_REFS 4
#define SIP_NO_BARRIER 7

/* history status codes (reference anneal.HistoryRecord.rejected, anneal.py:84) */
#define SIP_ST_ACCEPTED 0
#define SIP_ST_PRICED 1       /* measured, Metropolis said no                    */
#define SIP_ST_BOUNDARY 2     /* rejected="boundary"                             */
#define SIP_ST_DEPENDENCY 3   /* rejected="dependency"                           */
#define SIP_ST_TEST 4         /* rejected="test-failure"                         */
#define SIP_ST_MEASURE 5      /* rejected="measurement"                          */
#define SIP_ST_HWSAFE 6       /* extension: rejected="hw-safety" (hw_safe mode)  */

typedef struct sip_ctx sip_ctx;
typedef struct sip_kernel sip_kernel;
typedef struct sip_chains sip_chains;
typedef struct sip_module sip_module;
typedef struct sip_results sip_results;

/* one memory reference (reference deps.MemRef, deps.py:203-209) */
typedef struct {
  int64_t offset;
  int32_t base;   /* interned register id, -1 = none */
  uint8_t size;   /* bytes */
  uint8_t space;  /* 0 global 1 shared 2 local 3 unknown */
  uint8_t write;
  uint8_t pad;
} sip_memref;

/* Per-instruction tables of one listing (host arrays; see tables.py). */
typedef struct {
  int32_t n;              /* instructions                                   */
  int32_t words;          /* u64 words per register bitset                  */
  const uint32_t* ctrl;   /* [n] packed control (tables.py docstring)       */
  const uint32_t* lat;    /* [n] MachineConfig.latency_of                   */
  const uint8_t* klass;   /* [n] InstrClass code                            */
  const uint64_t* reads;  /* [n*words] deps.reads_writes()[0]               */
  const uint64_t* writes; /* [n*words] deps.reads_writes()[1]               */
  const sip_memref* refs; /* [n*SIP_MAX_REFS] deps.mem_refs                 */
  const uint8_t* nrefs;   /* [n]                                            */
  const uint8_t* cut;     /* [n+1] Kernel.block_boundaries as a bitmap      */
  const uint8_t* pin;     /* [n] hardware mode: never move (may be NULL)    */
  const uint64_t* guard;  /* [(n+1)*words] scoreboard-guard footprints of the */
                          /* sm100 classes (tables.py); NULL = a wait mask    */
                          /* pins its instruction (hw_safe rule 4)            */
} sip_tables;

typedef struct {
  int32_t budget;            /* AnnealConfig.iteration_budget (anneal.py:67)            */
  int32_t unsafe_moves;      /* AnnealConfig.unsafe_moves (anneal.py:54)                */
  int32_t hw_safe;           /* extension; 0 reproduces the reference bit for bit       */
  int32_t min_fixed_distance;/* hw_safe: cycles a fixed-latency RAW pair must keep      */
  const double* temperature; /* [budget] T at each iteration (repeated division)        */
} sip_anneal_cfg;

/* one HistoryRecord (anneal.py:76-99) in compact form */
typedef struct {
  double time;         /* candidate time (status ACCEPTED/PRICED)   */
  int32_t lo;          /* swap slot (lo, lo+1); -1 if none          */
  uint16_t candidate;  /* Action.candidate                          */
  uint8_t direction;   /* 0 up, 1 down                              */
  uint8_t status;      /* SIP_ST_*                                  */
} sip_record;

typedef struct {
  double t0;             /* AnnealState.baseline                      */
  double best_energy;    /* AnnealState.best_energy                   */
  double current_energy; /* AnnealState.current_energy                */
  int32_t best_iter;     /* iteration that produced best (-1 = none)  */
  int32_t ambiguous;     /* Metropolis draws within 4 ulp of exp()    */
  int64_t replayed;      /* scoreboard steps executed (instrumentation) */
  int32_t priced;        /* iterations whose candidate was priced        */
  int32_t pad;
} sip_chain_summary;

/* One epoch of a sharded search, reduced on the device (bench / run_search
 * sharding): the champion chain under driver.py:81-85's ranking and the sums. */
typedef struct {
  int32_t champion_chain;
  int32_t pad;
  double best_energy;
  int64_t best_seed;
  int64_t priced;
  int64_t replayed;
  int64_t ambiguous;
} sip_epoch_result;

/* ---- context -------------------------------------------------------- */
const char* sip_version(void);
int sip_device_count(int* count);
int sip_open(int device, sip_ctx** out);
int sip_close(sip_ctx* ctx);
const char* sip_last_error(sip_ctx* ctx);

/* ---- G1: listing tables + pair-legality matrix ------------------------
 * replaces deps.build_depgraph (deps.py:279-349) as used by
 * perturb.apply_action (perturb.py:86): E(a,b) rows for every
 * global-class instruction, built once per listing on the device.        */
int sip_kernel_create(sip_ctx* ctx, const sip_tables* t, sip_kernel** out);
int sip_kernel_destroy(sip_kernel* k);
int sip_kernel_candidates(sip_kernel* k, int32_t* count);
/* E rows, [k][ceil(n/32)] u32 each: after[g] bit x = E(g,x); before[g] bit x = E(x,g) */
int sip_legality_rows(sip_kernel* k, uint32_t* after, uint32_t* before);
/* deps.swap_legal (deps.py:352-358) for nq (schedule, lo) queries; sched is [nq*n] */
int sip_legality_query(sip_kernel* k, const uint16_t* sched, const int32_t* lo, int32_t nq,
                       int32_t hw_safe, int32_t min_fixed_distance, uint8_t* legal);

/* ---- scoreboard energy: machine.simulate (machine.py:116-161) -------- */
int sip_simulate(sip_kernel* k, const uint16_t* scheds, int32_t count, int64_t* totals,
                 int32_t* waited /* [count*n] or NULL */, int8_t* binding /* [count*n] or NULL */);

/* ---- G2: fused batched annealing, simulator energy --------------------
 * anneal.anneal (anneal.py:123-213) with SimulatorBackend, for `chains`
 * independent seeds at once (driver.run_search, driver.py:73-79).       */
int sip_anneal(sip_kernel* k, const sip_anneal_cfg* cfg, const int64_t* seeds, int32_t chains,
               sip_record* history /* [chains*budget] */, uint16_t* best /* [chains*n] */,
               uint16_t* current /* [chains*n] */, sip_chain_summary* summary /* [chains] */);

/* same, starting every chain from `start` (identity when NULL); `champion`
 * (optional, [n]) receives the best schedule over all chains ranked by
 * (best energy, seed) as driver.run_search ranks them (driver.py:81-85). */
int sip_anneal_ex(sip_kernel* k, const sip_anneal_cfg* cfg, const int64_t* seeds, int32_t chains,
                  const uint16_t* start, sip_record* history, uint16_t* best, uint16_t* current,
                  sip_chain_summary* summary, uint16_t* champion, int32_t* champion_chain);

/* same, but every chain's history and schedules stay on the device; only the
 * summaries come back.  Results are pulled per chain range on demand (the
 * public API's AnnealState materialises lazily).  A result set must be
 * destroyed before its sip_kernel.                                       */
/* fused chains with consecutive seeds seed_base + c (generated on the device),
 * reduced to one sip_epoch_result; `champion` receives that chain's best schedule */
int sip_anneal_epoch(sip_kernel* k, const sip_anneal_cfg* cfg, int64_t seed_base, int32_t chains,
                     const uint16_t* start, sip_epoch_result* result, uint16_t* champion);
int sip_anneal_keep(sip_kernel* k, const sip_anneal_cfg* cfg, const int64_t* seeds, int32_t chains,
                    const uint16_t* start, sip_chain_summary* summary, sip_results** out);
/* sip_anneal_keep without the summaries: seeds given, or seed_base + c generated on the
 * device when `seeds` is NULL (run_search's consecutive seeds, driver.py:73-79); the
 * champion under driver.py:81-85's ranking and the sums come back reduced on the device,
 * per-chain summaries stay in HBM until sip_results_summary reads a range of them. */
int sip_anneal_keep_reduced(sip_kernel* k, const sip_anneal_cfg* cfg, const int64_t* seeds, int64_t seed_base,
                            int32_t chains, const uint16_t* start, sip_epoch_result* result,
                            sip_results** out);
int sip_results_summary(sip_results* r, int32_t first, int32_t count, sip_chain_summary* summary);
int sip_results_fetch(sip_results* r, int32_t first, int32_t count, sip_record* history,
                      uint16_t* best, uint16_t* current);
int sip_results_destroy(sip_results* r);

/* device bytes one fused chain of `budget` iterations works on in HBM during a launch
 * (schedules -- or, for listings with at most 8 candidates, its candidate slots, the rows
 * being built only when read --, MT19937 words, checkpoints, logs, history): the
 * denominator of the engine's DRAM-traffic ratio in bench.py */
int sip_anneal_state_bytes(sip_kernel* k, int32_t budget, int64_t* per_chain);

/* chains that fill every SM once with the fused simulator-energy kernel (one
 * chain per thread at its occupancy on this listing): size `chains` of
 * sip_anneal_epoch / sip_anneal_keep in multiples of it to avoid a partial wave */
int sip_anneal_wave(sip_kernel* k, int32_t* chains);

/* page-locked host memory for result buffers the device writes whole (chain
 * summaries): full-rate DMA, no first-touch page faults.  The Python host
 * recycles these blocks in a pool.                                        */
int sip_host_alloc(size_t bytes, void** out);
int sip_host_free(void* p);

/* ---- G2 step mode: external energy (any backend.measure) ------------- */
int sip_chains_create(sip_kernel* k, const sip_anneal_cfg* cfg, const int64_t* seeds,
                      const double* t0, int32_t chains, sip_chains** out);
/* advance every live chain to its next legal proposal; lo[c] = -1 when the
 * chain has exhausted its budget.  sched (optional) receives [chains*n]
 * candidate schedules (identity order of the listing).                  */
int sip_chains_propose(sip_chains* s, int32_t* lo, uint16_t* sched);
/* feed back the candidate times (status SIP_ST_PRICED, SIP_ST_TEST or
 * SIP_ST_MEASURE per chain; ignored for chains with lo = -1)            */
int sip_chains_resolve(sip_chains* s, const double* t_curr, const uint8_t* status);
/* adopt schedule `src` of chain src_chain in every chain (epoch exchange) */
int sip_chains_adopt(sip_chains* s, const uint16_t* sched, double energy, double time);
int sip_chains_result(sip_chains* s, sip_record* history, uint16_t* best, uint16_t* current,
                      sip_chain_summary* summary);
int sip_chains_destroy(sip_chains* s);

/* ---- G3/G4: cubin frontend + candidate evaluator ----------------------
 * replaces backends.ExternalCommandBackend.measure (backends.py:108-116)
 * and the adapter process behind it (frontend/src/measure.ts:66-85).    */
typedef struct {
  uint32_t grid[3];
  uint32_t block[3];
  uint32_t cluster[3];   /* {0,0,0} or {1,1,1} = no cluster */
  uint32_t smem_bytes;          /* dynamic shared memory                     */
  const void* params;           /* argument payload buffer                   */
  const uint32_t* param_offsets;/* byte offset of argument i inside params   */
  uint32_t nparams;             /* number of kernel arguments                */
  uint32_t params_size;         /* payload bytes                             */
} sip_launch;

int sip_module_open(sip_ctx* ctx, const void* cubin, size_t size, const char* func,
                    sip_module** out);
int sip_module_close(sip_module* m);
/* instruction count, and the byte offset of .text.<func> inside the cubin */
int sip_module_info(sip_module* m, int32_t* n_instr, uint64_t* text_offset);
/* both 64-bit words of every instruction, [2n] */
int sip_module_words(sip_module* m, uint64_t* words);
/* 1 for instructions whose offset is named by EIATTR tables or relocations */
int sip_module_pins(sip_module* m, uint8_t* pin);
/* cubin with .text.<func> permuted: word[i] <- word[perm[i]]; *size in/out */
int sip_module_patch(sip_module* m, const uint16_t* perm, void* out, size_t* size);
/* load the permuted cubin (NULL = as compiled), time warmup+reps launches
 * inside one CUDA graph with per-launch events; median in ms.           */
int sip_measure(sip_module* m, const uint16_t* perm, const sip_launch* launch, int32_t warmup,
                int32_t reps, int32_t flush_l2, double* median_ms, double* raw_ms);
/* paired timing: baseline (perm_ref) and candidate (perm_cand) launches
 * alternate inside one CUDA graph (order rotated every rep, L2 flushed before
 * each launch); the per-pair ratio cand/ref cancels clock and power drift.
 * *ratio_median is the candidate's energy relative to the baseline.       */
int sip_measure_paired(sip_module* m, const uint16_t* perm_ref, const uint16_t* perm_cand,
                       const sip_launch* launch, int32_t warmup, int32_t reps, int32_t flush_l2,
                       double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                       double* raw_ratio);
/* k candidates (perms: [k][n]) each timed against perm_ref like sip_measure_paired,
 * all from one CUDA graph after parallel cubin loads; per-candidate outputs, and
 * status[i] = SIP_E_MEASURE for a candidate whose cubin failed to load (skipped). */
/* One nvcc reference per round (backends.py:108-116 median semantics per candidate): the
 * reference and the k candidates are warmed up once each, then each of `reps` reps launches
 * all k+1 modules once in a rotated order, event-timed; candidate i's ratio is the median
 * over reps of t_i / t_ref of the same rep.  Launch slot q uses parameter set L[q % nL]
 * (nL >= 3 buffer sets larger than L2 in rotation need no flush: flush_l2 = 0).  The
 * candidates' modules load on worker threads while the warm-ups already run, and the
 * launches go straight onto the stream (SIP_ROUND_GRAPH=1: one captured CUDA graph after
 * all loads); afterwards the module cache keeps the 64 most recent (SIP_MODULE_KEEP).
 * Replaces backends.ExternalCommandBackend.measure per candidate (backends.py:66-116). */
int sip_measure_round(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                      const sip_launch* L, int32_t nL, int32_t warmup, int32_t reps, int32_t flush_l2,
                      double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                      double* raw_ratio, int32_t* status);
int sip_measure_paired_batch(sip_module* m, const uint16_t* perm_ref, const uint16_t* perms, int32_t k,
                             const sip_launch* launch, int32_t warmup, int32_t reps, int32_t flush_l2,
                             double* ratio_median, double* ref_median_ms, double* cand_median_ms,
                             double* raw_ratio, int32_t* status);
/* run the permuted module once on the given launch (verification) */
int sip_run(sip_module* m, const uint16_t* perm, const sip_launch* launch);
/* same, enqueued on the context stream without synchronising (errors surface at
 * the next synchronising call, e.g. sip_verify_result)                      */
int sip_run_async(sip_module* m, const uint16_t* perm, const sip_launch* launch);

/* ---- G5/G6: probabilistic verification --------------------------------
 * replaces difftest.sample_inputs / run_tests compare (difftest.py:124-204) */
typedef struct {
  int64_t checked_elems;
  int64_t mismatched_elems;   /* outside |a-b| <= atol + rtol*|a|            */
  int64_t bitdiff_elems;      /* not bit-identical                           */
  int64_t failed_samples;
  int64_t first_fail_sample;  /* -1 if none                                  */
  int64_t first_fail_elem;    /* element index within that sample            */
  double max_abs_err;
} sip_cmp_result;

/* dtype: 0 = fp16, 1 = bf16 */
int sip_fill_normal(sip_ctx* ctx, void* dev, size_t count, int32_t dtype, uint64_t seed,
                    uint64_t stream, float sigma);
int sip_compare(sip_ctx* ctx, const void* ref, const void* cand, size_t count, int32_t dtype,
                double atol, double rtol, int64_t elems_per_sample, int64_t first_sample,
                sip_cmp_result* out);
/* accumulating compare for long verification runs (10M samples):
 * sip_verify_compare enqueues one batch (count elements = count/elems_per_sample
 * samples starting at global sample index first_sample) without synchronising;
 * sip_verify_result synchronises and reports the totals so far (first failure
 * as a global sample index, min over batches).  run_tests' verdict fields,
 * difftest.py:158-204.                                                      */
typedef struct sip_verify_acc sip_verify_acc;
int sip_verify_open(sip_ctx* ctx, int64_t max_samples, int64_t elems_per_sample, sip_verify_acc** out);
int sip_verify_compare(sip_verify_acc* acc, const void* ref, const void* cand, size_t count, int32_t dtype,
                       double atol, double rtol, int64_t first_sample);
int sip_verify_result(sip_verify_acc* acc, sip_cmp_result* out);
int sip_verify_close(sip_verify_acc* acc);
/* difftest.sample_inputs (difftest.py:124-141): CPython Random(f"{seed}:{s}")
 * streams generated on the device.  spec = (nbytes, cell, dist) per buffer
 * (dist 0 uniform, 1 small, 2 zero); out = [count][sum nbytes] host bytes. */
int sip_sample_inputs(sip_ctx* ctx, int64_t seed, int64_t first, int32_t count, int32_t nbuf,
                      const int32_t* nbytes, const int32_t* cell, const int32_t* dist,
                      uint8_t* out);

/* same stream written to a device buffer [count][sum nbytes] */
int sip_sample_inputs_device(sip_ctx* ctx, int64_t seed, int64_t first, int32_t count, int32_t nbuf,
                             const int32_t* nbytes, const int32_t* cell, const int32_t* dist, void* dev_out);

/* ---- GPU interpreter of the reference's integer SASS subset ------------
 * machine.CompiledKernel.run (machine.py:698-711): one device thread per
 * sample executes `prog` (64-byte ops compiled by interp.py) on its slice
 * region + s*stride of the buffers (virtual bases[b], lens[b] bytes at offs[b]).
 * status[s]: 0 ok, 1 global / 2 shared out of bounds, 3 uninitialised read
 * (strict), low byte = code, bits 8.. = access size; fault[s] = address.     */
int sip_vm_exec(sip_ctx* ctx, const void* prog, int32_t nops, int32_t nbuf, const int64_t* bases,
                const int32_t* lens, const int32_t* offs, void* region, int64_t stride, int32_t count,
                int32_t shared_bytes, int32_t strict, int32_t* status, int64_t* fault);
/* first differing cell of bytes [off, off+nbytes) between two regions, per sample (-1 = equal) */
int sip_vm_cell_diff(sip_ctx* ctx, const void* a, const void* b, int64_t stride, int32_t off, int32_t nbytes,
                     int32_t cell, int32_t count, int32_t* first_cell);

/* ---- tuning targets (G7/G8): launch descriptors for the shipped cubins -- */
/* GEMM+LeakyReLU: C[l] = leaky(A[l] (MxK, row-major) * B[l]^T (NxK, row-major)) fp16 */
int sip_target_gemm_launch(sip_ctx* ctx, const void* A, const void* B, void* C, int32_t M,
                           int32_t N, int32_t K, int32_t L, float slope, sip_launch* launch,
                           void* params, uint32_t params_cap);
/* attention fwd: O = softmax(Q K^T * scale) V; [B,H,S,D] fp16, D = 128 */
int sip_target_attn_launch(sip_ctx* ctx, const void* Q, const void* K, const void* V, void* O,
                           int32_t B, int32_t H, int32_t S, int32_t D, float scale,
                           sip_launch* launch, void* params, uint32_t params_cap);

/* ---- multi-GPU epoch exchange (G9) -------------------
 * One communicator per rank (one process per GPU) over NCCL (NVLink/NVSwitch on
 * one box).  libnccl.so.2 is opened at run time (the copy the process already
 * mapped, e.g. torch's, else the system one), so libsip keeps no link-time NCCL
 * dependency.  The reference runs chains sequentially and ranks them by
 * (best_time, seed) (driver.py:73-85); chains shard over ranks and every epoch
 * all ranks adopt the global best under that same key.                       */
typedef struct sip_comm sip_comm;
/* one rank's epoch champion: 24 bytes, all-gathered as raw bytes           */
typedef struct {
  double energy;   /* best energy of the rank's chains (lower is better)      */
  int64_t seed;    /* seed of that chain (the ranking tie-break)             */
  int32_t rank;    /* filled in by sip_nccl_exchange                          */
  int32_t pad;
} sip_best;
#define SIP_RED_SUM 0
#define SIP_RED_MAX 1
#define SIP_RED_MIN 2
/* rank 0 makes the id (ncclGetUniqueId); the caller hands it to the other ranks
 * (any rendezvous: a TCP store, a file) -- 128 bytes                         */
int sip_comm_unique_id(uint8_t id[128]);
int sip_comm_create(sip_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank, sip_comm** out);
int sip_comm_destroy(sip_comm* comm);
/* ncclAllGather of every rank's sip_best (24 B each), the winner = min (energy,
 * seed, rank); then ncclBroadcast of the winner's schedule (n u16) from its owner.
 * Host buffers: mine/sched_mine in; all (nranks entries, may be NULL), winner and
 * sched_out (n entries) out.  Collective: every rank calls it each epoch.     */
int sip_nccl_exchange(sip_comm* comm, const sip_best* mine, const uint16_t* sched_mine, int32_t n,
                      sip_best* all, sip_best* winner, uint16_t* sched_out);
/* in-place allreduce of `count` doubles (host buffer), op = SIP_RED_*: the
 * bench's max-over-ranks device times and summed counters                  */
int sip_comm_allreduce(sip_comm* comm, double* vals, int32_t count, int32_t op);
int sip_comm_barrier(sip_comm* comm);

#ifdef __cplusplus
}
#endif
#endif /* SIP_H */
