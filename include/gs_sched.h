/*
 * gs_sched.h — C ABI of the B200 candidate-scoring path.
 *
 * The reference (`gpusched`, pure Python + NumPy) has no FFI; its drop-in
 * boundary is the Python seam around `CostEvaluator` and `_cut`
 * (reference pkg/src/gpusched/search.py:90-124, 168-201).  Each entry point
 * below replaces one reference interface on that seam; the Python mirror in
 * paper_2012_07145_b200/ binds them with ctypes.
 *
 * Conventions: all array arguments are DEVICE pointers owned by the caller
 * unless named `host_*`; every call is stream-ordered on `stream`
 * (cudaStream_t passed as void*) and never synchronizes unless stated; the
 * return value is 0 on success or a negative GS_ERR_* code with a message
 * retrievable by gs_last_error().  Handles are immutable after creation
 * except gs_set_weights, and distinct handles are thread-safe.
 */
#ifndef GS_SCHED_H
#define GS_SCHED_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_MAX_NDIM 4
#define GS_NUM_FEATURES 56
#define GS_ALGO_DIM 10
#define GS_NUM_COEFFS 30

enum {
  GS_OK = 0,
  GS_ERR_ARG = -1,        /* bad argument / unsupported configuration     */
  GS_ERR_CUDA = -2,       /* CUDA runtime error                            */
  GS_ERR_CAPACITY = -3,   /* a candidate exceeded a workspace capacity     */
  GS_ERR_SCHEDULE = -4    /* a decision log is structurally illegal        */
};

/* Placement kinds (reference loopnest.py:23, PLACEMENT_KINDS order). */
enum { GS_ROOT = 0, GS_FUSE_BLOCK = 1, GS_FUSE_THREAD = 2, GS_INLINE = 3 };

/* Prune verdicts (reference options.py:48-50 PruneReport.REASONS order + 1). */
enum {
  GS_VALID = 0, GS_PRUNE_RECOMPUTE = 1, GS_PRUNE_IDLE_SMS = 2, GS_PRUNE_WARP_UTIL = 3,
  GS_PRUNE_SERIAL = 4, GS_PRUNE_THREAD_ALLOC = 5, GS_PRUNE_HW_LIMIT = 6
};

/* ---- candidate-independent pipeline descriptor (reference pipeline.py:25-173) */
typedef struct {
  int32_t ndim;
  int32_t extent[GS_MAX_NDIM];
  int32_t elem_bytes;
  int32_t is_external;
  int32_t is_output;
  int32_t n_stages;
  int32_t stage_begin;   /* first global stage index */
  int32_t name_rank;     /* rank in Python str order (hash canonical order) */
  int32_t pad;
} GsFunc;                /* 48 bytes */

typedef struct {
  int32_t func;
  int32_t n_access;
  int32_t access_begin;
  int32_t branching;     /* Strahler number (featurize.py:306-309) */
} GsStage;               /* 16 bytes */

typedef struct {
  int32_t producer;
  int32_t consumer;
  int32_t stage;         /* global stage index of the reading stage */
  int32_t window;        /* window volume (product of hi-lo+1) */
  int32_t s[GS_MAX_NDIM], lo[GS_MAX_NDIM], hi[GS_MAX_NDIM];
} GsAccess;              /* 64 bytes */

typedef struct {         /* reference machine.py:14-33 */
  int32_t warp_size, num_sms, max_threads_per_block, max_active_warps_per_sm,
          max_active_blocks_per_sm, shared_mem_per_block_limit, shared_mem_per_sm,
          global_transaction_bytes, shared_banks, bank_width_bytes;
} GsMachine;

typedef struct {         /* reference options.py:60-68 */
  double recompute_factor, min_blocks_per_sm_factor, warp_utilization_floor;
  int64_t unroll_budget, thread_alloc_bytes;
} GsThresholds;

typedef struct {
  int32_t n_funcs, n_stages, n_access;
  const GsFunc* funcs;           /* host pointers; copied at creation */
  const GsStage* stages;
  const GsAccess* access;
  const double* algo;            /* [n_stages][10] algorithm features */
  const uint8_t* name_repr;      /* concatenated Python repr() bytes of names */
  const int32_t* name_off;       /* [n_funcs + 1] offsets into name_repr */
  GsMachine machine;
  GsThresholds thresholds;
} GsPipelineDesc;

/* ---- one decision record, 16 bytes (reference loopnest.py:34-48) ------- */
typedef struct {
  uint16_t func;                 /* 0xFFFF = padding (end of log) */
  uint16_t consumer;             /* 0xFFFF = None */
  uint8_t kind;                  /* GS_ROOT .. GS_INLINE */
  uint8_t flags;                 /* bit0: serial present, bit1: thread present */
  uint8_t serial[GS_MAX_NDIM];
  uint8_t thread[GS_MAX_NDIM];
  uint16_t pad;
} GsDecision;

typedef struct GsPipeline* gs_pipeline_t;

const char* gs_last_error(void);
int gs_version(void);
/* Number of this library's own kernel launches so far (process-wide). */
int64_t gs_launch_count(void);

/* Pack + upload a pipeline; replaces the per-call `PipelineGraph` walk of
 * featurize.py:275-303 / resolve.py:207-226. */
int gs_pipeline_create(const GsPipelineDesc* desc, gs_pipeline_t* out);
int gs_pipeline_destroy(gs_pipeline_t p);
int gs_pipeline_max_rows(gs_pipeline_t p);

/* Upload coefficient-network weights (fp64 host arrays, reference tensor
 * names/shapes costmodel.py:183-220); call again whenever the Python-side
 * `evaluator.weights` object changes (driver.py:110, 219). Synchronous. */
int gs_set_weights(gs_pipeline_t p, int embed_dim, int hidden_dim,
                   const double* algo_w, const double* algo_b,
                   const double* sched_w, const double* sched_b,
                   const double* head_w, const double* head_b,
                   const double* out_w, const double* out_b);

/* K1: resolve + featurize + prune for N candidates (decision logs of
 * stride S).  Replaces featurize() (featurize.py:275-303) and prune()
 * (options.py:200-255).  Outputs, per candidate c and row r < n_rows[c]:
 * feats[(c*R + r)*56 + k] (fp64, FEATURE_ORDER), row_key[c*R + r] =
 * func << 8 | stage, verdict[c].  R = gs_pipeline_max_rows().  With
 * feats == NULL only the resolve + prune verdict (and n_rows) are produced. */
/* Exact sibling reuse in K1 (default on): each CTA walks a contiguous range
 * of candidates; when a candidate's decision structure (func, kind,
 * consumer per record) equals its predecessor's, the structural resolve is
 * reused, every func's geometry record is compared bit for bit with the
 * predecessor's, and a row is recomputed only if its own / host / kernel /
 * read-producer / thread-child records changed — otherwise its features are
 * copied, which is bit-identical by construction.  0 disables (every row of
 * every candidate is computed).  `row_src` (nullable, [N][R] int32) then
 * names, per row, the candidate whose row was actually computed and whose
 * features this row repeats bit for bit (itself when computed); gs_cost
 * uses it to evaluate the network once per distinct row.  2 = reuse, and
 * feats holds only the computed rows (row_src[c*R + r] == c): repeated rows
 * are left unwritten, for callers that consume features only through
 * gs_cost with row_src (the beam step) — gs_featurize then requires
 * row_src. */
int gs_set_reuse(gs_pipeline_t p, int enable);
/* The current reuse mode (-1 for a null handle). */
int gs_get_reuse(gs_pipeline_t p);

int gs_featurize(gs_pipeline_t p, const GsDecision* dec, int64_t n, int s,
                 double* feats, int32_t* row_key, int32_t* n_rows,
                 uint8_t* verdict, int32_t* row_src, void* stream);

/* gs_featurize with a caller-provided workspace: never allocates and never
 * synchronizes (CUDA-graph capturable).  Batches of >= 8192 candidates with
 * features use the two-phase sibling schedule, which saves one warp state
 * per decision-structure run; `max_runs` (<= 0: min(n/8, 1 GiB of states))
 * bounds how many runs get a state slot — a batch with more runs, or runs
 * shorter than 8 on average, takes the one-phase schedule on the device
 * (same results).  Size the workspace with
 * gs_featurize_workspace_bytes(p, n, s, max_runs). */
int64_t gs_featurize_workspace_bytes(gs_pipeline_t p, int64_t n, int s, int64_t max_runs);
int gs_featurize_ws(gs_pipeline_t p, const GsDecision* dec, int64_t n, int s,
                    double* feats, int32_t* row_key, int32_t* n_rows,
                    uint8_t* verdict, int32_t* row_src, int64_t max_runs,
                    void* workspace, int64_t ws_bytes, void* stream);

/* K2: basis + two-tower network + g.c + h + in-order stage sum.  Replaces
 * CostEvaluator.cost (search.py:115-124).  row_cost/basis_gh optional
 * (NULL = not written; basis_gh is [c*R + r][31] = g[30], h).  With
 * row_src (from gs_featurize, same batch) the network runs once per
 * distinct row and every other row takes its source row's cost (exact:
 * identical features give identical costs); row_cost is then required as
 * [N][R] scratch and ends up holding every row's cost.  basis_gh != NULL
 * disables the reuse. */
int gs_cost(gs_pipeline_t p, const double* feats, const int32_t* row_key,
            const int32_t* n_rows, const int32_t* row_src, int64_t n,
            double* total, double* row_cost, double* basis_gh, void* stream);

/* K2 totals only, with row reuse (the beam step's cut needs no per-row
 * costs): as gs_cost with row_src, but row_scratch ([N][R]) ends up
 * holding only the computed rows' costs — the other rows' costs are not
 * written back (770 MB per 1M-candidate C5 step).  Same totals, bit for
 * bit.  Replaces CostEvaluator.cost (search.py:115-124) for a batch. */
int gs_cost_totals(gs_pipeline_t p, const double* feats, const int32_t* row_key,
                   const int32_t* n_rows, const int32_t* row_src, int64_t n,
                   double* total, double* row_scratch, void* stream);

/* K3: blake2b-64 structural hash at `depth` (loopnest.py:131-165).  A
 * candidate whose (func, kind, consumer, serial/thread presence) fields
 * equal its predecessor's takes the predecessor's hash (equal canonical
 * bytes); only run heads are hashed.  Grows an internal n-byte scratch on
 * first use with a larger n (synchronizes `stream` then). */
int gs_struct_hash(gs_pipeline_t p, const GsDecision* dec, int64_t n, int s,
                   int depth, uint64_t* out, void* stream);
/* gs_struct_hash with a caller-provided workspace of
 * gs_struct_hash_workspace_bytes(n) bytes (never allocates or synchronizes). */
int64_t gs_struct_hash_workspace_bytes(int64_t n);
int gs_struct_hash_ws(gs_pipeline_t p, const GsDecision* dec, int64_t n, int s,
                      int depth, uint64_t* out, void* workspace, int64_t ws_bytes,
                      void* stream);
/* gs_struct_hash_ws at up to four depths in one pass over the records:
 * depths[0..ndepths) (host array), out = [ndepths][n] (depth-major).  The
 * beam step's pass-depth buckets and the bad-hash memo depths
 * (search.py:196-200: the bottom half's hashes at 1..num_passes) come from
 * one launch; the memo then gathers instead of re-hashing. */
int gs_struct_hash_depths_ws(gs_pipeline_t p, const GsDecision* dec, int64_t n, int s,
                             int ndepths, const int* depths, uint64_t* out,
                             void* workspace, int64_t ws_bytes, void* stream);

/* K4: bucket by hash + hierarchical-sampling representatives
 * (sampling.py:45-59, search.py:127-165).  `valid[i]` = verdict==0.
 * Writes rep candidate indices in (hash asc, permutation position) order to
 * rep_idx and their count to *n_reps (device int64), and the drawn
 * rejects (in draw order, for PruneReports) to rej_idx (nullable) and
 * their count to *n_rejects (device int64).  Needs a workspace of
 * gs_select_workspace_bytes(n) bytes. */
int64_t gs_select_workspace_bytes(int64_t n);
int gs_select_reps(const uint64_t* hashes, const uint8_t* verdict, int64_t n,
                   uint64_t phase_seed, void* workspace, int64_t ws_bytes,
                   int64_t* rep_idx, int64_t* n_reps, int64_t* rej_idx,
                   int64_t* n_rejects, void* stream);

/* K5: beam cut (search.py:76-87, 168-201): penalty for flagged hashes,
 * optional Gumbel(T) on log-cost, stable radix top-k.  keys: unpenalized
 * totals of the reps (rep order); pass_hash: hash at pass depth per rep;
 * flagged: sorted array of flagged hashes at that depth.  Writes the first
 * k rep positions (ascending key, ties by rep order) to out_pos and the
 * count to *n_out.  tie_band > 0: keys within that relative distance
 * are ordered by rep position (the reference's stable order of exact
 * ties, which its BLAS-order fp64 sums hit by rounding).  bottom (nullable) gets 1 for reps in the
 * bottom half by unpenalized cost (stable), the memo-flag set of
 * search.py:196-200.  Workspace: gs_topk_workspace_bytes(n). */
int64_t gs_topk_workspace_bytes(int64_t n);
int gs_beam_topk(const double* costs, const uint64_t* pass_hash, int64_t n,
                 const uint64_t* flagged, int64_t n_flagged, double penalty,
                 double temperature, uint64_t phase_seed, int64_t k, double tie_band,
                 void* workspace, int64_t ws_bytes, int64_t* out_pos,
                 int64_t* n_out, uint8_t* bottom, void* stream);
/* gs_beam_topk over the representatives as K4 left them: costs and
 * pass_hash are per CANDIDATE, rep_idx[i] (i < *n_reps, a device count,
 * at most n_max) the candidate of rep i.  Positions, the count and the
 * bottom flags refer to rep order, as in gs_beam_topk.  No host-side count:
 * a whole phase cut (K3 -> K1 -> K2 -> K4 -> K5) is CUDA-graph capturable.
 * Workspace: gs_topk_workspace_bytes(n_max). */
int gs_beam_topk_reps(const double* costs, const uint64_t* pass_hash, const int64_t* rep_idx,
                      int64_t n_max, const int64_t* n_reps, const uint64_t* flagged,
                      int64_t n_flagged, double penalty, double temperature, uint64_t phase_seed,
                      int64_t k, double tie_band, void* workspace, int64_t ws_bytes,
                      int64_t* out_pos, int64_t* n_out, uint8_t* bottom, void* stream);

/* K1 work counters accumulated since the last call (then reset);
 * synchronizes `stream`.  out[0] candidates, [1] candidates resolved
 * incrementally (sibling of the previous one), [2] feature rows computed,
 * [3] feature rows emitted, [4] func geometries (re)resolved, [5] shape of
 * the last K1 launch: scorer warps per CTA << 32 | shared bytes per warp. */
int gs_stats(gs_pipeline_t p, int64_t* out, void* stream);

/* Diagnostics: K1 per-phase warp cycles summed over scorer warps since the
 * last call (16 slots; all zero unless the library was built with
 * -DGS_PHASES): [0..6] record diff, resolve, prune, row flags, sibling
 * copy, row features, key/source writes; [8..13] inside a row: setup,
 * unions, load transactions, working set + store transactions, assembly,
 * (13 = loads end).  Synchronizes the device. */
int gs_debug_phases(int64_t* out);

/* ---- beam-step expansion --------------------------
 * Menus of reference options.py:25-37 (TilingConfig). */
typedef struct {
  int32_t serial_powers[8], n_serial_powers;
  int32_t odd_serial[8], n_odd_serial;
  int32_t innermost_thread[8], n_innermost;
  int32_t outer_thread[8], n_outer;
  int32_t unroll_budget, warp_size;
} GsTilingMenus;

/* Every phase-2 tiling of each parent's step-root decision, parents in
 * order, tilings in the reference order (search.py:223-235
 * `_phase2_candidates`, options.py:144-183).  parents: [n][S] records;
 * step[p]: index of the step root's (compute_root) record in parent p.
 * Writes offsets[0..n] (device int64: candidate range of each parent; the
 * total is offsets[n]) and, when out != NULL, the expanded records
 * out[offsets[n]][S] and (nullable) owner[] = parent index; out/owner hold
 * out_cap candidates and nothing is written past them.  Call once with
 * out == NULL to size `out`.  Workspace: gs_expand_workspace_bytes(n);
 * at most 2^20 parents per call.  More than 4096 tilings for one parent, a
 * step larger than out_cap (those parents are skipped), or a step record
 * that is not a compute_root decision raise GS_ERR_CAPACITY /
 * GS_ERR_SCHEDULE at gs_check. */
int64_t gs_expand_workspace_bytes(int64_t n_parents);
int gs_expand_step(gs_pipeline_t p, const GsDecision* parents, int64_t n_parents, int s,
                   const int32_t* step, const GsTilingMenus* menus, int64_t* offsets,
                   void* workspace, int64_t ws_bytes, GsDecision* out, int64_t out_cap,
                   int32_t* owner, void* stream);

/* Phase-1 placement menus.  Static per-func facts
 * the menus need, as the reference defines them (options.py:74-141,
 * loopnest.py:178-241; pipeline.py:127-134 consumers_of): flags[f] bits
 * 1 output, 2 single stage, 4 pointwise-called (every consumer reads f
 * through identity accesses, options.py:74-86), 8 inlinable (not an output,
 * one stage, no self-read), 16 cheap (ops <= CHEAP_INLINE_OPS); consumers
 * of f = cons[cons_off[f] .. cons_off[f+1]).  Host pointers; synchronous. */
int gs_set_placement_info(gs_pipeline_t p, const uint8_t* flags, const int32_t* cons_off,
                          const int32_t* cons, const int32_t* sched_order, int n_sched);

/* n complete random schedules, candidate i drawn by
 * default_rng((seed, first + i)) exactly as the reference test suite's
 * `_random_schedule` (tests/test_acceptance.py:136-160) draws: one menu
 * entry per func in scheduling order (sched_order of gs_set_placement_info),
 * a serial tiling for fuse_at_block, then a serial and a thread tiling per
 * compute_root func.  out: [n][s] records (s >= the schedulable funcs).
 * This is the §8(d) stress workload generator: independent candidates with
 * no shared decision structure, generated on the device. */
int gs_random_schedules(gs_pipeline_t p, uint64_t seed, int64_t first, int64_t n, int s,
                        const GsTilingMenus* menus, GsDecision* out, void* stream);

/* Every phase-1 candidate of each parent for `func` (search.py:204-220
 * `_phase1_candidates`): enumerate_compute_locations' menu (compute_root;
 * fuse_at_block / fuse_at_thread into each scheduled effective consumer in
 * name order when apply_decision would accept it; inline when cheap, or
 * alone when single-stage and pointwise-called; compute_root alone for
 * outputs), restricted to the kinds in restrict_mask (bit per GS_* kind;
 * 0xF = all; search.py:208-210), fuse_at_block entries crossed with every
 * serial tiling (options.py:144-162).  The new record is appended after the
 * parent's last one.  Outputs as gs_expand_step (offsets, out[out_cap][s],
 * owner).  A parent that already schedules `func` or has no free record
 * slot raises GS_ERR_SCHEDULE at gs_check.  Workspace:
 * gs_phase1_workspace_bytes(n). */
int64_t gs_phase1_workspace_bytes(int64_t n_parents);
int gs_expand_phase1(gs_pipeline_t p, const GsDecision* parents, int64_t n_parents, int s, int func,
                     int restrict_mask, const GsTilingMenus* menus, int64_t* offsets, void* workspace,
                     int64_t ws_bytes, GsDecision* out, int64_t out_cap, int32_t* owner, void* stream);

/* ---- machine oracle ------------------------------
 * The throughput knobs of reference machine.py:26-31 (not hardware limits). */
typedef struct {
  int32_t registers_per_thread_budget;   /* register_bytes_per_thread = 4 x this */
  int32_t pad;
  double compute_throughput;             /* scalar ops / s at full occupancy */
  double global_bandwidth, shared_bandwidth;   /* bytes / s */
  double kernel_launch_overhead;         /* s */
} GsOracleParams;

/* K1 (every row materialised, plus each row's kernel) then K6: the
 * reference's simulate_runtime (machine.py:108-167) for N candidates.
 * Device outputs per candidate: runtime[c] (s; NaN unless status 0),
 * spill_bytes[c] (> 0 iff registers spilled), status[c]: 0 ok, 1 a kernel
 * breaks a hardware limit, 2 not fully scheduled (the reference raises
 * ValueError for both).  Uses a grow-only internal feature workspace. */
int gs_simulate(gs_pipeline_t p, const GsDecision* dec, int64_t n, int s, const GsOracleParams* op,
                double* runtime, int64_t* spill_bytes, uint8_t* status, void* stream);

/* ---- the cost model off the beam step ------
 * Weights are ONE packed fp64 device array in the reference tensor order
 * (costmodel.py:183-193): algo_w[10][E] algo_b[E] sched_w[56][E] sched_b[E]
 * head_w[2E][H] head_b[H] out_w[H][30] out_b[30]; gs_model_params(E, H)
 * doubles. */
int gs_model_params(int embed_dim, int hidden_dim);

/* predict_coefficients (costmodel.py:316-324) and stage_cost /
 * CostBreakdown (costmodel.py:34-115) for n rows: algo [n][10], sched
 * [n][56] (raw schedule features).  coeffs_in (nullable) [n][30]: use these
 * coefficients instead of the network (stage_cost with given c; the caller
 * validates c > 0).  Outputs (nullable): coeffs_out [n][30]; breakdown
 * [n][7] = compute, load, store, malloc, parallelism, working_set, total —
 * the reference's term order and rounding (bit-exact for given c). */
int gs_predict(const double* weights, int embed_dim, int hidden_dim, const double* algo,
               const double* sched, const double* coeffs_in, int64_t n, double* coeffs_out,
               double* breakdown, void* stream);

/* train (costmodel.py:391-432): SGD with momentum on (log predicted total -
 * log runtime)^2, gradients through the network only (basis g, h fixed),
 * one persistent CTA running every epoch.  Samples: rows row_off[s] ..
 * row_off[s+1]-1 of algo [rows][10], sched [rows][56], g [rows][30], h
 * [rows]; runtime[s] > 0; order [epochs][n_samples] = each epoch's sample
 * permutation (the reference's default_rng(seed).permutation stream).
 * `weights` (device, packed) is updated in place; loss_hist[epoch] = mean
 * squared error of the epoch; *status (device int) = 0, or s + 1 when
 * sample s predicted a non-finite or non-positive total (training stops
 * there; the reference raises ValueError).  At most 1024 rows per sample.
 * Workspace: gs_train_workspace_bytes(E, H, max_rows). */
int64_t gs_train_workspace_bytes(int embed_dim, int hidden_dim, int max_rows);
int gs_train(double* weights, int embed_dim, int hidden_dim, const double* algo, const double* sched,
             const double* g, const double* h, const int64_t* row_off, const double* runtime,
             const int32_t* order, int n_samples, int epochs, double learning_rate, double momentum,
             int max_rows, void* workspace, int64_t ws_bytes, double* loss_hist, int* status,
             void* stream);

/* Device-side error word of the last K1 launch (capacity overflow etc.);
 * synchronizes `stream`. */
int gs_check(gs_pipeline_t p, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* GS_SCHED_H */
