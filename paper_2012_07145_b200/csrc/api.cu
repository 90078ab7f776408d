// extern "C" entry points of libgs_sched.so (declared in include/gs_sched.h).
#include "gs_internal.cuh"
#include <nvtx3/nvToolsExt.h>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>
#include <algorithm>

namespace gs {
Layout make_layout(int nd, int nf, int ns, int blob_bytes, int S, int R, int rcap, int pcap, int nwarps,
                   int spill, bool generic);
int launch_featurize(int nd, const PipeDev* P, const uint8_t* blob, const GsDecision* dec, int64_t n, int S,
                     double* feats, int32_t* row_key, int32_t* n_rows, uint8_t* verdict, int32_t* row_src,
                     const Layout& L, int nwarps, int grid, int* gerr, int reuse, uint8_t* gscratch,
                     uint8_t* heads, int mode, const int32_t* run_id, const int32_t* run_head,
                     const uint32_t* nruns, int64_t max_runs, uint8_t* slots, int64_t slot_bytes,
                     int32_t* row_kernel, cudaStream_t st);
int launch_simulate(const GsFunc* funcs, int nf, const GsDecision* dec, int64_t n, int S, const double* feats,
                    const int32_t* row_key, const int32_t* n_rows, const int32_t* row_kernel, int R,
                    const int32_t* stage_of_func, const double* algo, const GsMachine& m, const GsOracleParams& op,
                    double* runtime, int64_t* spill_bytes, uint8_t* status, cudaStream_t st);
void k1_prepare_runs(const GsDecision* dec, int64_t n, int S, uint8_t* heads, int32_t* run_id, int32_t* run_head,
                     uint32_t* sums, uint32_t* nruns, cudaStream_t st);
size_t k1_runs_sums_bytes(int64_t n);
int featurize_warps(const Layout& L1, int max_smem);
int read_phases(long long* out);
int launch_hoist(const NetDev& net, const double* algo, int n_stages, cudaStream_t st);
int launch_cost(const NetDev& net, const int32_t* stage_of_func, const double* feats, const int32_t* row_key,
                const int32_t* n_rows, const int32_t* row_src, int64_t n, int R, double* total, double* row_cost,
                double* basis_gh, unsigned* work, int num_sms, cudaStream_t st, bool rows_out = true);
int launch_hash(const GsDecision* dec, int64_t n, int S, int nf, HashDepths D, const int32_t* sorted_funcs,
                const uint8_t* names, const int32_t* name_off, uint64_t* out, uint8_t* head, int repr_bound,
                int num_sms, cudaStream_t st);
int64_t select_workspace_bytes(int64_t n);
int select_reps(const uint64_t* hashes, const uint8_t* verdict, int64_t n, uint64_t phase_seed, void* ws,
                int64_t ws_bytes, int64_t* rep_idx, int64_t* n_reps, int64_t* n_rejects, int64_t* rej_idx,
                cudaStream_t st);
int64_t topk_workspace_bytes(int64_t n);
int64_t expand_workspace_bytes(int64_t n);
int launch_expand(const GsFunc* funcs, const GsDecision* parents, int64_t n, int S, const int32_t* step,
                  const GsTilingMenus& m, int64_t* offsets, void* ws, int64_t ws_bytes, GsDecision* out,
                  int64_t out_cap, int32_t* owner, int* gerr, int num_sms, cudaStream_t st);
int serial_count(const GsTilingMenus& m, const GsFunc& fn);
int64_t phase1_workspace_bytes(int64_t n);
int launch_random_schedules(const GsFunc* funcs, int nf, const P1Static& st, const int32_t* order, int n_order,
                            const GsTilingMenus& m, uint64_t seed, int64_t first, int64_t n, int S, GsDecision* out,
                            int* gerr, cudaStream_t st_);
int launch_phase1(const GsFunc* funcs, int nf, const P1Static& st, const GsDecision* parents, int64_t n, int S,
                  int func, int restrict_mask, const GsTilingMenus& m, int n_serial, int64_t* offsets, void* ws,
                  int64_t ws_bytes, GsDecision* out, int64_t out_cap, int32_t* owner, int* gerr, int num_sms,
                  cudaStream_t st_);
int64_t train_cache_bytes(int E, int H, int max_rows);
int model_params(int E, int H);
int launch_predict(const double* w, int E, int H, const double* algo, const double* sched, const double* cin,
                   int64_t n, double* cout, double* breakdown, cudaStream_t st);
int launch_train(double* w, int E, int H, const double* algo, const double* sched, const double* g, const double* h,
                 const int64_t* row_off, const double* runtime, const int32_t* order, int n_samples, int epochs,
                 double lr, double momentum, double* cache, double* loss_hist, int* status, cudaStream_t st);
int beam_topk(const double* costs, const uint64_t* ph, const int64_t* rep, int64_t n, const int64_t* ndev,
              const uint64_t* flagged, int64_t nflag, double penalty, double temperature, uint64_t phase_seed,
              int64_t k, double band, void* ws, int64_t ws_bytes, int64_t* out_pos, int64_t* n_out, uint8_t* bottom,
              cudaStream_t st);
}  // namespace gs

using namespace gs;

static thread_local std::string g_err;

static int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) return fail(GS_ERR_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct GsPipeline {
  PipeDev host{};
  PipeDev* dev = nullptr;
  uint8_t* blob = nullptr;
  int32_t* stage_of_func = nullptr;
  double* algo = nullptr;
  int32_t* sorted = nullptr;
  uint8_t* names = nullptr;
  int32_t* name_off = nullptr;
  int* err = nullptr;
  NetDev net{};
  std::vector<double*> wbufs;
  int num_sms = 0;
  int max_smem = 0;
  int sm_smem = 0;       // shared memory per SM
  int cta_reserved = 0;  // shared memory the runtime reserves per CTA
  int rcap = 0, pcap = 0;
  int reuse = 1;
  int nwarps = getenv("GS_K1_WARPS") ? atoi(getenv("GS_K1_WARPS")) : kK1MaxWarps;   // diagnostics override
  int last_warps = 0, last_slice = 0;   // K1 launch shape (diagnostics)
  int repr_bound = 1 << 30;             // longest possible canonical repr (K3)
  // Library-owned workspaces of the convenience entry points (gs_featurize,
  // gs_struct_hash, gs_simulate), grown once per size class; the *_ws entry
  // points take the caller's workspace instead and never allocate.
  uint8_t* hscratch = nullptr;   // K3 run-head flags
  int64_t hcap = 0;
  uint8_t* k1ws = nullptr;       // K1 workspace (see K1Ws)
  int64_t k1cap = 0;
  uint8_t* p1flags = nullptr;    // phase-1 menus (gs_set_placement_info)
  int32_t* p1cons_off = nullptr;
  int16_t* p1cons = nullptr;
  int32_t* p1order = nullptr;    // schedulable funcs, scheduling order
  int p1norder = 0;
  std::vector<GsFunc> hfuncs;    // host copy of the funcs (menu sizes)
  uint8_t* simbuf = nullptr;     // K6: features, row keys / kernels, n_rows, verdicts (grow-only)
  int64_t simcap = 0;
};

// NVTX range per C-ABI entry point (header-only NVTX3; free when no tool
// is attached): profiles show each library call around its kernels.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
#define GS_NVTX(name) NvtxRange gs_nvtx_range_(name)

extern "C" {

const char* gs_last_error(void) { return g_err.c_str(); }
int gs_version(void) { return 1; }
int64_t gs_launch_count(void) { return (int64_t)g_launch_count.load(); }

int gs_pipeline_create(const GsPipelineDesc* d, gs_pipeline_t* out) {
  if (!d || !out || d->n_funcs <= 0 || d->n_funcs > 0x7FFF || d->n_stages < 0 || d->n_access < 0)
    return fail(GS_ERR_ARG, "bad pipeline descriptor");
  if (d->machine.warp_size != 32) return fail(GS_ERR_ARG, "only warp_size == 32 is supported");
  const int Mg = d->machine.global_transaction_bytes, Ms = d->machine.shared_banks * d->machine.bank_width_bytes;
  if (Mg < 1 || Mg > kMaxM || Ms < 1 || Ms > kMaxM)
    return fail(GS_ERR_ARG, "transaction / bank period must be in [1, 128] bytes");
  for (int s = 0; s < d->n_stages; ++s)
    if (d->stages[s].n_access > 0 && d->stages[s].access_begin + d->stages[s].n_access > d->n_access)
      return fail(GS_ERR_ARG, "stage access range out of bounds");
  auto* p = new GsPipeline();
  PipeDev& h = p->host;
  h.nf = d->n_funcs; h.ns = d->n_stages; h.na = d->n_access;
  int nd = 1, R = 0;
  for (int f = 0; f < h.nf; ++f) {
    nd = std::max(nd, d->funcs[f].ndim);
    if (!d->funcs[f].is_external) R += d->funcs[f].n_stages;
    if (d->funcs[f].n_stages > 255) { delete p; return fail(GS_ERR_ARG, "more than 255 stages in a func"); }
  }
  if (nd > GS_MAX_NDIM) { delete p; return fail(GS_ERR_ARG, "ndim > 4"); }
  h.nd = nd; h.max_rows = R; h.m = d->machine; h.th = d->thresholds;
  auto al = [](int x) { return (x + 15) & ~15; };
  h.off_stages = al(h.nf * (int)sizeof(GsFunc));
  h.off_access = h.off_stages + al(std::max(1, h.ns) * (int)sizeof(GsStage));
  h.blob_bytes = h.off_access + al(std::max(1, h.na) * (int)sizeof(GsAccess));
  std::vector<uint8_t> blob(h.blob_bytes, 0);
  memcpy(blob.data(), d->funcs, h.nf * sizeof(GsFunc));
  if (h.ns) memcpy(blob.data() + h.off_stages, d->stages, h.ns * sizeof(GsStage));
  if (h.na) memcpy(blob.data() + h.off_access, d->access, h.na * sizeof(GsAccess));
  // capacities for expanded reads / chain paths (per candidate, in shared memory)
  // Capacity bound for expanded reads / path entries of ANY decision log:
  // a stage of func g is expanded at most Q(g) times, Q(g) = 1 when g can
  // not be inlined, else max(1, sum of Q(consumer) over accesses reading g);
  // each access then appears in at most Q(its consumer) paths.
  {
    std::vector<int> Q(h.nf, 0), state(h.nf, 0), self(h.nf, 0);
    for (int a = 0; a < h.na; ++a)
      if (d->access[a].producer == d->access[a].consumer) self[d->access[a].producer] = 1;
    std::vector<std::vector<int>> readers(h.nf);
    for (int a = 0; a < h.na; ++a) readers[d->access[a].producer].push_back(d->access[a].consumer);
    // iterative post-order over the consumer DAG
    for (int root = 0; root < h.nf; ++root) {
      if (state[root] == 2) continue;
      std::vector<std::pair<int, size_t>> st{{root, 0}};
      state[root] = 1;
      while (!st.empty()) {
        auto& [g, it] = st.back();
        const bool elig = !d->funcs[g].is_output && !d->funcs[g].is_external && d->funcs[g].n_stages == 1 && !self[g];
        if (elig && it < readers[g].size()) {
          int c = readers[g][it++];
          if (state[c] == 0) { state[c] = 1; st.push_back({c, 0}); }
          continue;
        }
        long long q = 0;
        if (elig) for (int c : readers[g]) q += Q[c];
        Q[g] = (int)std::min<long long>(std::max<long long>(1, q), 1 << 20);
        state[g] = 2;
        st.pop_back();
      }
    }
    long long bound = 0;
    for (int a = 0; a < h.na; ++a) bound += Q[d->access[a].consumer];
    p->rcap = (int)std::min<long long>(32767, bound + 32);   // int16 read indices
    p->pcap = (int)std::min<long long>(65535, bound + 32);
  }
  cudaDeviceProp prop;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaGetDeviceProperties(&prop, dev));
  p->num_sms = prop.multiProcessorCount;
  p->max_smem = (int)prop.sharedMemPerBlockOptin;
  p->sm_smem = (int)prop.sharedMemPerMultiprocessor;
  p->cta_reserved = (int)prop.reservedSharedMemPerBlock;
  CK(cudaMalloc(&p->dev, sizeof(PipeDev)));
  CK(cudaMemcpy(p->dev, &h, sizeof(PipeDev), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&p->blob, h.blob_bytes));
  CK(cudaMemcpy(p->blob, blob.data(), h.blob_bytes, cudaMemcpyHostToDevice));
  p->hfuncs.assign(d->funcs, d->funcs + h.nf);
  std::vector<int32_t> sof(h.nf);
  for (int f = 0; f < h.nf; ++f) sof[f] = d->funcs[f].stage_begin;
  CK(cudaMalloc(&p->stage_of_func, 4 * h.nf));
  CK(cudaMemcpy(p->stage_of_func, sof.data(), 4 * h.nf, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&p->algo, 8 * GS_ALGO_DIM * std::max(1, h.ns)));
  if (h.ns) CK(cudaMemcpy(p->algo, d->algo, 8 * GS_ALGO_DIM * h.ns, cudaMemcpyHostToDevice));
  std::vector<int32_t> sorted(h.nf);
  for (int f = 0; f < h.nf; ++f) {
    int r = d->funcs[f].name_rank;
    if (r < 0 || r >= h.nf) { delete p; return fail(GS_ERR_ARG, "bad name_rank"); }
    sorted[r] = f;
  }
  CK(cudaMalloc(&p->sorted, 4 * h.nf));
  CK(cudaMemcpy(p->sorted, sorted.data(), 4 * h.nf, cudaMemcpyHostToDevice));
  const int nb = d->name_off[h.nf];
  {   // longest canonical repr any decision log can produce (K3 buffer choice):
      // header + per func "(name, 'fuse_at_thread', kernel, consumer, False, False), "
    int maxn = 4;
    for (int f = 0; f < h.nf; ++f) maxn = std::max(maxn, d->name_off[f + 1] - d->name_off[f]);
    long long b = 16;
    for (int f = 0; f < h.nf; ++f)
      b += 2 + 1 + (d->name_off[f + 1] - d->name_off[f]) + 2 + 16 + 2 + maxn + 2 + maxn + 14 + 1;
    p->repr_bound = (int)std::min<long long>(b, 1 << 30);
  }
  CK(cudaMalloc(&p->names, std::max(1, nb)));
  CK(cudaMemcpy(p->names, d->name_repr, nb, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&p->name_off, 4 * (h.nf + 1)));
  CK(cudaMemcpy(p->name_off, d->name_off, 4 * (h.nf + 1), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&p->err, 64));   // [0] error word, [2..13] K1 stats (u64), [14] K1 / [15] K2 work-unit counters
  CK(cudaMemset(p->err, 0, 64));
  *out = p;
  return GS_OK;
}

int gs_pipeline_destroy(gs_pipeline_t p) {
  if (!p) return GS_OK;
  cudaFree(p->dev); cudaFree(p->blob); cudaFree(p->stage_of_func); cudaFree(p->algo); cudaFree(p->sorted);
  cudaFree(p->names); cudaFree(p->name_off); cudaFree(p->err); cudaFree(p->hscratch); cudaFree(p->k1ws); cudaFree(p->simbuf);
  cudaFree(p->p1flags); cudaFree(p->p1cons_off); cudaFree(p->p1cons); cudaFree(p->p1order);
  for (double* b : p->wbufs) cudaFree(b);
  delete p;
  return GS_OK;
}

int gs_pipeline_max_rows(gs_pipeline_t p) { return p ? p->host.max_rows : 0; }

int gs_set_weights(gs_pipeline_t p, int E, int H, const double* aw, const double* ab, const double* sw,
                   const double* sb, const double* hw, const double* hb, const double* ow, const double* ob) {
  if (!p || E < 1 || E > 64 || H < 1 || H > 512) return fail(GS_ERR_ARG, "embed_dim must be in [1,64], hidden in [1,512]");
  for (double* b : p->wbufs) cudaFree(b);
  p->wbufs.clear();
  const double* src[8] = {aw, ab, sw, sb, hw, hb, ow, ob};
  const size_t cnt[8] = {(size_t)GS_ALGO_DIM * E, (size_t)E, (size_t)GS_NUM_FEATURES * E, (size_t)E,
                         (size_t)2 * E * H, (size_t)H, (size_t)H * GS_NUM_COEFFS, (size_t)GS_NUM_COEFFS};
  double* dst[8];
  for (int i = 0; i < 8; ++i) {
    CK(cudaMalloc(&dst[i], 8 * cnt[i]));
    CK(cudaMemcpy(dst[i], src[i], 8 * cnt[i], cudaMemcpyHostToDevice));
    p->wbufs.push_back(dst[i]);
  }
  double* hoisted;
  CK(cudaMalloc(&hoisted, 8 * (size_t)H * std::max(1, p->host.ns)));
  p->wbufs.push_back(hoisted);
  p->net = NetDev{E, H, dst[0], dst[1], dst[2], dst[3], dst[4], dst[5], dst[6], dst[7], hoisted};
  launch_hoist(p->net, p->algo, p->host.ns, 0);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  return GS_OK;
}

static Layout layout_for(gs_pipeline_t p, int S, int nwarps, int spill) {
  // machines other than the default (32 B transactions, 32 x 4 B banks) run
  // the generic counters and need their residue tables in the warp slice
  const GsMachine& m = p->host.m;
  const bool generic = !(m.global_transaction_bytes == 32 && m.shared_banks == 32 && m.bank_width_bytes == 4);
  return make_layout(p->host.nd, p->host.nf, p->host.ns, p->host.blob_bytes, S, std::max(1, p->host.max_rows),
                     p->rcap, p->pcap, nwarps, spill, generic);
}

int gs_set_reuse(gs_pipeline_t p, int enable) {
  if (!p) return fail(GS_ERR_ARG, "null pipeline");
  if (enable < 0 || enable > 2) return fail(GS_ERR_ARG, "reuse mode must be 0, 1 or 2");
  p->reuse = enable;
  return GS_OK;
}

int gs_get_reuse(gs_pipeline_t p) { return p ? p->reuse : -1; }

}  // extern "C"

// K1 launch shape and workspace.  One CTA per SM, as many independent
// scorer warps as shared memory holds; pipelines whose worst-case inline
// expansion would leave fewer than 4 warps keep the capacity-sized arrays
// in global scratch (`gscratch`) instead.  Batches of >= 8192 candidates
// with features may use the two-phase schedule: run ids / heads / count
// (device) and one saved warp state per run (`slots`, `max_runs` of them;
// the kernel falls back to the one-phase schedule when the batch has more
// runs, or runs shorter than 8 on average).
struct K1Plan {
  Layout L;              // modes 0 / 1 (one CTA per SM, as many warps as fit)
  int nwarps = 0;
  int64_t grid = 0;
  Layout L2;             // mode 2 (sibling slices): several smaller CTAs per SM
  int nwarps2 = 0;
  int64_t grid2 = 0;
  bool two_phase = false;
  int64_t slot_bytes = 0;
};

struct K1Ws {
  uint8_t* gscratch = nullptr;
  uint8_t* heads = nullptr;
  int32_t* run_id = nullptr;
  int32_t* run_head = nullptr;
  uint32_t* sums = nullptr;
  uint32_t* nruns = nullptr;
  uint8_t* slots = nullptr;
  int64_t max_runs = 0;
};

static int k1_plan(gs_pipeline_t p, int64_t n, int S, bool feats, int reuse, K1Plan& kp) {
  // Launch shapes (CTAs per SM x scorer warps per CTA).  The warps of a CTA
  // work in lockstep (featurize_kernel).  Both launches of the two-phase
  // schedule share one slice layout (the run-head launch saves warp states
  // the sibling launch restores), so they share the spill choice: the
  // capacity-sized structure arrays go to the warp's global scratch when
  // that buys more warps.  One CTA with the most warps runs best for every
  // mode now that a run slot saves only the persistent slice prefix:
  // 1M C5 step, sibling launch as 1 x 12 warps (spill 2) 58.5 ms K1, 2 x 5
  // (spill 1) 60.5 ms, 2 x 6 (spill 2) 62.7 ms; the 64K C2 steps 7.0 / 6.2
  // ms against 7.7 / 7.1 ms as 2 x 5 (earlier, with whole-slice slot
  // copies, 2 x 5 had won: 22.1 vs 23.1 ms on 240K candidates).
  // GS_K1_CTAS (sibling launch) / GS_K1_SPILL force the choice
  // (diagnostics).  Registers cap a SM at kK1MaxWarps warps.
  auto fit = [&](int ctas, int spill) {
    const Layout L1 = layout_for(p, S, 1, spill);
    const int per_cta = (p->sm_smem / ctas) - p->cta_reserved;
    const int budget = std::min(per_cta, p->max_smem) - L1.warps;
    const int w = budget > 0 ? budget / L1.warp_bytes : 0;
    return std::min({w, p->nwarps, kK1MaxWarps / ctas});
  };
  // the lowest spill level that reaches the most warps for `ctas`
  auto best = [&](int ctas) {
    int lvl = 0, w = fit(ctas, 0);
    for (int l = 1; l <= 2; ++l)
      if (fit(ctas, l) > w) { w = fit(ctas, l); lvl = l; }
    return lvl;
  };
  kp.two_phase = reuse && feats && n >= 8192;
  int spill = best(1);
  int ctas2 = 1;
  if (kp.two_phase) {
    if (const char* e = getenv("GS_K1_CTAS")) ctas2 = std::max(1, atoi(e));
    spill = best(ctas2);   // the sibling launch dominates: its best level for both launches
    if (fit(ctas2, spill) < 3) ctas2 = 1;   // too big for several CTAs per SM
  }
  if (const char* e = getenv("GS_K1_SPILL")) spill = std::min(2, std::max(0, atoi(e)));
  const int nwarps = fit(1, spill);
  if (nwarps < 1)
    return fail(GS_ERR_CAPACITY, "pipeline too large for one warp's shared-memory slice (" +
                                     std::to_string(layout_for(p, S, 1, 2).total) + " > " +
                                     std::to_string(p->max_smem) + " bytes)");
  kp.L = layout_for(p, S, nwarps, spill);
  kp.nwarps = nwarps;
  kp.grid = std::max<int64_t>(1, std::min<int64_t>((int64_t)p->num_sms, (n + nwarps - 1) / nwarps));
  kp.nwarps2 = std::max(1, fit(ctas2, spill));
  kp.L2 = layout_for(p, S, kp.nwarps2, spill);
  kp.grid2 = std::max<int64_t>(1, std::min<int64_t>((int64_t)p->num_sms * ctas2, (n + kp.nwarps2 - 1) / kp.nwarps2));
  kp.slot_bytes = (int64_t)kp.L.keep + kp.L.gkeep;   // persistent prefixes only
  return GS_OK;
}

static int64_t k1_default_runs(const K1Plan& kp, int64_t n) {
  return std::max<int64_t>(1, std::min<int64_t>(n / 8, ((int64_t)1 << 30) / std::max<int64_t>(1, kp.slot_bytes)));
}

// carve (base may be null: size only)
static int64_t k1_carve(const K1Plan& kp, int64_t n, int64_t max_runs, uint8_t* base, K1Ws& w) {
  int64_t o = 0;
  auto take = [&](int64_t bytes) { uint8_t* r = base ? base + o : nullptr; o += (bytes + 255) & ~(int64_t)255; return r; };
  w.gscratch = take(std::max(kp.grid * kp.nwarps, kp.grid2 * kp.nwarps2) * (int64_t)kp.L.gl_bytes);
  w.heads = take(std::max<int64_t>(1, n));
  w.max_runs = 0;
  if (kp.two_phase) {
    w.run_id = reinterpret_cast<int32_t*>(take(4 * n));
    w.run_head = reinterpret_cast<int32_t*>(take(4 * n));
    w.sums = reinterpret_cast<uint32_t*>(take((int64_t)k1_runs_sums_bytes(n)));
    w.nruns = reinterpret_cast<uint32_t*>(take(16));
    w.max_runs = max_runs;
    w.slots = take(max_runs * kp.slot_bytes);
  }
  return o;
}

// K1 with an explicit reuse mode, workspace and the optional per-row kernel output
static int featurize_impl(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, double* feats,
                          int32_t* row_key, int32_t* n_rows, uint8_t* verdict, int32_t* row_src,
                          int32_t* row_kernel, int reuse, const K1Plan& kp, const K1Ws& w, void* stream) {
  if (n == 0) return GS_OK;
  p->last_warps = kp.nwarps;
  p->last_slice = kp.L.warp_bytes;
  cudaStream_t st = (cudaStream_t)stream;
  int rc = 0;
  if (kp.two_phase) {
    // run heads first (each saves its warp state), then the siblings in
    // small slices that resume from their head's state, so runs split
    // across warps without re-resolving
    k1_prepare_runs(dec, n, S, w.heads, w.run_id, w.run_head, w.sums, w.nruns, st);
    for (int mode = 1; mode <= 2 && !rc; ++mode)
      rc = launch_featurize(p->host.nd, p->dev, p->blob, dec, n, S, feats, row_key, n_rows, verdict, row_src,
                            mode == 1 ? kp.L : kp.L2, mode == 1 ? kp.nwarps : kp.nwarps2,
                            (int)(mode == 1 ? kp.grid : kp.grid2), p->err, reuse, w.gscratch, w.heads, mode, w.run_id,
                            w.run_head, w.nruns, w.max_runs, w.slots, kp.slot_bytes, row_kernel, st);
  } else {
    rc = launch_featurize(p->host.nd, p->dev, p->blob, dec, n, S, feats, row_key, n_rows, verdict, row_src, kp.L,
                          kp.nwarps, (int)kp.grid, p->err, reuse, w.gscratch, w.heads, 0, nullptr, nullptr, nullptr,
                          0, nullptr, 0, row_kernel, st);
  }
  if (rc) return fail(GS_ERR_ARG, "unsupported ndim");
  CK(cudaGetLastError());
  return GS_OK;
}

// the convenience path: the library-owned K1 workspace, grown once per size
// class (synchronizing `stream` then)
static int featurize_owned(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, double* feats,
                           int32_t* row_key, int32_t* n_rows, uint8_t* verdict, int32_t* row_src,
                           int32_t* row_kernel, int reuse, void* stream) {
  if (n == 0) return GS_OK;
  K1Plan kp;
  int rc = k1_plan(p, n, S, feats != nullptr, reuse, kp);
  if (rc) return rc;
  K1Ws w;
  const int64_t runs = k1_default_runs(kp, n);
  const int64_t need = k1_carve(kp, n, runs, nullptr, w);
  if (need > p->k1cap) {
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    if (p->k1ws) CK(cudaFree(p->k1ws));
    p->k1ws = nullptr;
    p->k1cap = 0;
    CK(cudaMalloc(&p->k1ws, (size_t)need));
    p->k1cap = need;
  }
  k1_carve(kp, n, runs, p->k1ws, w);
  return featurize_impl(p, dec, n, S, feats, row_key, n_rows, verdict, row_src, row_kernel, reuse, kp, w, stream);
}

extern "C" {

int gs_featurize(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, double* feats, int32_t* row_key,
                 int32_t* n_rows, uint8_t* verdict, int32_t* row_src, void* stream) {
  GS_NVTX("gs_featurize");
  if (!p || S < 1 || n < 0) return fail(GS_ERR_ARG, "bad featurize arguments");
  if (p->reuse == 2 && feats && !row_src) return fail(GS_ERR_ARG, "reuse mode 2 (computed rows only) needs row_src");
  return featurize_owned(p, dec, n, S, feats, row_key, n_rows, verdict, row_src, nullptr, p->reuse, stream);
}

int64_t gs_featurize_workspace_bytes(gs_pipeline_t p, int64_t n, int s, int64_t max_runs) {
  if (!p || s < 1 || n < 0) return -1;
  K1Plan kp;
  if (k1_plan(p, std::max<int64_t>(n, 1), s, true, p->reuse, kp)) return -1;
  K1Ws w;
  return k1_carve(kp, n, max_runs > 0 ? max_runs : k1_default_runs(kp, n), nullptr, w);
}

int gs_featurize_ws(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, double* feats, int32_t* row_key,
                    int32_t* n_rows, uint8_t* verdict, int32_t* row_src, int64_t max_runs, void* workspace,
                    int64_t ws_bytes, void* stream) {
  GS_NVTX("gs_featurize_ws");
  if (!p || S < 1 || n < 0) return fail(GS_ERR_ARG, "bad featurize arguments");
  if (p->reuse == 2 && feats && !row_src) return fail(GS_ERR_ARG, "reuse mode 2 (computed rows only) needs row_src");
  if (n == 0) return GS_OK;
  K1Plan kp;
  int rc = k1_plan(p, n, S, feats != nullptr, p->reuse, kp);
  if (rc) return rc;
  K1Ws w;
  const int64_t runs = max_runs > 0 ? max_runs : k1_default_runs(kp, n);
  if (k1_carve(kp, n, runs, nullptr, w) > ws_bytes || (!workspace && ws_bytes > 0))
    return fail(GS_ERR_ARG, "featurize workspace too small (gs_featurize_workspace_bytes)");
  k1_carve(kp, n, runs, static_cast<uint8_t*>(workspace), w);
  return featurize_impl(p, dec, n, S, feats, row_key, n_rows, verdict, row_src, nullptr, p->reuse, kp, w, stream);
}

int gs_simulate(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, const GsOracleParams* op,
                double* runtime, int64_t* spill_bytes, uint8_t* status, void* stream) {
  GS_NVTX("gs_simulate");
  if (!p || !op || S < 1 || n < 0 || (n > 0 && (!dec || !runtime || !spill_bytes || !status)))
    return fail(GS_ERR_ARG, "bad simulate arguments");
  if (op->registers_per_thread_budget <= 0) return fail(GS_ERR_ARG, "registers_per_thread_budget must be positive");
  if (n == 0) return GS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const int R = std::max(1, p->host.max_rows);
  const int64_t fb = n * R * GS_NUM_FEATURES * 8, kb = ((n * R * 4 + 255) / 256) * 256;
  const int64_t need = fb + 2 * kb + ((n * 4 + 255) / 256) * 256 + n + 256;
  if (need > p->simcap) {
    CK(cudaStreamSynchronize(st));
    if (p->simbuf) CK(cudaFree(p->simbuf));
    p->simbuf = nullptr;
    p->simcap = 0;
    CK(cudaMalloc(&p->simbuf, (size_t)need));
    p->simcap = need;
  }
  double* feats = reinterpret_cast<double*>(p->simbuf);
  int32_t* row_key = reinterpret_cast<int32_t*>(p->simbuf + fb);
  int32_t* row_kernel = reinterpret_cast<int32_t*>(p->simbuf + fb + kb);
  int32_t* n_rows = reinterpret_cast<int32_t*>(p->simbuf + fb + 2 * kb);
  uint8_t* verdict = p->simbuf + fb + 2 * kb + ((n * 4 + 255) / 256) * 256;
  int rc = featurize_owned(p, dec, n, S, feats, row_key, n_rows, verdict, nullptr, row_kernel, p->reuse ? 1 : 0,
                           stream);
  if (rc) return rc;
  launch_simulate(reinterpret_cast<const GsFunc*>(p->blob), p->host.nf, dec, n, S, feats, row_key, n_rows,
                  row_kernel, R, p->stage_of_func, p->algo, p->host.m, *op, runtime, spill_bytes, status, st);
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_check(gs_pipeline_t p, void* stream) {
  if (!p) return fail(GS_ERR_ARG, "null pipeline");
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  int e = 0;
  CK(cudaMemcpy(&e, p->err, sizeof(int), cudaMemcpyDeviceToHost));
  CK(cudaMemset(p->err, 0, sizeof(int)));
  if (e & 32) return fail(GS_ERR_SCHEDULE, "illegal decision log (bad func / consumer / duplicate / no fusion source)");
  if (e) return fail(GS_ERR_CAPACITY, "candidate exceeded a device workspace capacity (flags " + std::to_string(e) + ")");
  return GS_OK;
}

int gs_cost(gs_pipeline_t p, const double* feats, const int32_t* row_key, const int32_t* n_rows,
            const int32_t* row_src, int64_t n, double* total, double* row_cost, double* basis_gh, void* stream) {
  GS_NVTX("gs_cost");
  if (!p || !p->net.sched_w) return fail(GS_ERR_ARG, "weights not set (gs_set_weights)");
  if (row_src && !row_cost) return fail(GS_ERR_ARG, "row reuse (row_src) needs the row_cost buffer");
  int rc = launch_cost(p->net, p->stage_of_func, feats, row_key, n_rows, row_src, n, std::max(1, p->host.max_rows),
                       total, row_cost, basis_gh, reinterpret_cast<unsigned*>(p->err + 15), p->num_sms,
                       (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "unsupported network dims");
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_cost_totals(gs_pipeline_t p, const double* feats, const int32_t* row_key, const int32_t* n_rows,
                   const int32_t* row_src, int64_t n, double* total, double* row_scratch, void* stream) {
  GS_NVTX("gs_cost_totals");
  if (!p || !p->net.sched_w) return fail(GS_ERR_ARG, "weights not set (gs_set_weights)");
  if (n > 0 && (!row_src || !row_scratch)) return fail(GS_ERR_ARG, "gs_cost_totals needs row_src and the row scratch");
  int rc = launch_cost(p->net, p->stage_of_func, feats, row_key, n_rows, row_src, n, std::max(1, p->host.max_rows),
                       total, row_scratch, nullptr, reinterpret_cast<unsigned*>(p->err + 15), p->num_sms,
                       (cudaStream_t)stream, false);
  if (rc) return fail(GS_ERR_ARG, "unsupported network dims");
  CK(cudaGetLastError());
  return GS_OK;
}

int64_t gs_struct_hash_workspace_bytes(int64_t n) { return (std::max<int64_t>(1, n) + 255) & ~(int64_t)255; }

int gs_struct_hash_ws(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, int depth, uint64_t* out,
                      void* workspace, int64_t ws_bytes, void* stream) {
  GS_NVTX("gs_struct_hash_ws");
  if (!p || depth < 0) return fail(GS_ERR_ARG, "depth must be >= 0");
  if (ws_bytes < gs_struct_hash_workspace_bytes(n) || !workspace)
    return fail(GS_ERR_ARG, "hash workspace too small (gs_struct_hash_workspace_bytes)");
  return gs_struct_hash_depths_ws(p, dec, n, S, 1, &depth, out, workspace, ws_bytes, stream);
}

int gs_struct_hash_depths_ws(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, int ndepths,
                             const int* depths, uint64_t* out, void* workspace, int64_t ws_bytes, void* stream) {
  GS_NVTX("gs_struct_hash_depths_ws");
  if (!p || ndepths < 1 || ndepths > 4 || !depths) return fail(GS_ERR_ARG, "1..4 depths");
  HashDepths D{};
  D.n = ndepths;
  for (int k = 0; k < ndepths; ++k) {
    if (depths[k] < 0) return fail(GS_ERR_ARG, "depth must be >= 0");
    D.d[k] = depths[k];
  }
  if (ws_bytes < gs_struct_hash_workspace_bytes(n) || !workspace)
    return fail(GS_ERR_ARG, "hash workspace too small (gs_struct_hash_workspace_bytes)");
  int rc = launch_hash(dec, n, S, p->host.nf, D, p->sorted, p->names, p->name_off, out,
                       static_cast<uint8_t*>(workspace), p->repr_bound, p->num_sms, (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "too many funcs for the hash kernel");
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_struct_hash(gs_pipeline_t p, const GsDecision* dec, int64_t n, int S, int depth, uint64_t* out,
                   void* stream) {
  GS_NVTX("gs_struct_hash");
  if (!p || depth < 0) return fail(GS_ERR_ARG, "depth must be >= 0");
  if (n > p->hcap) {   // one-time growth of the run-head scratch
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    if (p->hscratch) CK(cudaFree(p->hscratch));
    p->hscratch = nullptr;
    p->hcap = 0;
    CK(cudaMalloc(&p->hscratch, (size_t)n));
    p->hcap = n;
  }
  HashDepths D{};
  D.n = 1;
  D.d[0] = depth;
  int rc = launch_hash(dec, n, S, p->host.nf, D, p->sorted, p->names, p->name_off, out, p->hscratch,
                       p->repr_bound, p->num_sms, (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "too many funcs for the hash kernel");
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_stats(gs_pipeline_t p, int64_t* out, void* stream) {
  if (!p || !out) return fail(GS_ERR_ARG, "null argument");
  CK(cudaStreamSynchronize((cudaStream_t)stream));
  CK(cudaMemcpy(out, p->err + 2, 5 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  CK(cudaMemset(p->err + 2, 0, 6 * sizeof(int64_t)));
  out[5] = (int64_t)p->last_warps << 32 | p->last_slice;
  return GS_OK;
}

int gs_debug_phases(int64_t* out) {
  if (!out) return fail(GS_ERR_ARG, "null argument");
  CK(cudaDeviceSynchronize());
  if (read_phases(reinterpret_cast<long long*>(out))) return fail(GS_ERR_CUDA, "phase counters unavailable");
  return GS_OK;
}

int64_t gs_select_workspace_bytes(int64_t n) { return select_workspace_bytes(n); }

int gs_select_reps(const uint64_t* hashes, const uint8_t* verdict, int64_t n, uint64_t phase_seed, void* ws,
                   int64_t ws_bytes, int64_t* rep_idx, int64_t* n_reps, int64_t* rej_idx, int64_t* n_rejects,
                   void* stream) {
  GS_NVTX("gs_select_reps");
  int rc = select_reps(hashes, verdict, n, phase_seed, ws, ws_bytes, rep_idx, n_reps, n_rejects, rej_idx,
                       (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "select_reps: workspace too small or n too large");
  CK(cudaGetLastError());
  return GS_OK;
}

int64_t gs_topk_workspace_bytes(int64_t n) { return topk_workspace_bytes(n); }

int64_t gs_expand_workspace_bytes(int64_t n_parents) { return expand_workspace_bytes(n_parents); }

int gs_expand_step(gs_pipeline_t p, const GsDecision* parents, int64_t n_parents, int s, const int32_t* step,
                   const GsTilingMenus* menus, int64_t* offsets, void* workspace, int64_t ws_bytes, GsDecision* out,
                   int64_t out_cap, int32_t* owner, void* stream) {
  GS_NVTX("gs_expand_step");
  if (!p || !menus || !offsets || s < 1 || n_parents < 0) return fail(GS_ERR_ARG, "bad expand arguments");
  const GsTilingMenus& m = *menus;
  if (m.n_serial_powers < 0 || m.n_serial_powers > 8 || m.n_odd_serial < 0 || m.n_odd_serial > 8 ||
      m.n_innermost < 1 || m.n_innermost > 8 || m.n_outer < 1 || m.n_outer > 8 || m.warp_size < 1)
    return fail(GS_ERR_ARG, "tiling menus out of range");
  for (int i = 0; i < m.n_serial_powers; ++i)
    if (m.serial_powers[i] < 1 || m.serial_powers[i] > 255) return fail(GS_ERR_ARG, "serial menu value out of range");
  for (int i = 0; i < m.n_odd_serial; ++i)
    if (m.odd_serial[i] < 1 || m.odd_serial[i] > 255) return fail(GS_ERR_ARG, "serial menu value out of range");
  for (int i = 0; i < m.n_innermost; ++i)
    if (m.innermost_thread[i] < 1 || m.innermost_thread[i] > 255) return fail(GS_ERR_ARG, "thread menu value out of range");
  for (int i = 0; i < m.n_outer; ++i)
    if (m.outer_thread[i] < 1 || m.outer_thread[i] > 255) return fail(GS_ERR_ARG, "thread menu value out of range");
  int rc = launch_expand(reinterpret_cast<const GsFunc*>(p->blob), parents, n_parents, s, step, m, offsets, workspace,
                         ws_bytes, out, out_cap, owner, p->err, p->num_sms, (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "expand: workspace too small or more than 2^20 parents");
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_beam_topk(const double* costs, const uint64_t* pass_hash, int64_t n, const uint64_t* flagged,
                 int64_t n_flagged, double penalty, double temperature, uint64_t phase_seed, int64_t k, double tie_band, void* ws,
                 int64_t ws_bytes, int64_t* out_pos, int64_t* n_out, uint8_t* bottom, void* stream) {
  GS_NVTX("gs_beam_topk");
  int rc = beam_topk(costs, pass_hash, nullptr, n, nullptr, flagged, n_flagged, penalty, temperature, phase_seed, k,
                     tie_band, ws, ws_bytes, out_pos, n_out, bottom, (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "beam_topk: workspace too small, k out of 1..16384 or negative tie band");
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_beam_topk_reps(const double* costs, const uint64_t* pass_hash, const int64_t* rep_idx, int64_t n_max,
                      const int64_t* n_reps, const uint64_t* flagged, int64_t n_flagged, double penalty,
                      double temperature, uint64_t phase_seed, int64_t k, double tie_band, void* ws, int64_t ws_bytes,
                      int64_t* out_pos, int64_t* n_out, uint8_t* bottom, void* stream) {
  GS_NVTX("gs_beam_topk_reps");
  if (!rep_idx || !n_reps) return fail(GS_ERR_ARG, "beam_topk_reps: rep_idx and n_reps are required");
  int rc = beam_topk(costs, pass_hash, rep_idx, n_max, n_reps, flagged, n_flagged, penalty, temperature, phase_seed, k,
                     tie_band, ws, ws_bytes, out_pos, n_out, bottom, (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "beam_topk: workspace too small, k out of 1..16384 or negative tie band");
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_model_params(int E, int H) { return (E < 1 || H < 1) ? -1 : model_params(E, H); }

int gs_predict(const double* weights, int E, int H, const double* algo, const double* sched, const double* coeffs_in,
               int64_t n, double* coeffs_out, double* breakdown, void* stream) {
  GS_NVTX("gs_predict");
  if (!weights && !coeffs_in) return fail(GS_ERR_ARG, "predict: weights or coefficients required");
  if (!sched && breakdown) return fail(GS_ERR_ARG, "predict: the breakdown needs the schedule features");
  if (!coeffs_in && (!algo || !sched)) return fail(GS_ERR_ARG, "predict: the network needs algo and schedule rows");
  if (launch_predict(weights, E, H, algo, sched, coeffs_in, n, coeffs_out, breakdown, (cudaStream_t)stream))
    return fail(GS_ERR_ARG, "predict: unsupported network dims (2*embed <= 128)");
  CK(cudaGetLastError());
  return GS_OK;
}

int64_t gs_train_workspace_bytes(int E, int H, int max_rows) {
  if (E < 1 || H < 1 || max_rows < 0) return -1;
  return train_cache_bytes(E, H, max_rows);
}

int gs_train(double* weights, int E, int H, const double* algo, const double* sched, const double* g, const double* h,
             const int64_t* row_off, const double* runtime, const int32_t* order, int n_samples, int epochs,
             double learning_rate, double momentum, int max_rows, void* workspace, int64_t ws_bytes, double* loss_hist,
             int* status, void* stream) {
  GS_NVTX("gs_train");
  if (!weights || n_samples < 1 || epochs < 0 || max_rows < 1 || max_rows > 1024)
    return fail(GS_ERR_ARG, "train: bad arguments (1..1024 stage rows per sample)");
  if (ws_bytes < train_cache_bytes(E, H, max_rows) || !workspace)
    return fail(GS_ERR_ARG, "train: workspace too small (gs_train_workspace_bytes)");
  int rc = launch_train(weights, E, H, algo, sched, g, h, row_off, runtime, order, n_samples, epochs, learning_rate,
                        momentum, static_cast<double*>(workspace), loss_hist, status, (cudaStream_t)stream);
  if (rc) return fail(GS_ERR_ARG, "train: unsupported network dims (embed, hidden <= 64)");
  CK(cudaGetLastError());
  return GS_OK;
}

int gs_set_placement_info(gs_pipeline_t p, const uint8_t* flags, const int32_t* cons_off, const int32_t* cons,
                          const int32_t* sched_order, int n_sched) {
  if (!p || !flags || !cons_off || (n_sched > 0 && !sched_order) || n_sched < 0) return fail(GS_ERR_ARG, "null argument");
  for (int i = 0; i < n_sched; ++i)
    if (sched_order[i] < 0 || sched_order[i] >= p->host.nf) return fail(GS_ERR_ARG, "schedule order out of range");
  const int nf = p->host.nf;
  const int nc = cons_off[nf];
  if (cons_off[0] != 0 || nc < 0 || (nc > 0 && !cons)) return fail(GS_ERR_ARG, "bad consumer CSR");
  std::vector<int16_t> c16(std::max(1, nc));
  for (int i = 0; i < nc; ++i) {
    if (cons[i] < 0 || cons[i] >= nf) return fail(GS_ERR_ARG, "consumer index out of range");
    c16[i] = (int16_t)cons[i];
  }
  cudaFree(p->p1flags); cudaFree(p->p1cons_off); cudaFree(p->p1cons);
  p->p1flags = nullptr; p->p1cons_off = nullptr; p->p1cons = nullptr;
  CK(cudaMalloc(&p->p1flags, std::max(1, nf)));
  CK(cudaMemcpy(p->p1flags, flags, nf, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&p->p1cons_off, 4 * (nf + 1)));
  CK(cudaMemcpy(p->p1cons_off, cons_off, 4 * (nf + 1), cudaMemcpyHostToDevice));
  CK(cudaMalloc(&p->p1cons, 2 * c16.size()));
  CK(cudaMemcpy(p->p1cons, c16.data(), 2 * c16.size(), cudaMemcpyHostToDevice));
  cudaFree(p->p1order);
  p->p1order = nullptr;
  CK(cudaMalloc(&p->p1order, 4 * std::max(1, n_sched)));
  if (n_sched) CK(cudaMemcpy(p->p1order, sched_order, 4 * n_sched, cudaMemcpyHostToDevice));
  p->p1norder = n_sched;
  return GS_OK;
}

int gs_random_schedules(gs_pipeline_t p, uint64_t seed, int64_t first, int64_t n, int s, const GsTilingMenus* menus,
                        GsDecision* out, void* stream) {
  GS_NVTX("gs_random_schedules");
  if (!p || !menus || !out || s < 1 || n < 0 || first < 0) return fail(GS_ERR_ARG, "bad random-schedule arguments");
  if (!p->p1flags) return fail(GS_ERR_ARG, "placement info not set (gs_set_placement_info)");
  if (s < p->p1norder) return fail(GS_ERR_ARG, "record stride below the number of schedulable funcs");
  P1Static st{p->p1flags, p->p1cons_off, p->p1cons, p->sorted};
  const int rc = launch_random_schedules(reinterpret_cast<const GsFunc*>(p->blob), p->host.nf, st, p->p1order,
                                        p->p1norder, *menus, seed, first, n, s, out, p->err, (cudaStream_t)stream);
  if (rc == -3) return fail(GS_ERR_CUDA, "random schedules: could not raise the per-thread stack limit");
  if (rc) return fail(GS_ERR_ARG, "random schedules: more than 512 funcs");
  CK(cudaGetLastError());
  return GS_OK;
}

int64_t gs_phase1_workspace_bytes(int64_t n_parents) { return phase1_workspace_bytes(n_parents); }

int gs_expand_phase1(gs_pipeline_t p, const GsDecision* parents, int64_t n_parents, int s, int func,
                     int restrict_mask, const GsTilingMenus* menus, int64_t* offsets, void* workspace,
                     int64_t ws_bytes, GsDecision* out, int64_t out_cap, int32_t* owner, void* stream) {
  GS_NVTX("gs_expand_phase1");
  if (!p || !menus || !offsets || s < 1 || n_parents < 0) return fail(GS_ERR_ARG, "bad phase-1 arguments");
  if (!p->p1flags) return fail(GS_ERR_ARG, "placement info not set (gs_set_placement_info)");
  if (func < 0 || func >= p->host.nf || p->hfuncs[func].is_external)
    return fail(GS_ERR_ARG, "func out of range or an external input");
  const GsTilingMenus& m = *menus;
  if (m.n_serial_powers < 0 || m.n_serial_powers > 8 || m.n_odd_serial < 0 || m.n_odd_serial > 8 || m.warp_size < 1)
    return fail(GS_ERR_ARG, "tiling menus out of range");
  const int nser = serial_count(m, p->hfuncs[func]);
  P1Static st{p->p1flags, p->p1cons_off, p->p1cons, p->sorted};
  int rc = launch_phase1(reinterpret_cast<const GsFunc*>(p->blob), p->host.nf, st, parents, n_parents, s, func,
                         restrict_mask & 0xF, m, nser, offsets, workspace, ws_bytes, out, out_cap, owner, p->err,
                         p->num_sms, (cudaStream_t)stream);
  if (rc == -1) return fail(GS_ERR_ARG, "phase 1: more than 2^20 parents or 512 funcs");
  if (rc == -3) return fail(GS_ERR_CUDA, "phase 1: could not raise the per-thread stack limit");
  if (rc) return fail(GS_ERR_ARG, "phase 1: workspace too small (gs_phase1_workspace_bytes)");
  CK(cudaGetLastError());
  return GS_OK;
}

}  // extern "C"
