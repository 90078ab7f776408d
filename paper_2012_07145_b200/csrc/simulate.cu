// K6 — batched machine oracle: the reference's
// deterministic stand-in for compiling and benchmarking a schedule,
// `simulate_runtime` (machine.py:108-167), over K1's feature rows.
//
// One thread per candidate.  Kernels are visited in the reference's order
// (cs.kernels: compute_root decisions in decision order, resolve.py:258) and
// each kernel's member rows in row order (the featurize dict order), so
// every fp64 sum and product is formed in the reference's order, with no
// FMA contraction.
#include "gs_internal.cuh"

namespace gs {

// feature indices (reference FEATURE_ORDER)
constexpr int kNumScalars = 0, kNumBlocks = 23, kShLoads = 31, kGlLoads = 32, kShStores = 33, kGlStores = 34,
              kWsThread = 39, kMaxWarpOcc = 42;

__global__ void simulate_kernel(const GsFunc* __restrict__ funcs, int nf, const GsDecision* __restrict__ dec,
                                int64_t n, int S, const double* __restrict__ feats, const int32_t* __restrict__ row_key,
                                const int32_t* __restrict__ n_rows, const int32_t* __restrict__ row_kernel, int R,
                                const int32_t* __restrict__ stage_of_func, const double* __restrict__ algo,
                                GsMachine m, GsOracleParams op, double* __restrict__ runtime,
                                int64_t* __restrict__ spill_bytes, uint8_t* __restrict__ status) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const GsDecision* d = dec + c * S;
  const int nr = n_rows[c];
  const int32_t* rk = row_kernel + c * R;
  // fully scheduled (loopnest.py:112-124; the reference raises ValueError):
  // every non-external func has a decision, roots carry serial and thread
  // tilings, fuse_at_block decisions a serial tiling
  int scheduled = 0, required = 0;
  bool tiled = true;
  for (int f = 0; f < nf; ++f) required += !funcs[f].is_external;
  for (int i = 0; i < S; ++i) {
    if (d[i].func == 0xFFFF) continue;
    ++scheduled;
    if (d[i].kind == GS_ROOT && (d[i].flags & 3) != 3) tiled = false;
    if (d[i].kind == GS_FUSE_BLOCK && !(d[i].flags & 1)) tiled = false;
  }
  uint8_t st = scheduled == required && tiled ? 0 : 2;
  // hardware limits of any kernel (validate_limits; the reference raises)
  for (int r = 0; r < nr && st == 0; ++r)
    if (rk[r] >= 0 && (rk[r] & 0x40000000)) st = 1;
  const int64_t budget = (int64_t)op.registers_per_thread_budget * 4;   // register_bytes_per_thread
  double total = 0.0;
  int64_t spill = 0;
  if (st == 0) {
    for (int i = 0; i < S; ++i) {
      if (d[i].func == 0xFFFF || d[i].kind != GS_ROOT) continue;
      const int owner = d[i].func;
      double work = 0.0, gbytes = 0.0, sbytes = 0.0, occ = 1.0, blocks = 0.0;
      int64_t kspill = 0;
      bool first = true;
      for (int r = 0; r < nr; ++r) {
        if (rk[r] < 0 || (rk[r] & 0x3FFFFFFF) != owner) continue;
        const double* F = feats + ((int64_t)c * R + r) * GS_NUM_FEATURES;
        const int key = row_key[(int64_t)c * R + r];
        const double* a = algo + (int64_t)(stage_of_func[key >> 8] + (key & 255)) * GS_ALGO_DIM;
        double ops = 0.0;   // float(sum(op_counts)): small integers, exact
        for (int q = 0; q < 7; ++q) ops = __dadd_rn(ops, a[q]);
        work = __dadd_rn(work, __dmul_rn(F[kNumScalars], __dadd_rn(1.0, ops)));
        gbytes = __dadd_rn(gbytes, __dmul_rn(__dmul_rn(F[kNumBlocks], __dadd_rn(F[kGlLoads], F[kGlStores])),
                                             (double)m.global_transaction_bytes));
        sbytes = __dadd_rn(sbytes, __dmul_rn(__dmul_rn(__dmul_rn(F[kNumBlocks], __dadd_rn(F[kShLoads], F[kShStores])),
                                                       (double)m.shared_banks),
                                             (double)m.bank_width_bytes));
        if (F[kMaxWarpOcc] < occ) occ = F[kMaxWarpOcc];
        const int64_t ws = (int64_t)F[kWsThread];   // int(): truncation
        if (ws > budget && ws - budget > kspill) kspill = ws - budget;
        if (first) { blocks = F[kNumBlocks]; first = false; }   // kern.num_blocks
      }
      double balance = __ddiv_rn(blocks, __dmul_rn(2.0, (double)m.num_sms));
      if (balance > 1.0) balance = 1.0;
      double util = __dmul_rn(occ, balance);
      if (util < 1e-3) util = 1e-3;
      const double ct = __ddiv_rn(work, __dmul_rn(op.compute_throughput, util));
      const double mt = __dadd_rn(__ddiv_rn(gbytes, op.global_bandwidth), __ddiv_rn(sbytes, op.shared_bandwidth));
      double t = ct >= mt ? ct : mt;
      if (kspill > 0) {
        spill += kspill;
        t = __dmul_rn(t, __dadd_rn(2.0, __ddiv_rn((double)kspill, (double)budget)));
      }
      total = __dadd_rn(total, __dadd_rn(t, op.kernel_launch_overhead));
    }
  }
  runtime[c] = st == 0 ? total : __longlong_as_double(0x7FF8000000000000ll);
  spill_bytes[c] = spill;
  status[c] = st;
}

int launch_simulate(const GsFunc* funcs, int nf, const GsDecision* dec, int64_t n, int S, const double* feats,
                    const int32_t* row_key, const int32_t* n_rows, const int32_t* row_kernel, int R,
                    const int32_t* stage_of_func, const double* algo, const GsMachine& m, const GsOracleParams& op,
                    double* runtime, int64_t* spill_bytes, uint8_t* status, cudaStream_t st) {
  if (n == 0) return 0;
  simulate_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(funcs, nf, dec, n, S, feats, row_key, n_rows,
                                                              row_kernel, R, stage_of_func, algo, m, op, runtime,
                                                              spill_bytes, status);
  g_launch_count++;
  return 0;
}

}  // namespace gs
