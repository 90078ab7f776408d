// K7 — the cost model off the beam-step path: coefficients and the six-term
// stage-cost breakdown for arbitrary (algo, schedule) rows, and on-device
// training (reference costmodel.py:34-115 stage_cost / CostBreakdown,
// 271-293 _forward, 296-313 _backward, 316-337 predict_coefficients /
// pipeline_cost, 391-432 train).
//
// Weights travel as one packed fp64 array in the reference's tensor order
// (costmodel.py:183-193): algo_w[10][E] algo_b[E] sched_w[56][E] sched_b[E]
// head_w[2E][H] head_b[H] out_w[H][30] out_b[30].
//
// predict_kernel: one thread per row.  Network as K2 (fp64, FMA chains);
// the breakdown follows stage_cost term by term with explicit
// round-to-nearest multiplies / adds / divides (no FMA contraction), so for
// given coefficients it is bit-identical to the reference.
//
// train_kernel: the reference's SGD-with-momentum loop is sequential over
// samples (every sample updates the weights the next one sees), so ONE CTA
// runs all epochs: the weights live in shared memory, each thread owns
// ~8 parameters (their velocities in registers), and per sample
//   forward   — one warp per stage row (lanes over the hidden units), the
//               activations cached in global scratch (L2-resident);
//   loss      — thread 0 sums the rows' g.c + h in row order, exactly the
//               reference's `total += float(g @ coeffs) + h`;
//   backward  — one warp per row for the deltas, then every thread sums its
//               parameters' outer-product terms over the rows in row order
//               (the reference's `grads += np.outer(...)` order: bit-exact
//               given equal activations) and applies v = m*v - lr*g, w += v
//               with the reference's rounding steps.
#include "gs_internal.cuh"

namespace gs {

constexpr double kModelEps = 1e-8;   // costmodel.py:27
constexpr int kTrainNT = 1024;
constexpr int kTrainOwn = 16;        // parameters per thread (E, H <= 64: 8286 <= 16 x 1024)

struct WOff {   // offsets of the packed tensors
  int aw, ab, sw, sb, hw, hb, ow, ob, total;
  __host__ __device__ WOff(int E, int H) {
    aw = 0; ab = aw + GS_ALGO_DIM * E; sw = ab + E; sb = sw + GS_NUM_FEATURES * E; hw = sb + E;
    hb = hw + 2 * E * H; ow = hb + H; ob = ow + H * GS_NUM_COEFFS; total = ob + GS_NUM_COEFFS;
  }
};

__device__ __forceinline__ double npy_logaddexp0(double z) {   // numpy logaddexp(0, z)
  if (z == 0.0) return 0.6931471805599453;
  const double t = -z;
  if (t > 0) return log1p(exp(-t));
  return z + log1p(exp(t));
}

// reference stage_cost (costmodel.py:50-115); out: compute, load, store,
// malloc, parallelism, working_set, total
__device__ void stage_cost_terms(const double* __restrict__ f, const double* __restrict__ c, double* out) {
  auto F = [&](int i) { return f[i]; };
  const bool inl = F(50) > 0;
  double compute = __dmul_rn(F(0), inl ? c[3] : c[1]);
  const double num_threads = __dmul_rn(F(23), F(26));
  const double points = __dmul_rn(num_threads, F(1));
  compute = __dadd_rn(compute, __dmul_rn(points, inl ? c[4] : c[19]));
  const double idle = __ddiv_rn(ceil(__ddiv_rn(F(46), F(49))), fmax(1.0, F(48)));
  compute = __dmul_rn(compute, idle);
  if (!inl) compute = __ddiv_rn(compute, __dsub_rn(1.0, F(30)));
  // num_realizations * (c5 UGLr + c16 USLr + c8 URLr + c6 UGBr + c20 USBr + c7 URBr
  //                     + c18 UGLt + c17 USLt + c2 URLt + c13 UGBt + c11 USBt + c0 URBt)
  const int ci[12] = {5, 16, 8, 6, 20, 7, 18, 17, 2, 13, 11, 0};
  const int fi[12] = {5, 6, 7, 2, 3, 4, 11, 12, 13, 8, 9, 10};
  double s = __dmul_rn(c[ci[0]], F(fi[0]));
#pragma unroll
  for (int i = 1; i < 12; ++i) s = __dadd_rn(s, __dmul_rn(c[ci[i]], F(fi[i])));
  double load = __dmul_rn(F(44), s);
  load = __dadd_rn(load, __dmul_rn(__dmul_rn(c[10], F(0)), F(51)));
  load = __dadd_rn(load, __dmul_rn(__dmul_rn(c[12], F(0)), F(52)));
  load = __dadd_rn(load, __dmul_rn(__dmul_rn(c[14], F(46)), F(53)));
  load = __dadd_rn(load, __dmul_rn(__dmul_rn(c[15], F(46)), F(54)));
  double gl = __dmul_rn(F(23), F(32));
  if (!inl) gl = __dmul_rn(gl, __ddiv_rn(1.0, F(38)));
  double sl = __dmul_rn(F(23), F(31));
  if (!inl) sl = __dmul_rn(sl, __ddiv_rn(1.0, F(36)));
  load = __dadd_rn(__dadd_rn(load, gl), sl);
  const double sst = __dmul_rn(__dmul_rn(c[29], F(23)), F(33));
  double gst = __dmul_rn(__dmul_rn(c[21], F(23)), F(34));
  if (!inl) gst = __dmul_rn(gst, __ddiv_rn(1.0, F(37)));
  double store = __dadd_rn(sst, gst);
  if (F(47) > 1) store = __dadd_rn(store, __ddiv_rn(__dmul_rn(c[22], F(0)), fmax(1.0, F(20))));
  const double malloc_ = __dmul_rn(c[24], F(44));
  const double launches = __dmul_rn(F(45), F(47) > 1 ? c[25] : 0.0);
  const double tasks = __dmul_rn(__dmul_rn(F(45), __dsub_rn(F(47), 1.0)), c[26]);
  const double par = __dadd_rn(tasks, launches);
  const double ws = __dmul_rn(F(55), c[9]);
  out[0] = compute; out[1] = load; out[2] = store; out[3] = malloc_; out[4] = par; out[5] = ws;
  // CostBreakdown.total: compute + store + load + malloc + parallelism + working_set
  out[6] = __dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(__dadd_rn(compute, store), load), malloc_), par), ws);
}

// one row's forward (thread-serial): coefficients c[30]
__device__ void forward_row(const double* __restrict__ w, int E, int H, const double* __restrict__ xa,
                            const double* __restrict__ sched, double* __restrict__ c) {
  const WOff o(E, H);
  double h1[128];
  for (int j = 0; j < E; ++j) {
    double za = 0.0, zs = 0.0;
    for (int i = 0; i < GS_ALGO_DIM; ++i) za = fma(xa[i], w[o.aw + i * E + j], za);
    for (int i = 0; i < GS_NUM_FEATURES; ++i) zs = fma(log1p(sched[i]), w[o.sw + i * E + j], zs);
    za += w[o.ab + j];
    zs += w[o.sb + j];
    h1[j] = za > 0.0 ? za : 0.0;
    h1[E + j] = zs > 0.0 ? zs : 0.0;
  }
  double zo[GS_NUM_COEFFS];
  for (int k = 0; k < GS_NUM_COEFFS; ++k) zo[k] = 0.0;
  for (int u = 0; u < H; ++u) {
    double z = 0.0;
    for (int j = 0; j < 2 * E; ++j) z = fma(h1[j], w[o.hw + j * H + u], z);
    z += w[o.hb + u];
    if (z > 0.0)
      for (int k = 0; k < GS_NUM_COEFFS; ++k) zo[k] = fma(z, w[o.ow + u * GS_NUM_COEFFS + k], zo[k]);
  }
  for (int k = 0; k < GS_NUM_COEFFS; ++k) c[k] = npy_logaddexp0(zo[k] + w[o.ob + k]) + kModelEps;
}

__global__ void predict_kernel(const double* __restrict__ w, int E, int H, const double* __restrict__ algo,
                               const double* __restrict__ sched, const double* __restrict__ cin, int64_t n,
                               double* __restrict__ cout, double* __restrict__ breakdown) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  double c[GS_NUM_COEFFS];
  if (cin) {
    for (int k = 0; k < GS_NUM_COEFFS; ++k) c[k] = cin[r * GS_NUM_COEFFS + k];
  } else {
    forward_row(w, E, H, algo + r * GS_ALGO_DIM, sched + r * GS_NUM_FEATURES, c);
  }
  if (cout)
    for (int k = 0; k < GS_NUM_COEFFS; ++k) cout[r * GS_NUM_COEFFS + k] = c[k];
  if (breakdown) stage_cost_terms(sched + r * GS_NUM_FEATURES, c, breakdown + r * 7);
}

// ---------------------------------------------------------------- training --
// per-row activation cache in global scratch (doubles)
struct RowCache {
  int xs, za, zs, zh, zo, dzo, dzh, dza, dzs, stride;
  __host__ __device__ RowCache(int E, int H) {
    xs = 0; za = xs + GS_NUM_FEATURES; zs = za + E; zh = zs + E; zo = zh + H; dzo = zo + GS_NUM_COEFFS;
    dzh = dzo + GS_NUM_COEFFS; dza = dzh + H; dzs = dza + E; stride = dzs + E;
  }
};

__global__ void __launch_bounds__(kTrainNT, 1) train_kernel(
    double* __restrict__ wglob, int E, int H, const double* __restrict__ algo, const double* __restrict__ sched,
    const double* __restrict__ g, const double* __restrict__ h, const int64_t* __restrict__ row_off,
    const double* __restrict__ runtime, const int32_t* __restrict__ order, int n_samples, int epochs, double lr,
    double momentum, double* __restrict__ cache, double* __restrict__ loss_hist, int* __restrict__ status) {
  extern __shared__ __align__(16) double wsm[];   // packed weights
  __shared__ double s_val[1024];                  // per-row g.c + h (rows <= 1024)
  __shared__ double s_dtotal;
  __shared__ int s_bad;
  const WOff o(E, H);
  const RowCache rc(E, H);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = kTrainNT / 32;
  for (int i = tid; i < o.total; i += kTrainNT) wsm[i] = wglob[i];
  double vel[kTrainOwn];
#pragma unroll
  for (int k = 0; k < kTrainOwn; ++k) vel[k] = 0.0;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  for (int ep = 0; ep < epochs; ++ep) {
    double epoch_loss = 0.0;   // thread 0
    for (int q = 0; q < n_samples; ++q) {
      const int smp = order[(int64_t)ep * n_samples + q];
      const int64_t r0 = row_off[smp];
      const int nr = (int)(row_off[smp + 1] - r0);
      // ---- forward: one warp per row
      for (int r = warp; r < nr; r += nwarps) {
        double* cr = cache + (int64_t)r * rc.stride;
        const double* xa = algo + (r0 + r) * GS_ALGO_DIM;
        const double* sc = sched + (r0 + r) * GS_NUM_FEATURES;
        for (int i = lane; i < GS_NUM_FEATURES; i += 32) cr[rc.xs + i] = log1p(sc[i]);
        __syncwarp();
        for (int j = lane; j < E; j += 32) {
          double za = 0.0, zs = 0.0;
          for (int i = 0; i < GS_ALGO_DIM; ++i) za = fma(xa[i], wsm[o.aw + i * E + j], za);
          for (int i = 0; i < GS_NUM_FEATURES; ++i) zs = fma(cr[rc.xs + i], wsm[o.sw + i * E + j], zs);
          cr[rc.za + j] = za + wsm[o.ab + j];
          cr[rc.zs + j] = zs + wsm[o.sb + j];
        }
        __syncwarp();
        for (int u = lane; u < H; u += 32) {
          double z = 0.0;
          for (int j = 0; j < E; ++j) z = fma(fmax(cr[rc.za + j], 0.0), wsm[o.hw + j * H + u], z);
          for (int j = 0; j < E; ++j) z = fma(fmax(cr[rc.zs + j], 0.0), wsm[o.hw + (E + j) * H + u], z);
          cr[rc.zh + u] = z + wsm[o.hb + u];
        }
        __syncwarp();
        double part = 0.0;
        if (lane < GS_NUM_COEFFS) {
          double z = 0.0;
          for (int u = 0; u < H; ++u) z = fma(fmax(cr[rc.zh + u], 0.0), wsm[o.ow + u * GS_NUM_COEFFS + lane], z);
          z += wsm[o.ob + lane];
          cr[rc.zo + lane] = z;
          const double c = npy_logaddexp0(z) + kModelEps;
          part = __dmul_rn(g[(r0 + r) * GS_NUM_COEFFS + lane], c);
        }
        // g . c in coefficient order (a sequential dot), then + h
        double dot = 0.0;
        for (int k = 0; k < GS_NUM_COEFFS; ++k) dot = __dadd_rn(dot, __shfl_sync(0xffffffffu, part, k));
        if (lane == 0) s_val[r] = __dadd_rn(dot, h[r0 + r]);
        __syncwarp();
      }
      __syncthreads();
      if (tid == 0) {
        double total = 0.0;
        for (int r = 0; r < nr; ++r) total = __dadd_rn(total, s_val[r]);
        if (!isfinite(total) || total <= 0.0) {
          s_bad = smp + 1;
        } else {
          const double err = __dsub_rn(log(total), log(runtime[smp]));
          epoch_loss = __dadd_rn(epoch_loss, __dmul_rn(err, err));
          s_dtotal = __ddiv_rn(__dmul_rn(2.0, err), total);
        }
      }
      __syncthreads();
      if (s_bad) break;
      const double dtotal = s_dtotal;
      // ---- backward deltas: one warp per row
      for (int r = warp; r < nr; r += nwarps) {
        double* cr = cache + (int64_t)r * rc.stride;
        if (lane < GS_NUM_COEFFS) {
          const double zo = cr[rc.zo + lane];
          const double dc = __dmul_rn(dtotal, g[(r0 + r) * GS_NUM_COEFFS + lane]);
          cr[rc.dzo + lane] = __dmul_rn(dc, exp(-npy_logaddexp0(-zo)));   // softplus' = sigmoid
        }
        __syncwarp();
        for (int u = lane; u < H; u += 32) {   // deh = dzo W_o^T; dzh = deh * (zh > 0)
          double d = 0.0;
          for (int k = 0; k < GS_NUM_COEFFS; ++k) d = fma(cr[rc.dzo + k], wsm[o.ow + u * GS_NUM_COEFFS + k], d);
          cr[rc.dzh + u] = cr[rc.zh + u] > 0.0 ? d : 0.0;
        }
        __syncwarp();
        for (int j = lane; j < 2 * E; j += 32) {   // dh1 = dzh W_h^T
          double d = 0.0;
          for (int u = 0; u < H; ++u) d = fma(cr[rc.dzh + u], wsm[o.hw + j * H + u], d);
          if (j < E) cr[rc.dza + j] = cr[rc.za + j] > 0.0 ? d : 0.0;
          else cr[rc.dzs + (j - E)] = cr[rc.zs + (j - E)] > 0.0 ? d : 0.0;
        }
        __syncwarp();
      }
      __syncthreads();
      // ---- gradients (row order) + momentum update of this thread's parameters
#pragma unroll 1
      for (int k = 0; k < kTrainOwn; ++k) {
        const int p = tid + k * kTrainNT;
        if (p >= o.total) break;
        double gr = 0.0;
        if (p < o.ab) {                          // algo_w[i][j] += xa_i dza_j
          const int i = p / E, j = p % E;
          for (int r = 0; r < nr; ++r)
            gr = __dadd_rn(gr, __dmul_rn(algo[(r0 + r) * GS_ALGO_DIM + i], cache[(int64_t)r * rc.stride + rc.dza + j]));
        } else if (p < o.sw) {                   // algo_b
          const int j = p - o.ab;
          for (int r = 0; r < nr; ++r) gr = __dadd_rn(gr, cache[(int64_t)r * rc.stride + rc.dza + j]);
        } else if (p < o.sb) {                   // sched_w[i][j] += xs_i dzs_j
          const int i = (p - o.sw) / E, j = (p - o.sw) % E;
          for (int r = 0; r < nr; ++r) {
            const double* cr = cache + (int64_t)r * rc.stride;
            gr = __dadd_rn(gr, __dmul_rn(cr[rc.xs + i], cr[rc.dzs + j]));
          }
        } else if (p < o.hw) {                   // sched_b
          const int j = p - o.sb;
          for (int r = 0; r < nr; ++r) gr = __dadd_rn(gr, cache[(int64_t)r * rc.stride + rc.dzs + j]);
        } else if (p < o.hb) {                   // head_w[i][u] += h1_i dzh_u
          const int i = (p - o.hw) / H, u = (p - o.hw) % H;
          for (int r = 0; r < nr; ++r) {
            const double* cr = cache + (int64_t)r * rc.stride;
            const double x = i < E ? fmax(cr[rc.za + i], 0.0) : fmax(cr[rc.zs + i - E], 0.0);
            gr = __dadd_rn(gr, __dmul_rn(x, cr[rc.dzh + u]));
          }
        } else if (p < o.ow) {                   // head_b
          const int u = p - o.hb;
          for (int r = 0; r < nr; ++r) gr = __dadd_rn(gr, cache[(int64_t)r * rc.stride + rc.dzh + u]);
        } else if (p < o.ob) {                   // out_w[u][k] += eh_u dzo_k
          const int u = (p - o.ow) / GS_NUM_COEFFS, kk = (p - o.ow) % GS_NUM_COEFFS;
          for (int r = 0; r < nr; ++r) {
            const double* cr = cache + (int64_t)r * rc.stride;
            gr = __dadd_rn(gr, __dmul_rn(fmax(cr[rc.zh + u], 0.0), cr[rc.dzo + kk]));
          }
        } else {                                 // out_b
          const int kk = p - o.ob;
          for (int r = 0; r < nr; ++r) gr = __dadd_rn(gr, cache[(int64_t)r * rc.stride + rc.dzo + kk]);
        }
        vel[k] = __dsub_rn(__dmul_rn(momentum, vel[k]), __dmul_rn(lr, gr));
      }
      __syncthreads();   // every forward/backward read of the weights is done
#pragma unroll
      for (int k = 0; k < kTrainOwn; ++k) {
        const int p = tid + k * kTrainNT;
        if (p < o.total) wsm[p] = __dadd_rn(wsm[p], vel[k]);
      }
      __syncthreads();
    }
    if (s_bad) break;
    if (tid == 0) loss_hist[ep] = __ddiv_rn(epoch_loss, (double)n_samples);
  }
  if (tid == 0) *status = s_bad;
  for (int i = tid; i < o.total; i += kTrainNT) wglob[i] = wsm[i];
}

int64_t train_cache_bytes(int E, int H, int max_rows) {
  const RowCache rc(E, H);
  return (int64_t)8 * rc.stride * (max_rows > 0 ? max_rows : 1);
}

int model_params(int E, int H) { return WOff(E, H).total; }

int launch_predict(const double* w, int E, int H, const double* algo, const double* sched, const double* cin,
                   int64_t n, double* cout, double* breakdown, cudaStream_t st) {
  if (n <= 0) return 0;
  if (E < 1 || H < 1 || 2 * E > 128) return -1;
  predict_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(w, E, H, algo, sched, cin, n, cout, breakdown);
  g_launch_count++;
  return 0;
}

int launch_train(double* w, int E, int H, const double* algo, const double* sched, const double* g, const double* h,
                 const int64_t* row_off, const double* runtime, const int32_t* order, int n_samples, int epochs,
                 double lr, double momentum, double* cache, double* loss_hist, int* status, cudaStream_t st) {
  if (E < 1 || H < 1 || E > 64 || H > 64) return -1;
  const int smem = 8 * WOff(E, H).total;
  if (cudaFuncSetAttribute(train_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess) return -2;
  train_kernel<<<1, kTrainNT, smem, st>>>(w, E, H, algo, sched, g, h, row_off, runtime, order, n_samples, epochs, lr,
                                          momentum, cache, loss_hist, status);
  g_launch_count++;
  return 0;
}

}  // namespace gs
