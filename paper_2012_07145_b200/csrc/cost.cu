// K2 — basis (g, h) + two-tower coefficient network + g.c + h + in-order
// stage sum, fused over a feature tile (reference costmodel.py:118-176,
// 271-293; search.py:115-124).
//
// Layout: one thread per stage row; the network weights (fp64) live in
// shared memory and are read as warp-wide broadcasts; the algorithm-side
// tower and its head contribution are hoisted to one 64-vector per stage
// (`hoist_kernel`, recomputed only when the weights change).  Per-row costs
// go to a shared-memory tile and one thread per candidate adds them up in
// row order, exactly the reference's `total += c` sequence.
// Arithmetic is fp64 end to end (the reference is fp64; parity target 1e-5
// relative, measured ~1e-15), the basis without FMA contraction.
#include "gs_internal.cuh"
#include "fastmath.cuh"

namespace gs {

constexpr double kEps = 1e-8;

__global__ void hoist_kernel(NetDev net, const double* __restrict__ algo, int n_stages) {
  int s = blockIdx.x;
  if (s >= n_stages) return;
  __shared__ double ea[128];
  const int E = net.E, H = net.H;
  for (int j = threadIdx.x; j < E; j += blockDim.x) {
    double z = net.algo_b[j];
    for (int i = 0; i < GS_ALGO_DIM; ++i) z = fma(algo[s * GS_ALGO_DIM + i], net.algo_w[i * E + j], z);
    ea[j] = z > 0.0 ? z : 0.0;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < H; o += blockDim.x) {
    double z = net.head_b[o];
    for (int j = 0; j < E; ++j) z = fma(ea[j], net.head_w[j * H + o], z);
    net.hoisted[s * H + o] = z;
  }
}

// numpy npy_logaddexp(0, z): z == 0 -> log 2; z < 0 -> log1p(exp(z));
// z > 0 -> z + log1p(exp(-z)).  Written without branches: exp and log1p
// see the same argument bits (exp(-|z|)) and 0 + v = v on the z < 0 side,
// so two independent evaluations can interleave.
__device__ __forceinline__ double softplus_bf(double z) {
  const double v = fmax(z, 0.0) + log1p_fast(exp(-fabs(z)));
  return z == 0.0 ? 0.6931471805599453 : v;
}

// reference stage_cost_basis (costmodel.py:118-176): fills g, returns h
__device__ __forceinline__ double basis_g(const double* __restrict__ f, double* g) {
  auto F = [&](int i) { return f[i]; };
  const bool inl = F(50) > 0;
  double scale = __ddiv_rn(ceil(__ddiv_rn(F(46), F(49))), fmax(1.0, F(48)));
  if (!inl) scale = __ddiv_rn(scale, __dsub_rn(1.0, F(30)));
  const double pts = __dmul_rn(__dmul_rn(F(23), F(26)), F(1));
#pragma unroll
  for (int i = 0; i < GS_NUM_COEFFS; ++i) g[i] = 0.0;
  g[inl ? 3 : 1] = __dmul_rn(F(0), scale);
  g[inl ? 4 : 19] = __dmul_rn(pts, scale);
  const double r = F(44);
  g[5] = __dmul_rn(r, F(5));  g[16] = __dmul_rn(r, F(6));  g[8] = __dmul_rn(r, F(7));
  g[6] = __dmul_rn(r, F(2));  g[20] = __dmul_rn(r, F(3));  g[7] = __dmul_rn(r, F(4));
  g[18] = __dmul_rn(r, F(11)); g[17] = __dmul_rn(r, F(12)); g[2] = __dmul_rn(r, F(13));
  g[13] = __dmul_rn(r, F(8)); g[11] = __dmul_rn(r, F(9));  g[0] = __dmul_rn(r, F(10));
  g[10] = __dmul_rn(F(0), F(51));
  g[12] = __dmul_rn(F(0), F(52));
  g[14] = __dmul_rn(F(46), F(53));
  g[15] = __dmul_rn(F(46), F(54));
  double gl = __dmul_rn(F(23), F(32));
  double sl = __dmul_rn(F(23), F(31));
  if (!inl) { gl = __ddiv_rn(gl, F(38)); sl = __ddiv_rn(sl, F(36)); }
  const double h = __dadd_rn(gl, sl);
  g[29] = __dmul_rn(F(23), F(33));
  double gs = __dmul_rn(F(23), F(34));
  if (!inl) gs = __ddiv_rn(gs, F(37));
  g[21] = gs;
  if (F(47) > 1) g[22] = __ddiv_rn(F(0), fmax(1.0, F(20)));
  g[24] = F(44);
  if (F(47) > 1) g[25] = F(45);
  g[26] = __dmul_rn(F(45), __dsub_rn(F(47), 1.0));
  g[9] = F(55);
  return h;
}

// returns g.c + h, writes g and h to gout (may be null)
// c: the 30 coefficients, strided by ZS (per-thread column of a
// shared-memory scratch; ZS = threads per block)
template <int ZS>
__device__ double basis_dot(const double* __restrict__ f, const double* __restrict__ c, double* gout) {
  double g[GS_NUM_COEFFS];
  const double h = basis_g(f, g);
  double dot = 0.0;
#pragma unroll
  for (int i = 0; i < GS_NUM_COEFFS; ++i) dot = fma(g[i], c[i * ZS], dot);
  if (gout) {
#pragma unroll
    for (int i = 0; i < GS_NUM_COEFFS; ++i) gout[i] = g[i];
    gout[GS_NUM_COEFFS] = h;
  }
  return __dadd_rn(dot, h);
}

template <int MAXE, int ZS>
__device__ double stage_row_cost(const NetDev& net, const double* __restrict__ sw, const double* __restrict__ whs,
                           const double* __restrict__ wo, const double* __restrict__ bs,
                           const double* __restrict__ bo, const double* __restrict__ f, int stage,
                           double* gout, double* zs) {
  const int E = net.E, H = net.H;
  double es[MAXE];
#pragma unroll
  for (int j = 0; j < MAXE; ++j) es[j] = j < E ? bs[j] : 0.0;
  for (int k = 0; k < GS_NUM_FEATURES; ++k) {
    const double fk = f[k];
    const double x = fk == 0.0 ? 0.0 : log1p_fast(fk);   // log1p(+0) = +0: skip the sequence for absent features
#pragma unroll
    for (int j = 0; j < MAXE; ++j) if (j < E) es[j] = fma(x, sw[k * E + j], es[j]);
  }
#pragma unroll
  for (int j = 0; j < MAXE; ++j) es[j] = es[j] > 0.0 ? es[j] : 0.0;
  double zo[GS_NUM_COEFFS];
#pragma unroll
  for (int o = 0; o < GS_NUM_COEFFS; ++o) zo[o] = bo[o];
  const double* hp = net.hoisted + (int64_t)stage * H;
  // four hidden units at a time: four independent FMA chains over the
  // embedding (the single chain is latency-bound), same per-unit order
  constexpr int HU = 4;   // 1M C5 K2: 2 units 9.65 ms, 4 8.40 ms, 8 8.85 ms
  int i = 0;
  for (; i + HU <= H; i += HU) {
    double z[HU];
#pragma unroll
    for (int u = 0; u < HU; ++u) z[u] = __ldg(hp + i + u);
#pragma unroll
    for (int j = 0; j < MAXE; ++j)
      if (j < E) {
        const double* wr = whs + j * H + i;
#pragma unroll
        for (int u = 0; u < HU; ++u) z[u] = fma(es[j], wr[u], z[u]);
      }
#pragma unroll
    for (int u = 0; u < HU; ++u) {
      if (z[u] > 0.0) {
#pragma unroll
        for (int o = 0; o < GS_NUM_COEFFS; ++o) zo[o] = fma(z[u], wo[(i + u) * GS_NUM_COEFFS + o], zo[o]);
      }
    }
  }
  for (; i < H; ++i) {
    double z = __ldg(hp + i);
#pragma unroll
    for (int j = 0; j < MAXE; ++j) if (j < E) z = fma(es[j], whs[j * H + i], z);
    if (z > 0.0) {
#pragma unroll
      for (int o = 0; o < GS_NUM_COEFFS; ++o) zo[o] = fma(z, wo[i * GS_NUM_COEFFS + o], zo[o]);
    }
  }
  // softplus through a per-thread shared-memory column and a rolled loop:
  // thirty inlined exp + log1p sequences were ~80% of the kernel's code
  // and overflowed the instruction cache
#pragma unroll
  for (int o = 0; o < GS_NUM_COEFFS; ++o) zs[o * ZS] = zo[o];
  // two independent (branch-free) evaluations per step: one exp + log1p
  // sequence alone is a dependent chain the warp cannot hide (8.65 -> 8.40
  // ms per 1M C5 K2; three per step: 8.8 ms)
  static_assert(GS_NUM_COEFFS % 2 == 0, "");
#pragma unroll 1
  for (int o = 0; o < GS_NUM_COEFFS; o += 2) {
    const double a = softplus_bf(zs[o * ZS]), b = softplus_bf(zs[(o + 1) * ZS]);
    zs[o * ZS] = a + kEps;
    zs[(o + 1) * ZS] = b + kEps;
  }
  return basis_dot<ZS>(f, zs, gout);
}

template <int MAXE>
__global__ void __launch_bounds__(128) cost_kernel(NetDev net, const int32_t* __restrict__ stage_of_func,
                                                   const double* __restrict__ feats,
                                                   const int32_t* __restrict__ row_key,
                                                   const int32_t* __restrict__ n_rows, int64_t n, int R, int CB,
                                                   double* __restrict__ total, double* __restrict__ row_cost,
                                                   double* __restrict__ basis_gh) {
  extern __shared__ __align__(16) double smd[];
  const int E = net.E, H = net.H;
  double* sw = smd;                          // 56*E
  double* whs = sw + GS_NUM_FEATURES * E;    // E*H (sched half of head_w)
  double* wo = whs + E * H;                  // H*30
  double* bs = wo + H * GS_NUM_COEFFS;       // E
  double* bo = bs + E;                       // 30
  double* buf = bo + GS_NUM_COEFFS;          // CB*R
  double* zs = buf + CB * R + threadIdx.x;   // 30 x 128 softplus scratch
  for (int i = threadIdx.x; i < GS_NUM_FEATURES * E; i += blockDim.x) sw[i] = net.sched_w[i];
  for (int i = threadIdx.x; i < E * H; i += blockDim.x) whs[i] = net.head_w[E * H + i];
  for (int i = threadIdx.x; i < H * GS_NUM_COEFFS; i += blockDim.x) wo[i] = net.out_w[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) bs[i] = net.sched_b[i];
  for (int i = threadIdx.x; i < GS_NUM_COEFFS; i += blockDim.x) bo[i] = net.out_b[i];
  __syncthreads();
  for (int64_t c0 = (int64_t)blockIdx.x * CB; c0 < n; c0 += (int64_t)gridDim.x * CB) {
    const int ncb = (int)((n - c0) < CB ? (n - c0) : CB);
    for (int idx = threadIdx.x; idx < ncb * R; idx += blockDim.x) {
      const int cl = idx / R, r = idx % R;
      const int64_t c = c0 + cl;
      if (r >= n_rows[c]) continue;
      const int64_t row = c * R + r;
      const int key = row_key[row];
      const int stage = stage_of_func[key >> 8] + (key & 255);
      const double v = stage_row_cost<MAXE, 128>(net, sw, whs, wo, bs, bo, feats + row * GS_NUM_FEATURES, stage,
                                       basis_gh ? basis_gh + row * (GS_NUM_COEFFS + 1) : nullptr, zs);
      buf[idx] = v;
      if (row_cost) row_cost[row] = v;
    }
    __syncthreads();
    if (threadIdx.x < ncb) {
      const int64_t c = c0 + threadIdx.x;
      double t = 0.0;
      const int nr = n_rows[c];
      for (int r = 0; r < nr; ++r) t = __dadd_rn(t, buf[threadIdx.x * R + r]);
      total[c] = t;
    }
    __syncthreads();
  }
}

// Exact row reuse (gs_featurize row_src): a row whose features repeat
// candidate row_src[row]'s row bit for bit has that row's cost, so the
// network runs once per distinct row.  Pass A: every warp scans 32-row
// slabs (2048-row spans, round-robin over the grid) and queues its computed rows in a
// 64-entry shared-memory ring; whenever 32 are queued, one per lane runs
// the network, so lanes stay full and no block-wide barrier or per-chunk
// tail idles the SM.  Pass B gathers every row's cost from its source and
// adds a candidate's rows in order.
#ifndef GS_K2_WARPS
#define GS_K2_WARPS 12
#endif
constexpr int kRowsWarps = GS_K2_WARPS;   // one CTA per SM; 240K C5: 8 warps 3.08 ms, 12 2.63 ms, 16 (128 registers, spills) 3.24 ms
constexpr unsigned kRing = 256;   // per-warp queue (>= 31 + kBatch slabs x 32)

template <int MAXE>
__global__ void __launch_bounds__(kRowsWarps * 32, 1) cost_rows_kernel(NetDev net, const int32_t* __restrict__ stage_of_func,
                                                        const double* __restrict__ feats,
                                                        const int32_t* __restrict__ row_key,
                                                        const int32_t* __restrict__ n_rows,
                                                        const int32_t* __restrict__ row_src, int64_t n, int R,
                                                        double* __restrict__ row_cost, unsigned* __restrict__ work,
                                                        int64_t kSpan) {
  extern __shared__ __align__(16) double smd[];
  __shared__ int64_t ring[kRowsWarps][kRing];
  const int E = net.E, H = net.H;
  double* sw = smd;
  double* whs = sw + GS_NUM_FEATURES * E;
  double* wo = whs + E * H;
  double* bs = wo + H * GS_NUM_COEFFS;
  double* bo = bs + E;
  double* zs = bo + GS_NUM_COEFFS + threadIdx.x;   // 30 x (threads) softplus scratch
  for (int i = threadIdx.x; i < GS_NUM_FEATURES * E; i += blockDim.x) sw[i] = net.sched_w[i];
  for (int i = threadIdx.x; i < E * H; i += blockDim.x) whs[i] = net.head_w[E * H + i];
  for (int i = threadIdx.x; i < H * GS_NUM_COEFFS; i += blockDim.x) wo[i] = net.out_w[i];
  for (int i = threadIdx.x; i < E; i += blockDim.x) bs[i] = net.sched_b[i];
  for (int i = threadIdx.x; i < GS_NUM_COEFFS; i += blockDim.x) bo[i] = net.out_b[i];
  __syncthreads();
  const int64_t total_rows = n * (int64_t)R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t* q = ring[warp];
  auto run = [&](int64_t row) {
    const int key = row_key[row];
    const int stage = stage_of_func[key >> 8] + (key & 255);
    row_cost[row] = stage_row_cost<MAXE, kRowsWarps * 32>(net, sw, whs, wo, bs, bo, feats + row * GS_NUM_FEATURES, stage, nullptr,
                                         zs);
  };
  // warps take 2048-row spans and walk a span's slabs in
  // order, so a queue holds rows of neighbouring candidates (siblings: the
  // same stages, similar features, little divergence).  The ownership
  // flags of 4 slabs are loaded together (4 loads in flight per lane) into
  // a circular queue; the network is evaluated at ONE call site (its code
  // is large: a second inlined copy would thrash the instruction cache).
  // kSpan: rows per claimed span (a multiple of 32 x kBatch; smaller for
  // small batches, so every warp gets spans)
  constexpr int kBatch = 4;
  // spans are claimed dynamically (the computed-row density varies along
  // the batch, so a static round-robin leaves SMs idle at the end)
  auto claim = [&]() -> int64_t {
    unsigned v = 0;
    if (lane == 0) v = atomicAdd(work, 1u);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  int64_t sp = claim(), s0 = sp * kSpan;
  unsigned head = 0, tail = 0;
  for (;;) {
    while (tail - head < 32 && s0 < total_rows) {
      const int64_t end = sp * kSpan + kSpan < total_rows ? sp * kSpan + kSpan : total_rows;
      unsigned tm = 0;
#pragma unroll
      for (int u = 0; u < kBatch; ++u) {
        const int64_t row = s0 + 32 * u + lane;
        if (row < end) {
          const int64_t c = row / R;
          const int r = (int)(row - c * R);
          tm |= (unsigned)(r < __ldg(n_rows + c) && __ldg(row_src + row) == (int32_t)c) << u;
        }
      }
#pragma unroll 1
      for (int u = 0; u < kBatch; ++u) {
        const bool t = (tm >> u) & 1u;
        const unsigned b = __ballot_sync(0xffffffffu, t);
        if (t) q[(tail + __popc(b & ((1u << lane) - 1))) & (kRing - 1)] = s0 + 32 * u + lane;
        tail += __popc(b);
      }
      s0 += 32 * kBatch;
      if (s0 >= end) { sp = claim(); s0 = sp * kSpan; }
    }
    if (tail == head) break;
    __syncwarp();
    if (head + lane < tail) run(q[(head + lane) & (kRing - 1)]);
    head += tail - head < 32 ? tail - head : 32;
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// K2 on the fp64 tensor cores (DMMA m8n8k4).  Same queue/claim structure as
// cost_rows_kernel, but a warp evaluates its 32 queued rows TOGETHER: the
// three layers are 32-row GEMMs (X[32x56]·Ws, relu(E)[32xE]·Whs[E:], relu(Z)
// [32xH]·Wo) issued as m8n8k4 fp64 MMAs, one per 256 FMAs instead of one
// DFMA per 32.  The weights live in shared memory pre-arranged in B-fragment
// order (frag[kb][nb][lane] = B[4kb + lane%4][8nb + lane/4]), so each
// fragment is one conflict-free 8-byte load per lane.  The log1p of the
// features is taken directly in A-fragment order (lane 4r+j owns
// X[r][4kb+j]); C fragments are turned into the next layer's A fragments
// with quad shuffles.  The pre-softplus outputs go through a per-warp
// shared-memory tile so that the row's owner lane does softplus + the basis
// dot exactly as the scalar path does.  The MMAs accumulate in the scalar
// chains' order (bias, then k ascending, FMA rounding per step): costs are
// bit-identical to cost_kernel's (tests/test_gpu_reuse.py asserts equality).
#ifndef GS_K2M_WARPS
#define GS_K2M_WARPS 16
#endif
constexpr int kMmaWarps = GS_K2M_WARPS;
constexpr unsigned kRingM = 512;   // per-warp queue of row indices (< 2^32 rows per launch)
constexpr int kCS = 33;   // per-warp coefficient tile row stride (doubles)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// A fragment of k-block (4h + j) within an 8-column C tile: lane 4r+j takes
// column 4h+j of row r, held by lane 4r + 2h + j/2 as element j%2
__device__ __forceinline__ double c_to_a(double c0, double c1, int h, int lane) {
  const int src = (lane & ~3) | (2 * h + ((lane & 3) >> 1));
  const double v0 = __shfl_sync(0xffffffffu, c0, src), v1 = __shfl_sync(0xffffffffu, c1, src);
  return (lane & 1) ? v1 : v0;
}

template <int E, int H>
__global__ void __launch_bounds__(kMmaWarps * 32, 1) cost_rows_mma_kernel(
    NetDev net, const int32_t* __restrict__ stage_of_func, const double* __restrict__ feats,
    const int32_t* __restrict__ row_key, const int32_t* __restrict__ n_rows, const int32_t* __restrict__ row_src,
    int64_t n, int R, double* __restrict__ row_cost, unsigned* __restrict__ work, int64_t kSpan) {
  static_assert(E % 8 == 0 && H % 8 == 0 && E <= 64 && H <= 128, "");
  constexpr int KB1 = GS_NUM_FEATURES / 4, NB1 = E / 8;   // layer 1: 14 k-blocks x E/8 n-tiles
  constexpr int KB2 = E / 4, NB2 = H / 8;                 // layer 2
  constexpr int NB3 = 4;                                  // 30 coefficients padded to 32
  extern __shared__ __align__(16) double smd[];
  __shared__ uint32_t ring[kMmaWarps][kRingM];
  double* w1 = smd;                          // KB1*NB1*32
  double* w2 = w1 + KB1 * NB1 * 32;          // KB2*NB2*32
  double* w3 = w2 + KB2 * NB2 * 32;          // (H/4)*NB3*32
  double* bs = w3 + (H / 4) * NB3 * 32;      // E
  double* bo = bs + E;                       // 32
  double* cs = bo + 32;                      // kMmaWarps x 32 x kCS
  for (int i = threadIdx.x; i < KB1 * NB1 * 32; i += blockDim.x) {
    const int l = i & 31, t = i >> 5, nb = t % NB1, kb = t / NB1;
    w1[i] = net.sched_w[(4 * kb + (l & 3)) * E + 8 * nb + (l >> 2)];
  }
  for (int i = threadIdx.x; i < KB2 * NB2 * 32; i += blockDim.x) {
    const int l = i & 31, t = i >> 5, nb = t % NB2, kb = t / NB2;
    w2[i] = net.head_w[(E + 4 * kb + (l & 3)) * H + 8 * nb + (l >> 2)];
  }
  for (int i = threadIdx.x; i < (H / 4) * NB3 * 32; i += blockDim.x) {
    const int l = i & 31, t = i >> 5, nb = t % NB3, kb = t / NB3;
    const int o = 8 * nb + (l >> 2);
    w3[i] = o < GS_NUM_COEFFS ? net.out_w[(4 * kb + (l & 3)) * GS_NUM_COEFFS + o] : 0.0;
  }
  for (int i = threadIdx.x; i < E; i += blockDim.x) bs[i] = net.sched_b[i];
  for (int i = threadIdx.x; i < 32; i += blockDim.x) bo[i] = i < GS_NUM_COEFFS ? net.out_b[i] : 0.0;
  __syncthreads();
  const int64_t total_rows = n * (int64_t)R;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int qr = lane >> 2, qc = lane & 3;
  uint32_t* q = ring[warp];
  double* ct = cs + warp * 32 * kCS;

  // the warp's 32 queued rows (cnt valid; the rest repeat row 0 and are not written)
  auto run_warp = [&](unsigned h0, int cnt) {
    int64_t rrow[4];
    const double* hz[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int r = 8 * mt + qr;
      rrow[mt] = q[(h0 + (r < cnt ? r : 0)) & (kRingM - 1)];
      const int key = __ldg(row_key + rrow[mt]);
      hz[mt] = net.hoisted + (int64_t)(stage_of_func[key >> 8] + (key & 255)) * H;
    }
    // layer 1: E1 = relu(log1p(X) Ws + bs)
    double e1[4][NB1][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nb = 0; nb < NB1; ++nb) {
        e1[mt][nb][0] = bs[8 * nb + 2 * qc];
        e1[mt][nb][1] = bs[8 * nb + 2 * qc + 1];
      }
    // feature loads run two k-blocks ahead of their log1p (the loads are
    // L2 / HBM latency; without the prefetch they were the top stall)
    const double* fp[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) fp[mt] = feats + rrow[mt] * GS_NUM_FEATURES + qc;
    double f0[4], f1[4];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) { f0[mt] = __ldg(fp[mt]); f1[mt] = __ldg(fp[mt] + 4); }
#pragma unroll 1
    for (int kb = 0; kb < KB1; ++kb) {
      double a[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const double fk = f0[mt];
        f0[mt] = f1[mt];
        if (kb + 2 < KB1) f1[mt] = __ldg(fp[mt] + 4 * (kb + 2));
        a[mt] = fk == 0.0 ? 0.0 : log1p_fast(fk);
      }
#pragma unroll
      for (int nb = 0; nb < NB1; ++nb) {
        const double b = w1[(kb * NB1 + nb) * 32 + lane];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(e1[mt][nb][0], e1[mt][nb][1], a[mt], b);
      }
    }
    // relu(E1) as layer-2 A fragments, parked in the warp's coefficient tile
    // (fragment order: one conflict-free load per lane; keeps the 32 doubles
    // out of registers so 16 warps fit without spills)
    static_assert(4 * KB2 * 32 <= 32 * kCS, "");
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nb = 0; nb < NB1; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          ct[(mt * KB2 + 2 * nb + h) * 32 + lane] =
              c_to_a(fmax(e1[mt][nb][0], 0.0), fmax(e1[mt][nb][1], 0.0), h, lane);
    __syncwarp();
    // layers 2 + 3, one 8-unit block of the hidden layer at a time
    double zo[4][NB3][2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int ot = 0; ot < NB3; ++ot) {
        zo[mt][ot][0] = bo[8 * ot + 2 * qc];
        zo[mt][ot][1] = bo[8 * ot + 2 * qc + 1];
      }
#pragma unroll 1
    for (int nb = 0; nb < NB2; ++nb) {
      double z[4][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        z[mt][0] = __ldg(hz[mt] + 8 * nb + 2 * qc);
        z[mt][1] = __ldg(hz[mt] + 8 * nb + 2 * qc + 1);
      }
#pragma unroll
      for (int kb = 0; kb < KB2; ++kb) {
        const double b = w2[(kb * NB2 + nb) * 32 + lane];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) dmma(z[mt][0], z[mt][1], ct[(mt * KB2 + kb) * 32 + lane], b);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        double a3[4];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt) a3[mt] = c_to_a(fmax(z[mt][0], 0.0), fmax(z[mt][1], 0.0), h, lane);
#pragma unroll
        for (int ot = 0; ot < NB3; ++ot) {
          const double b = w3[((2 * nb + h) * NB3 + ot) * 32 + lane];
#pragma unroll
          for (int mt = 0; mt < 4; ++mt) dmma(zo[mt][ot][0], zo[mt][ot][1], a3[mt], b);
        }
      }
    }
    __syncwarp();
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int ot = 0; ot < NB3; ++ot) {
        ct[(8 * mt + qr) * kCS + 8 * ot + 2 * qc] = zo[mt][ot][0];
        ct[(8 * mt + qr) * kCS + 8 * ot + 2 * qc + 1] = zo[mt][ot][1];
      }
    __syncwarp();
    if (lane < cnt) {
      const int64_t row = q[(h0 + lane) & (kRingM - 1)];
      double* c = ct + lane * kCS;
      // basis first: a coefficient whose g is exactly 0 adds fma(0, c, dot)
      // = dot, so its softplus is skipped (rows have ~12 of 30 non-zero; the
      // lane walks its own mask, two evaluations per step).  Bit-identical
      // to evaluating all thirty (softplus is finite for finite z).
      double g[GS_NUM_COEFFS];
      const double hb = basis_g(feats + row * GS_NUM_FEATURES, g);
      unsigned msk = 0;
#pragma unroll
      for (int i = 0; i < GS_NUM_COEFFS; ++i) msk |= (unsigned)(g[i] != 0.0) << i;
#pragma unroll 1
      while (msk) {
        const int i1 = __ffs(msk) - 1;
        msk &= msk - 1;
        const int i2 = msk ? __ffs(msk) - 1 : i1;
        msk &= msk - 1;
        const double x = softplus_bf(c[i1]), y = softplus_bf(c[i2]);
        c[i1] = x + kEps;
        c[i2] = y + kEps;
      }
      double dot = 0.0;
#pragma unroll
      for (int i = 0; i < GS_NUM_COEFFS; ++i)
        if (g[i] != 0.0) dot = fma(g[i], c[i], dot);
      row_cost[row] = __dadd_rn(dot, hb);
    }
    __syncwarp();
  };

  // queue fill: each lane takes 4 consecutive rows per group (one 16-byte
  // row_src load when aligned; n_rows once per candidate it touches), three
  // 128-row groups per step
  constexpr int kV = 3;
  static_assert(kRingM >= 31 + 128 * kV, "");
  const bool vec = ((uintptr_t)row_src & 15) == 0;
  auto claim = [&]() -> int64_t {
    unsigned v = 0;
    if (lane == 0) v = atomicAdd(work, 1u);
    return (int64_t)__shfl_sync(0xffffffffu, v, 0);
  };
  int64_t sp = claim(), s0 = sp * kSpan;
  unsigned head = 0, tail = 0;
  for (;;) {
    while (tail - head < 32 && s0 < total_rows) {
      const int64_t end = sp * kSpan + kSpan < total_rows ? sp * kSpan + kSpan : total_rows;
      unsigned tm = 0;   // bit 4u + e: row s0 + 128u + 4 lane + e is computed
#pragma unroll
      for (int u = 0; u < kV; ++u) {
        const int64_t r0 = s0 + 128 * u + 4 * lane;
        if (r0 < end) {
          int v[4];
          if (vec && r0 + 3 < end) {
            const int4 w = __ldg(reinterpret_cast<const int4*>(row_src + r0));
            v[0] = w.x; v[1] = w.y; v[2] = w.z; v[3] = w.w;
          } else {
#pragma unroll
            for (int e = 0; e < 4; ++e) v[e] = r0 + e < end ? __ldg(row_src + r0 + e) : -1;
          }
          const uint32_t c0 = (uint32_t)r0 / (uint32_t)R;   // rows < 2^32 on this path
          int r = (int)((uint32_t)r0 - c0 * (uint32_t)R);
          uint32_t c = c0;
          int nr = __ldg(n_rows + c0);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            if (e > 0 && ++r >= R) { r = 0; ++c; nr = r0 + e < end ? __ldg(n_rows + c) : 0; }
            tm |= (unsigned)(r < nr && v[e] == (int32_t)c) << (4 * u + e);
          }
        }
      }
#pragma unroll 1
      for (int u = 0; u < kV; ++u) {
        const unsigned mine = (tm >> (4 * u)) & 15u;
        const int cntl = __popc(mine);
        int incl = cntl;   // inclusive prefix of the lanes' counts: rows stay in order
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int y = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += y;
        }
        unsigned pos = tail + (unsigned)(incl - cntl);
        for (int e = 0; e < 4; ++e)
          if ((mine >> e) & 1u) q[(pos++) & (kRingM - 1)] = (uint32_t)(s0 + 128 * u + 4 * lane + e);
        tail += (unsigned)__shfl_sync(0xffffffffu, incl, 31);
      }
      s0 += 128 * kV;
      if (s0 >= end) { sp = claim(); s0 = sp * kSpan; }
    }
    if (tail == head) break;
    __syncwarp();
    const int cnt = tail - head < 32 ? (int)(tail - head) : 32;
    run_warp(head, cnt);
    head += cnt;
  }
}

template <int E, int H>
int mma_smem_bytes() {
  return ((GS_NUM_FEATURES / 4) * (E / 8) * 32 + (E / 4) * (H / 8) * 32 + (H / 4) * 4 * 32 + E + 32 +
          kMmaWarps * 32 * kCS) * 8;
}

__global__ void __launch_bounds__(128) stage_sum_kernel(const int32_t* __restrict__ n_rows,
                                                        const int32_t* __restrict__ row_src,
                                                        const double* __restrict__ row_cost, int64_t n, int R,
                                                        int CB, double* __restrict__ total,
                                                        double* __restrict__ row_cost_out) {
  extern __shared__ __align__(16) double buf[];   // CB*R
  for (int64_t c0 = (int64_t)blockIdx.x * CB; c0 < n; c0 += (int64_t)gridDim.x * CB) {
    const int ncb = (int)((n - c0) < CB ? (n - c0) : CB);
    for (int idx = threadIdx.x; idx < ncb * R; idx += blockDim.x) {
      const int cl = idx / R, r = idx % R;
      const int64_t c = c0 + cl;
      if (r >= n_rows[c]) continue;
      const int64_t row = c * R + r;
      const int64_t src = (int64_t)row_src[row] * R + r;
      const double v = row_cost[src];
      buf[idx] = v;
      if (row_cost_out && src != row) row_cost_out[row] = v;
    }
    __syncthreads();
    if (threadIdx.x < ncb) {
      const int64_t c = c0 + threadIdx.x;
      double t = 0.0;
      const int nr = n_rows[c];
      for (int r = 0; r < nr; ++r) t = __dadd_rn(t, buf[threadIdx.x * R + r]);
      total[c] = t;
    }
    __syncthreads();
  }
}

int launch_hoist(const NetDev& net, const double* algo, int n_stages, cudaStream_t st) {
  if (n_stages == 0) return 0;
  hoist_kernel<<<n_stages, 64, 0, st>>>(net, algo, n_stages); g_launch_count++;
  return 0;
}

int cost_smem_bytes(int E, int H, int CB, int R) {
  return (GS_NUM_FEATURES * E + E * H + H * GS_NUM_COEFFS + E + GS_NUM_COEFFS + CB * R + GS_NUM_COEFFS * 128) * 8;
}

int launch_cost(const NetDev& net, const int32_t* stage_of_func, const double* feats, const int32_t* row_key,
                const int32_t* n_rows, const int32_t* row_src, int64_t n, int R, double* total, double* row_cost,
                double* basis_gh, unsigned* work, int num_sms, cudaStream_t st, bool rows_out) {
  if (n == 0) return 0;
  if (row_src && row_cost && !basis_gh) {
    if (n * (int64_t)R / 128 >= 0xFFFFFFFFll) return -1;
    cudaMemsetAsync(work, 0, sizeof(unsigned), st);
    if (net.E > 64) return -1;
    const int smA = (GS_NUM_FEATURES * net.E + net.E * net.H + net.H * GS_NUM_COEFFS + net.E + GS_NUM_COEFFS +
                     GS_NUM_COEFFS * kRowsWarps * 32) * 8;
    const int64_t slabs = (n * (int64_t)R + kRowsWarps * 32 - 1) / (kRowsWarps * 32);
    const int gridA = (int)(slabs < (int64_t)num_sms ? slabs : (int64_t)num_sms);
    // spans of 2,048 rows, down to 128 when the batch has fewer than four
    // spans per warp (a 64K-candidate C2 step left most warps idle)
    const int64_t rows_total = n * (int64_t)R, warps = (int64_t)gridA * kRowsWarps;
    int64_t span = 2048;
    while (span > 128 && rows_total / span < 4 * warps) span >>= 1;
    static const bool scalar_only = getenv("GS_K2_SCALAR") != nullptr;   // A/B switch for the DMMA path
    if (net.E == 32 && net.H == 64 && !scalar_only && rows_total < 0xFFFFFFFFll) {
      const int smM = mma_smem_bytes<32, 64>();
      const int64_t wM = (int64_t)gridA * kMmaWarps;
      int64_t spanM = 2048;
      while (spanM > 128 && rows_total / spanM < 4 * wM) spanM >>= 1;
      cudaFuncSetAttribute(cost_rows_mma_kernel<32, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smM);
      cost_rows_mma_kernel<32, 64><<<gridA, kMmaWarps * 32, smM, st>>>(net, stage_of_func, feats, row_key, n_rows,
                                                                      row_src, n, R, row_cost, work, spanM);
    } else if (net.E <= 32) {
      cudaFuncSetAttribute(cost_rows_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smA);
      cost_rows_kernel<32><<<gridA, kRowsWarps * 32, smA, st>>>(net, stage_of_func, feats, row_key, n_rows, row_src,
                                                                n, R, row_cost, work, span);
    } else {
      cudaFuncSetAttribute(cost_rows_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smA);
      cost_rows_kernel<64><<<gridA, kRowsWarps * 32, smA, st>>>(net, stage_of_func, feats, row_key, n_rows, row_src,
                                                                n, R, row_cost, work, span);
    }
    g_launch_count++;
    int CB = 1024 / (R > 0 ? R : 1);
    if (CB < 1) CB = 1;
    if (CB > 128) CB = 128;
    const int smB = CB * R * 8;
    const int64_t blocks = (n + CB - 1) / CB;
    const int gridB = (int)(blocks < (int64_t)num_sms * 16 ? blocks : (int64_t)num_sms * 16);
    cudaFuncSetAttribute(stage_sum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smB);
    stage_sum_kernel<<<gridB, 128, smB, st>>>(n_rows, row_src, row_cost, n, R, CB, total,
                                              rows_out ? row_cost : nullptr);
    g_launch_count++;
    return 0;
  }
  int CB = 512 / (R > 0 ? R : 1);
  if (CB < 1) CB = 1;
  if (CB > 128) CB = 128;
  const int smem = cost_smem_bytes(net.E, net.H, CB, R);
  int64_t blocks = (n + CB - 1) / CB;
  int64_t cap = (int64_t)num_sms * 8;
  int grid = (int)(blocks < cap ? blocks : cap);
  if (net.E <= 32) {
    cudaFuncSetAttribute(cost_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cost_kernel<32><<<grid, 128, smem, st>>>(net, stage_of_func, feats, row_key, n_rows, n, R, CB, total,
                                             row_cost, basis_gh); g_launch_count++;
  } else if (net.E <= 64) {
    cudaFuncSetAttribute(cost_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cost_kernel<64><<<grid, 128, smem, st>>>(net, stage_of_func, feats, row_key, n_rows, n, R, CB, total,
                                             row_cost, basis_gh); g_launch_count++;
  } else {
    return -1;
  }
  return 0;
}

}  // namespace gs
