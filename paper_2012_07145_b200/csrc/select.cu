// K4 — structural-hash bucketing + hierarchical-sampling representatives
//      (reference sampling.py:45-59, search.py:127-165)
// K5 — beam cut: pass penalty, optional Gumbel(T) noise, stable top-k by a
//      hand-written single-CTA radix select + bitonic sort, and the
//      bottom-half flags for the bad-hash memo (search.py:76-87, 168-201).
//
// Bucketing: a stable LSD radix sort of (hash, candidate index) puts every
// bucket contiguous, buckets in ascending hash order and members in
// insertion order — exactly `for h in sorted(buckets)` over dict buckets.
// Each bucket then re-creates NumPy's stream default_rng((phase_seed, h)):
// SeedSequence hash-mix -> PCG64 (128-bit LCG, XSL-RR output) ->
// Fisher-Yates `permutation(B)` with masked-rejection bounded draws on
// buffered 32-bit halves, and walks it until quota = max(1, floor(log2 B))
// valid members are taken (one thread per bucket; the draws are sequential
// by construction).
#include "gs_internal.cuh"
#include <cub/cub.cuh>

namespace gs {

typedef unsigned __int128 u128;

// ---------------------------------------------------------------- RNG ----
struct Pcg64 {
  u128 state, inc;
  uint32_t buf;
  bool has_buf;

  __device__ static uint32_t hashmix(uint32_t v, uint32_t& hc) {
    v ^= hc;
    hc *= 0x931E8875u;
    v *= hc;
    return v ^ (v >> 16);
  }
  __device__ static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = 0xCA01F9DDu * x - 0x4973F715u * y;
    return r ^ (r >> 16);
  }
  // SeedSequence(entropy = uint32 words).generate_state(4, uint64)
  __device__ void seed(const uint32_t* ent, int n_ent) {
    uint32_t pool[4];
    uint32_t hc = 0x43B0D7E5u;
    for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n_ent ? ent[i] : 0u, hc);
    for (int s = 0; s < 4; ++s)
      for (int d = 0; d < 4; ++d)
        if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
    for (int s = 4; s < n_ent; ++s)
      for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
    uint32_t o[8];
    uint32_t hb = 0x8B51F9DDu;
    for (int i = 0; i < 8; ++i) {
      uint32_t v = pool[i & 3];
      v ^= hb;
      hb *= 0x58F38DEDu;
      v *= hb;
      o[i] = v ^ (v >> 16);
    }
    uint64_t w[4];
    for (int i = 0; i < 4; ++i) w[i] = (uint64_t)o[2 * i] | ((uint64_t)o[2 * i + 1] << 32);
    const u128 sd = ((u128)w[0] << 64) | w[1];
    const u128 sq = ((u128)w[2] << 64) | w[3];
    inc = (sq << 1) | 1;
    state = 0;
    step();
    state += sd;
    step();
    has_buf = false;
    buf = 0;
  }
  __device__ void step() {
    const u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
    state = state * mult + inc;
  }
  __device__ uint64_t next64() {
    step();
    uint64_t x = (uint64_t)(state >> 64) ^ (uint64_t)state;
    unsigned rot = (unsigned)(state >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  __device__ uint32_t next32() {
    if (has_buf) { has_buf = false; return buf; }
    uint64_t v = next64();
    has_buf = true;
    buf = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  __device__ uint64_t interval(uint64_t mx) {   // numpy random_interval
    if (mx == 0) return 0;
    uint64_t mask = mx;
    mask |= mask >> 1; mask |= mask >> 2; mask |= mask >> 4;
    mask |= mask >> 8; mask |= mask >> 16; mask |= mask >> 32;
    if (mx <= 0xFFFFFFFFull) {
      uint64_t v;
      while ((v = (next32() & mask)) > mx) {}
      return v;
    }
    uint64_t v;
    while ((v = (next64() & mask)) > mx) {}
    return v;
  }
  __device__ double next_double() { return (double)(next64() >> 11) * (1.0 / 9007199254740992.0); }
};

__device__ int words_of(uint64_t x, uint32_t* out) {
  if (x == 0) { out[0] = 0; return 1; }
  int n = 0;
  while (x) { out[n++] = (uint32_t)x; x >>= 32; }
  return n;
}

__device__ void seed_pair(Pcg64& g, uint64_t a, uint64_t b) {
  uint32_t ent[4];
  int n = words_of(a, ent);
  n += words_of(b, ent + n);
  g.seed(ent, n);
}

// ------------------------------------------------------------ K4 kernels ---
__global__ void iota_kernel(uint32_t* v, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

__global__ void head_kernel(const uint64_t* __restrict__ k, int64_t n, uint32_t* __restrict__ head) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) head[i] = (i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}

__global__ void starts_kernel(const uint32_t* __restrict__ head, const uint32_t* __restrict__ bid, int64_t n,
                              uint32_t* __restrict__ starts, uint32_t* __restrict__ nb) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && head[i]) starts[bid[i]] = (uint32_t)i;
  if (i == n - 1) { uint32_t b = bid[i] + head[i]; *nb = b; starts[b] = (uint32_t)n; }
}

__global__ void quota_kernel(const uint32_t* __restrict__ starts, const uint32_t* __restrict__ nb, int64_t n,
                             uint32_t* __restrict__ quota) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  if (b >= *nb) { quota[b] = 0; return; }
  uint32_t B = starts[b + 1] - starts[b];
  int q = 63 - __clzll((unsigned long long)B);   // floor(log2 B)
  quota[b] = q < 1 ? 1u : (uint32_t)q;
}

__global__ void walk_kernel(const uint64_t* __restrict__ keys, const uint32_t* __restrict__ members,
                            const uint32_t* __restrict__ starts, const uint32_t* __restrict__ nb,
                            const uint32_t* __restrict__ qoff, const uint32_t* __restrict__ quota,
                            const uint8_t* __restrict__ verdict, uint64_t phase_seed,
                            uint32_t* __restrict__ perm, int64_t* __restrict__ slot,
                            uint32_t* __restrict__ taken, int64_t* __restrict__ rej,
                            uint32_t* __restrict__ rejn) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= *nb) return;
  const uint32_t s0 = starts[b], B = starts[b + 1] - s0;
  uint32_t* p = perm + s0;
  for (uint32_t i = 0; i < B; ++i) p[i] = i;
  Pcg64 g;
  seed_pair(g, phase_seed, keys[s0]);
  for (uint32_t i = B - 1; i >= 1; --i) {   // numpy Generator.shuffle (Fisher-Yates)
    uint32_t j = (uint32_t)g.interval(i);
    uint32_t t = p[i]; p[i] = p[j]; p[j] = t;
  }
  const uint32_t q = quota[b];
  uint32_t t = 0, r = 0;
  for (uint32_t i = 0; i < B; ++i) {
    const uint32_t m = members[s0 + p[i]];
    if (verdict[m] == 0) {
      slot[qoff[b] + t] = m;
      if (++t == q) break;
    } else {
      rej[s0 + r] = m;
      ++r;
    }
  }
  taken[b] = t;
  rejn[b] = r;
}

__global__ void gather_kernel(const uint32_t* __restrict__ nb, int64_t n, const uint32_t* __restrict__ qoff,
                              const uint32_t* __restrict__ taken, const uint32_t* __restrict__ toff,
                              const int64_t* __restrict__ slot, int64_t* __restrict__ rep_idx,
                              const uint32_t* __restrict__ starts, const uint32_t* __restrict__ rejn,
                              const uint32_t* __restrict__ roff, const int64_t* __restrict__ rej,
                              int64_t* __restrict__ rej_idx, int64_t* __restrict__ n_reps,
                              int64_t* __restrict__ n_rejects) {
  int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t NB = *nb;
  if (b < NB) {
    for (uint32_t t = 0; t < taken[b]; ++t) rep_idx[toff[b] + t] = slot[qoff[b] + t];
    if (rej_idx)
      for (uint32_t t = 0; t < rejn[b]; ++t) rej_idx[roff[b] + t] = rej[starts[b] + t];
  }
  if (b == 0) {
    *n_reps = (int64_t)toff[NB - 1] + taken[NB - 1];
    *n_rejects = (int64_t)roff[NB - 1] + rejn[NB - 1];
  }
}

// workspace carve-up for K4
struct SelWs {
  uint64_t* keys_out; uint32_t* vals_in; uint32_t* vals_out; uint32_t* head; uint32_t* bid;
  uint32_t* starts; uint32_t* nb; uint32_t* quota; uint32_t* qoff; uint32_t* taken; uint32_t* toff;
  uint32_t* rejn; uint32_t* roff; uint32_t* perm; int64_t* slot; int64_t* rej; void* cub; size_t cub_bytes;
};

static size_t align256(size_t x) { return (x + 255) & ~size_t(255); }

static size_t cub_temp_bytes(int64_t n) {
  size_t a = 0, b = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)(n + 1));
  return a > b ? a : b;
}

static size_t carve(SelWs& w, void* base, int64_t n) {
  size_t o = 0;
  auto take = [&](size_t bytes) { size_t r = o; o += align256(bytes); return r; };
  size_t o_keys = take(8 * n), o_vi = take(4 * n), o_vo = take(4 * n), o_head = take(4 * n),
         o_bid = take(4 * n), o_starts = take(4 * (n + 1)), o_nb = take(4), o_quota = take(4 * n),
         o_qoff = take(4 * n), o_taken = take(4 * n), o_toff = take(4 * n), o_rejn = take(4 * n),
         o_roff = take(4 * n), o_perm = take(4 * n), o_slot = take(8 * n), o_rej = take(8 * n);
  size_t cb = cub_temp_bytes(n);
  size_t o_cub = take(cb);
  if (base) {
    char* p = (char*)base;
    w.keys_out = (uint64_t*)(p + o_keys); w.vals_in = (uint32_t*)(p + o_vi); w.vals_out = (uint32_t*)(p + o_vo);
    w.head = (uint32_t*)(p + o_head); w.bid = (uint32_t*)(p + o_bid); w.starts = (uint32_t*)(p + o_starts);
    w.nb = (uint32_t*)(p + o_nb); w.quota = (uint32_t*)(p + o_quota); w.qoff = (uint32_t*)(p + o_qoff);
    w.taken = (uint32_t*)(p + o_taken); w.toff = (uint32_t*)(p + o_toff); w.rejn = (uint32_t*)(p + o_rejn);
    w.roff = (uint32_t*)(p + o_roff); w.perm = (uint32_t*)(p + o_perm); w.slot = (int64_t*)(p + o_slot);
    w.rej = (int64_t*)(p + o_rej); w.cub = p + o_cub; w.cub_bytes = cb;
  }
  return o;
}

int64_t select_workspace_bytes(int64_t n) {
  SelWs w;
  return (int64_t)carve(w, nullptr, n < 1 ? 1 : n);
}

int select_reps(const uint64_t* hashes, const uint8_t* verdict, int64_t n, uint64_t phase_seed, void* ws,
                int64_t ws_bytes, int64_t* rep_idx, int64_t* n_reps, int64_t* n_rejects, int64_t* rej_idx,
                cudaStream_t st) {
  if (n <= 0) {
    cudaMemsetAsync(n_reps, 0, 8, st);
    cudaMemsetAsync(n_rejects, 0, 8, st);
    return 0;
  }
  if (n >= (int64_t)0xFFFFFFFF) return -1;
  SelWs w;
  if ((int64_t)carve(w, ws, n) > ws_bytes) return -2;
  const int T = 256;
  const unsigned G = (unsigned)((n + T - 1) / T);
  cudaMemsetAsync(w.taken, 0, 4 * n, st);
  cudaMemsetAsync(w.rejn, 0, 4 * n, st);
  iota_kernel<<<G, T, 0, st>>>(w.vals_in, n); g_launch_count++;
  size_t cb = w.cub_bytes;
  cub::DeviceRadixSort::SortPairs(w.cub, cb, hashes, w.keys_out, w.vals_in, w.vals_out, (int)n, 0, 64, st);
  head_kernel<<<G, T, 0, st>>>(w.keys_out, n, w.head); g_launch_count++;
  cb = w.cub_bytes;
  cub::DeviceScan::ExclusiveSum(w.cub, cb, w.head, w.bid, (int)n, st);
  starts_kernel<<<G, T, 0, st>>>(w.head, w.bid, n, w.starts, w.nb); g_launch_count++;
  quota_kernel<<<G, T, 0, st>>>(w.starts, w.nb, n, w.quota); g_launch_count++;
  cb = w.cub_bytes;
  cub::DeviceScan::ExclusiveSum(w.cub, cb, w.quota, w.qoff, (int)n, st);
  walk_kernel<<<G, 64, 0, st>>>(w.keys_out, w.vals_out, w.starts, w.nb, w.qoff, w.quota, verdict, phase_seed,
                                w.perm, w.slot, w.taken, w.rej, w.rejn); g_launch_count++;
  // zero unused tails so the scans see only live buckets
  cb = w.cub_bytes;
  cub::DeviceScan::ExclusiveSum(w.cub, cb, w.taken, w.toff, (int)n, st);
  cb = w.cub_bytes;
  cub::DeviceScan::ExclusiveSum(w.cub, cb, w.rejn, w.roff, (int)n, st);
  gather_kernel<<<G, T, 0, st>>>(w.nb, n, w.qoff, w.taken, w.toff, w.slot, rep_idx, w.starts, w.rejn, w.roff,
                                 w.rej, rej_idx, n_reps, n_rejects); g_launch_count++;
  return 0;
}

// ------------------------------------------------------------ K5 kernels ---
__device__ __forceinline__ uint64_t sortable(double x) {
  if (x == 0.0) x = 0.0;   // -0.0 == 0.0 in the reference's sort
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}

__global__ void keys_kernel(const double* __restrict__ costs, const uint64_t* __restrict__ ph, int64_t n,
                            const uint64_t* __restrict__ flagged, int64_t nflag, double penalty,
                            uint64_t* __restrict__ key, uint64_t* __restrict__ ckey, double* __restrict__ kval) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double c = costs[i];
  bool f = false;
  if (nflag > 0) {
    int64_t lo = 0, hi = nflag;
    const uint64_t h = ph[i];
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (flagged[mid] < h) lo = mid + 1; else hi = mid; }
    f = lo < nflag && flagged[lo] == h;
  }
  double k = f ? c * penalty : c;   // apply_pass_penalty (search.py:76-87)
  kval[i] = k;
  key[i] = sortable(k);
  ckey[i] = sortable(c);
}

// Gumbel noise on log-cost (search.py:185-192): sequential draws, rep order
__global__ void gumbel_kernel(double* __restrict__ kval, uint64_t* __restrict__ key, int64_t n,
                              double temperature, uint64_t phase_seed) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  Pcg64 g;
  seed_pair(g, phase_seed, 0x657870ULL);
  for (int64_t i = 0; i < n; ++i) {
    double u;
    do { u = 1.0 - g.next_double(); } while (!(u < 1.0));
    const double gum = -log(-log(u));
    const double k = kval[i] > 1e-300 ? kval[i] : 1e-300;
    const double v = log(k) + gum * temperature;
    kval[i] = v;
    key[i] = sortable(v);
  }
}

// Single-CTA stable radix select: the element of stable rank `target` by
// (key, position); returns its key and how many keys are strictly smaller.
template <int NT>
__device__ void radix_select(const uint64_t* __restrict__ key, int64_t n, int64_t target, uint64_t& kstar,
                             int64_t& less) {
  __shared__ unsigned int hist[256];
  __shared__ uint64_t s_prefix;
  __shared__ int64_t s_rank;
  __shared__ int64_t s_less;
  if (threadIdx.x == 0) { s_prefix = 0; s_rank = target; s_less = 0; }
  __syncthreads();
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    const uint64_t pmask = pass == 0 ? 0ull : (~0ull << (64 - 8 * pass));
    for (int i = threadIdx.x; i < 256; i += NT) hist[i] = 0;
    __syncthreads();
    const uint64_t pre = s_prefix;
    for (int64_t i = threadIdx.x; i < n; i += NT) {
      const uint64_t k = key[i];
      if ((k & pmask) == pre) atomicAdd(&hist[(k >> shift) & 255], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t r = s_rank, acc = 0;
      int d = 0;
      for (; d < 256; ++d) {
        if (acc + hist[d] > r) break;
        acc += hist[d];
      }
      s_rank = r - acc;
      s_less += acc;
      s_prefix = pre | ((uint64_t)d << shift);
    }
    __syncthreads();
  }
  kstar = s_prefix;
  less = s_less;
}

// flags[i] = 1 iff element i is among the first `count` by (key, position)
template <int NT>
__device__ void stable_prefix_flags(const uint64_t* __restrict__ key, int64_t n, int64_t count,
                                    uint8_t* __restrict__ flags, bool invert) {
  uint64_t kstar;
  int64_t less;
  if (count <= 0) {
    for (int64_t i = threadIdx.x; i < n; i += NT) flags[i] = invert ? 1 : 0;
    return;
  }
  if (count >= n) {
    for (int64_t i = threadIdx.x; i < n; i += NT) flags[i] = invert ? 0 : 1;
    return;
  }
  radix_select<NT>(key, n, count - 1, kstar, less);
  const int64_t eq_take = count - less;   // equal keys admitted, in position order
  __shared__ int64_t base;
  __shared__ int wsum[NT / 32];
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < n; c0 += NT) {
    const int64_t i = c0 + threadIdx.x;
    const bool in = i < n;
    const uint64_t k = in ? key[i] : ~0ull;
    const bool eq = in && k == kstar;
    unsigned bal = __ballot_sync(0xffffffffu, eq);
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    const int64_t rank_eq = base + before + __popc(bal & ((1u << lane) - 1));
    if (in) {
      bool sel = k < kstar || (eq && rank_eq < eq_take);
      flags[i] = (uint8_t)(invert ? !sel : sel);
    }
    __syncthreads();
    if (threadIdx.x == 0) { int t = 0; for (int w = 0; w < NT / 32; ++w) t += wsum[w]; base += t; }
    __syncthreads();
  }
}

constexpr int kTopNT = 1024;
constexpr int kSortCap = 2048;

__global__ void __launch_bounds__(kTopNT) topk_kernel(const uint64_t* __restrict__ key, const uint64_t* __restrict__ ckey,
                                                     int64_t n, int64_t k, uint8_t* __restrict__ sel,
                                                     int64_t* __restrict__ out_pos, int64_t* __restrict__ n_out,
                                                     uint8_t* __restrict__ bottom) {
  stable_prefix_flags<kTopNT>(key, n, k, sel, false);
  __syncthreads();
  // gather the selected (<= k) in position order, then bitonic sort by (key, pos)
  __shared__ uint64_t sk[kSortCap];
  __shared__ int64_t sp[kSortCap];
  __shared__ int64_t cnt;
  __shared__ int wsum[kTopNT / 32];
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (int64_t c0 = 0; c0 < n; c0 += kTopNT) {
    const int64_t i = c0 + threadIdx.x;
    const bool s = i < n && sel[i];
    unsigned bal = __ballot_sync(0xffffffffu, s);
    int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wsum[warp] = __popc(bal);
    __syncthreads();
    int before = 0;
    for (int w = 0; w < warp; ++w) before += wsum[w];
    const int64_t pos = cnt + before + __popc(bal & ((1u << lane) - 1));
    if (s && pos < kSortCap) { sk[pos] = key[i]; sp[pos] = i; }
    __syncthreads();
    if (threadIdx.x == 0) { int t = 0; for (int w = 0; w < kTopNT / 32; ++w) t += wsum[w]; cnt += t; }
    __syncthreads();
  }
  const int m = (int)(cnt < kSortCap ? cnt : kSortCap);
  int P = 1;
  while (P < m) P <<= 1;
  for (int i = m + threadIdx.x; i < P; i += kTopNT) { sk[i] = ~0ull; sp[i] = INT64_MAX; }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += kTopNT) {
        int j = i ^ stride;
        if (j > i) {
          bool up = (i & size) == 0;
          bool gt = sk[i] > sk[j] || (sk[i] == sk[j] && sp[i] > sp[j]);
          if (gt == up) {
            uint64_t tk = sk[i]; sk[i] = sk[j]; sk[j] = tk;
            int64_t tp = sp[i]; sp[i] = sp[j]; sp[j] = tp;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < m; i += kTopNT) out_pos[i] = sp[i];
  if (threadIdx.x == 0) *n_out = m;
  __syncthreads();
  // bottom half by unpenalized cost (stable), only when n > 1 (search.py:196-200)
  if (bottom) {
    if (n > 1) stable_prefix_flags<kTopNT>(ckey, n, n / 2, bottom, true);
    else for (int64_t i = threadIdx.x; i < n; i += kTopNT) bottom[i] = 0;
  }
}

// k > kSortCap (e.g. sampling-free exhaustive searches): full stable sort
__global__ void bottom_from_sorted(const uint32_t* __restrict__ order, int64_t n, uint8_t* __restrict__ bottom) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) bottom[order[i]] = (n > 1 && i >= n / 2) ? 1 : 0;
}
__global__ void copy_pos(const uint32_t* __restrict__ order, int64_t k, int64_t* __restrict__ out,
                         int64_t* __restrict__ n_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = order[i];
  if (i == 0) *n_out = k;
}

// Tie band: after an exact sort by key, adjacent keys within `band`
// (relative) join one group; the final order is (group, position).  The
// reference orders exact ties by representative position (stable sort); its
// fp64 sums of permuted per-stage costs tie by rounding luck, which ours
// (ulp-different row costs) cannot reproduce bit for bit.
__global__ void band_flags(const uint64_t* __restrict__ skey, const double* __restrict__ kval,
                           const uint32_t* __restrict__ order, int64_t n, double band,
                           uint32_t* __restrict__ brk) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (i == 0) { brk[i] = 0; return; }
  const double a = kval[order[i - 1]], b = kval[order[i]];
  const double m = fmax(fabs(a), fabs(b));
  brk[i] = (b - a) > band * m ? 1u : 0u;
  (void)skey;
}
__global__ void band_keys(const uint32_t* __restrict__ gid, const uint32_t* __restrict__ order, int64_t n,
                          uint64_t* __restrict__ key2) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) key2[i] = ((uint64_t)gid[i] << 32) | order[i];
}

static size_t sort_temp_bytes(int64_t n) {
  size_t a = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, a, (const uint64_t*)nullptr, (uint64_t*)nullptr,
                                  (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  return a;
}

int64_t topk_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  size_t scan = 0;
  cub::DeviceScan::InclusiveSum(nullptr, scan, (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n);
  size_t sk = 0;
  cub::DeviceRadixSort::SortKeys(nullptr, sk, (const uint64_t*)nullptr, (uint64_t*)nullptr, (int)n);
  size_t tmp = std::max(std::max(scan, sk), sort_temp_bytes(n));
  return (int64_t)(align256(8 * n) * 6 + align256(n) + align256(4 * n) * 4 + align256(tmp));
}

struct TopkWs {
  uint64_t *key, *ckey, *kout, *key2, *key2o;
  double* kval;
  uint8_t* sel;
  uint32_t *vin, *vout, *brk, *gid;
  void* tmp;
  size_t tmp_bytes;
};

// order[i] = position of the i-th element by (band group of key, position)
static void band_order(TopkWs& w, const uint64_t* key, const double* val, int64_t n, double band,
                       cudaStream_t st) {
  const unsigned G = (unsigned)((n + 255) / 256);
  iota_kernel<<<G, 256, 0, st>>>(w.vin, n); g_launch_count++;
  size_t tb = w.tmp_bytes;
  cub::DeviceRadixSort::SortPairs(w.tmp, tb, key, w.kout, w.vin, w.vout, (int)n, 0, 64, st);
  band_flags<<<G, 256, 0, st>>>(w.kout, val, w.vout, n, band, w.brk); g_launch_count++;
  tb = w.tmp_bytes;
  cub::DeviceScan::InclusiveSum(w.tmp, tb, w.brk, w.gid, (int)n, st);
  band_keys<<<G, 256, 0, st>>>(w.gid, w.vout, n, w.key2); g_launch_count++;
  tb = w.tmp_bytes;
  cub::DeviceRadixSort::SortKeys(w.tmp, tb, w.key2, w.key2o, (int)n, 0, 64, st);
}

__global__ void pos_from_key2(const uint64_t* __restrict__ key2o, int64_t k, int64_t* __restrict__ out,
                              int64_t* __restrict__ n_out) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k) out[i] = (int64_t)(key2o[i] & 0xFFFFFFFFull);
  if (i == 0) *n_out = k;
}
__global__ void bottom_from_key2(const uint64_t* __restrict__ key2o, int64_t n, uint8_t* __restrict__ bottom) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) bottom[key2o[i] & 0xFFFFFFFFull] = (n > 1 && i >= n / 2) ? 1 : 0;
}

int beam_topk(const double* costs, const uint64_t* ph, int64_t n, const uint64_t* flagged, int64_t nflag,
              double penalty, double temperature, uint64_t phase_seed, int64_t k, double band, void* ws,
              int64_t ws_bytes, int64_t* out_pos, int64_t* n_out, uint8_t* bottom, cudaStream_t st) {
  if (n <= 0) { cudaMemsetAsync(n_out, 0, 8, st); return 0; }
  if (topk_workspace_bytes(n) > ws_bytes) return -2;
  if (n >= (int64_t)0xFFFFFFFF) return -3;
  if (k > n) k = n;
  char* p = (char*)ws;
  TopkWs w;
  w.key = (uint64_t*)p; p += align256(8 * n);
  w.ckey = (uint64_t*)p; p += align256(8 * n);
  w.kval = (double*)p; p += align256(8 * n);
  w.kout = (uint64_t*)p; p += align256(8 * n);
  w.key2 = (uint64_t*)p; p += align256(8 * n);
  w.key2o = (uint64_t*)p; p += align256(8 * n);
  w.sel = (uint8_t*)p; p += align256(n);
  w.vin = (uint32_t*)p; p += align256(4 * n);
  w.vout = (uint32_t*)p; p += align256(4 * n);
  w.brk = (uint32_t*)p; p += align256(4 * n);
  w.gid = (uint32_t*)p; p += align256(4 * n);
  w.tmp = p;
  w.tmp_bytes = (size_t)(ws_bytes - (int64_t)(p - (char*)ws));
  const unsigned G = (unsigned)((n + 255) / 256);
  keys_kernel<<<G, 256, 0, st>>>(costs, ph, n, flagged, nflag, penalty, w.key, w.ckey, w.kval); g_launch_count++;
  if (temperature > 0) { gumbel_kernel<<<1, 32, 0, st>>>(w.kval, w.key, n, temperature, phase_seed); g_launch_count++; }
  if (band > 0) {
    band_order(w, w.key, w.kval, n, band, st);
    pos_from_key2<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(w.key2o, k, out_pos, n_out); g_launch_count++;
    if (bottom) {
      band_order(w, w.ckey, costs, n, band, st);
      bottom_from_key2<<<G, 256, 0, st>>>(w.key2o, n, bottom); g_launch_count++;
    }
    return 0;
  }
  if (k <= kSortCap) {   // exact keys: hand-written single-CTA radix select + bitonic sort
    topk_kernel<<<1, kTopNT, 0, st>>>(w.key, w.ckey, n, k, w.sel, out_pos, n_out, bottom); g_launch_count++;
    return 0;
  }
  iota_kernel<<<G, 256, 0, st>>>(w.vin, n); g_launch_count++;
  size_t tb = w.tmp_bytes;
  cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.key, w.kout, w.vin, w.vout, (int)n, 0, 64, st);
  copy_pos<<<(unsigned)((k + 255) / 256), 256, 0, st>>>(w.vout, k, out_pos, n_out); g_launch_count++;
  if (bottom) {
    tb = w.tmp_bytes;
    cub::DeviceRadixSort::SortPairs(w.tmp, tb, w.ckey, w.kout, w.vin, w.vout, (int)n, 0, 64, st);
    bottom_from_sorted<<<G, 256, 0, st>>>(w.vout, n, bottom); g_launch_count++;
  }
  return 0;
}

}  // namespace gs
