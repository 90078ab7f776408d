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
#include "scan.cuh"
#include "rng.cuh"
#include <algorithm>

namespace gs {

// PCG64 jump-ahead: advance the LCG by `delta` steps in O(log delta)
// (the classic "LCG skip" of Brown; lets every thread start at its own draw).
__device__ void pcg_advance(Pcg64& g, uint64_t delta) {
  u128 mult = ((u128)0x2360ED051FC65DA4ULL << 64) | 0x4385DF649FCCF645ULL;
  u128 plus = g.inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1) { acc_mult *= mult; acc_plus = acc_plus * mult + plus; }
    plus = (mult + 1) * plus;
    mult *= mult;
    delta >>= 1;
  }
  g.state = acc_mult * g.state + acc_plus;
}

// ------------------------------------------------------- radix sort ------
// Stable LSD radix sort of (u64 key, u32 value) pairs, 8 passes of 8 bits.
// Per pass: a per-tile digit histogram (digit-major, so one exclusive scan
// gives every (digit, tile) its scatter base), the scan, and a stable
// scatter that ranks equal digits inside a 1024-element round with
// __match_any_sync and a per-warp count table.
constexpr int kRsNT = 1024;
constexpr int kRsIPT = 4;
constexpr int kRsTile = kRsNT * kRsIPT;

__global__ void __launch_bounds__(kRsNT) rs_hist(const uint64_t* __restrict__ key, int64_t nmax,
                                                 const uint32_t* __restrict__ dcount, int shift,
                                                 uint32_t* __restrict__ hist, int ntiles) {
  __shared__ uint32_t h[256];
  for (int d = threadIdx.x; d < 256; d += kRsNT) h[d] = 0;
  __syncthreads();
  const int64_t n = count_of(nmax, dcount);
  const int64_t base = (int64_t)blockIdx.x * kRsTile;
  for (int j = 0; j < kRsIPT; ++j) {
    const int64_t i = base + j * kRsNT + threadIdx.x;
    if (i < n) atomicAdd(&h[(key[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  for (int d = threadIdx.x; d < 256; d += kRsNT) hist[(int64_t)d * ntiles + blockIdx.x] = h[d];
}

__global__ void __launch_bounds__(kRsNT) rs_scatter(const uint64_t* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                    uint64_t* __restrict__ kout, uint32_t* __restrict__ vout,
                                                    int64_t nmax, const uint32_t* __restrict__ dcount, int shift,
                                                    const uint32_t* __restrict__ hist, int ntiles) {
  __shared__ uint32_t cnt[32][256];
  __shared__ uint32_t base[256];
  __shared__ uint32_t rtot[256];
  const int64_t n = count_of(nmax, dcount);
  const int64_t t0 = (int64_t)blockIdx.x * kRsTile;
  if (t0 >= n) return;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < 256; d += kRsNT) base[d] = hist[(int64_t)d * ntiles + blockIdx.x];
  for (int round = 0; round < kRsIPT; ++round) {
    for (int x = threadIdx.x; x < 32 * 256; x += kRsNT) (&cnt[0][0])[x] = 0;
    __syncthreads();
    const int64_t i = t0 + (int64_t)round * kRsNT + threadIdx.x;
    const bool in = i < n;
    const uint64_t k = in ? kin[i] : 0ull;
    const uint32_t v = in ? vin[i] : 0u;
    const uint32_t d = in ? (uint32_t)((k >> shift) & 255) : 256u;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    if (in && lane == __ffs(peers) - 1) cnt[warp][d] = __popc(peers);
    __syncthreads();
    if (threadIdx.x < 256) {
      uint32_t off = 0;
      for (int w = 0; w < 32; ++w) {
        const uint32_t c = cnt[w][threadIdx.x];
        cnt[w][threadIdx.x] = off;
        off += c;
      }
      rtot[threadIdx.x] = off;
    }
    __syncthreads();
    if (in) {
      const uint32_t dst = base[d] + cnt[warp][d] + __popc(peers & ((1u << lane) - 1u));
      kout[dst] = k;
      vout[dst] = v;
    }
    __syncthreads();
    if (threadIdx.x < 256) base[threadIdx.x] += rtot[threadIdx.x];
    __syncthreads();
  }
}

static int64_t rs_tiles_of(int64_t n) { return n < 1 ? 1 : (n + kRsTile - 1) / kRsTile; }
static size_t rs_hist_bytes(int64_t n) { return align256(4 * 256 * rs_tiles_of(n)); }
static size_t rs_sums_bytes(int64_t n) { return align256(4 * (scan_tiles_of(256 * rs_tiles_of(n)) + 1)); }

// Sorted pairs end up back in (k0, v0).
static void radix_sort_pairs(uint64_t* k0, uint32_t* v0, uint64_t* k1, uint32_t* v1, int64_t nmax,
                             const uint32_t* dcount, uint32_t* hist, uint32_t* sums, cudaStream_t st) {
  const int nt = (int)rs_tiles_of(nmax);
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 8 * pass;
    rs_hist<<<nt, kRsNT, 0, st>>>(k0, nmax, dcount, shift, hist, nt); g_launch_count++;
    scan_u32(hist, hist, (int64_t)256 * nt, nullptr, false, sums, nullptr, st);
    rs_scatter<<<nt, kRsNT, 0, st>>>(k0, v0, k1, v1, nmax, dcount, shift, hist, nt); g_launch_count++;
    uint64_t* tk = k0; k0 = k1; k1 = tk;
    uint32_t* tv = v0; v0 = v1; v1 = tv;
  }
}

// ------------------------------------------------------------ K4 kernels ---
// Buckets come from runs: a run is a stretch of consecutive candidates with
// one hash (a beam step's siblings), so only run heads are sorted.  The
// stable sort of (hash, run) puts every bucket's runs together in insertion
// order — `for h in sorted(buckets)` over the reference's dict buckets.
__device__ __forceinline__ uint32_t run_head(const uint64_t* __restrict__ h, int64_t i) {
  return (i == 0 || h[i] != h[i - 1]) ? 1u : 0u;
}

__global__ void k4_heads(const uint64_t* __restrict__ h, int64_t n, uint32_t* __restrict__ head) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) head[i] = run_head(h, i);
}

__global__ void k4_runs(const uint64_t* __restrict__ h, int64_t n, const uint32_t* __restrict__ runid,
                        uint64_t* __restrict__ rkey, uint32_t* __restrict__ rval, uint32_t* __restrict__ rstart) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t hd = run_head(h, i);
  if (hd) {
    const uint32_t r = runid[i];
    rkey[r] = h[i];
    rval[r] = r;
    rstart[r] = (uint32_t)i;
  }
  if (i == n - 1) rstart[runid[i] + hd] = (uint32_t)n;
}

__global__ void k4_sorted(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ sval,
                          const uint32_t* __restrict__ rstart, const uint32_t* __restrict__ m_dev, int64_t nmax,
                          uint32_t* __restrict__ len, uint32_t* __restrict__ bhead) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= (int64_t)*m_dev) return;
  const uint32_t r = sval[j];
  len[j] = rstart[r + 1] - rstart[r];
  bhead[j] = (j == 0 || skey[j] != skey[j - 1]) ? 1u : 0u;
}

__global__ void k4_buckets(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ bid,
                           const uint32_t* __restrict__ m_dev, int64_t n, uint32_t* __restrict__ bstart,
                           uint32_t* __restrict__ cum, uint32_t* __restrict__ nb_dev) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t m = *m_dev;
  if (j >= m) return;
  const bool hd = j == 0 || skey[j] != skey[j - 1];
  if (hd) bstart[bid[j]] = (uint32_t)j;
  if (j == m - 1) {
    const uint32_t nb = bid[j] + (hd ? 1u : 0u);
    bstart[nb] = (uint32_t)m;
    cum[m] = (uint32_t)n;
    *nb_dev = nb;
  }
}

constexpr uint32_t kBigBucket = 1024;          // buckets walked by a CTA (k4_walk_big)
constexpr int kWalkSmemEntries = 50 * 1024;   // 200 KB of u32: a big bucket's permutation in shared memory

// quota = max(1, floor(log2 B)); buckets of >= kBigBucket members are also
// listed for k4_walk_big (in any order: buckets are independent)
__global__ void k4_quota(const uint32_t* __restrict__ bstart, const uint32_t* __restrict__ cum,
                         const uint32_t* __restrict__ nb_dev, uint32_t* __restrict__ quota,
                         uint32_t* __restrict__ big, uint32_t* __restrict__ big_cnt) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= (int64_t)*nb_dev) return;
  const uint32_t B = cum[bstart[b + 1]] - cum[bstart[b]];
  const int q = 63 - __clzll((unsigned long long)B);   // floor(log2 B)
  quota[b] = q < 1 ? 1u : (uint32_t)q;
  if (B >= kBigBucket) big[atomicAdd(big_cnt, 1u)] = (uint32_t)b;
}

// numpy default_rng((phase_seed, h)).permutation(B) (Fisher-Yates with
// bounded draws), then the draw walk of search.py:151-164 until quota valid
// members are taken.  Member j of a bucket is found in its runs (insertion
// order) by binary search on the run offsets.  `p` holds B entries (global
// or shared memory); one thread.
__device__ __forceinline__ void walk_bucket(int64_t b, uint32_t* p, const uint64_t* __restrict__ skey,
                                            const uint32_t* __restrict__ sval, const uint32_t* __restrict__ rstart,
                                            const uint32_t* __restrict__ cum, const uint32_t* __restrict__ bstart,
                                            const uint32_t* __restrict__ qoff, const uint32_t* __restrict__ quota,
                                            const uint8_t* __restrict__ verdict, uint64_t phase_seed, bool filled,
                                            int64_t* __restrict__ slot, uint32_t* __restrict__ taken,
                                            int64_t* __restrict__ rej, uint32_t* __restrict__ rejn) {
  const uint32_t r0 = bstart[b], r1 = bstart[b + 1];
  const uint32_t s0 = cum[r0], B = cum[r1] - s0;
  if (!filled)
    for (uint32_t i = 0; i < B; ++i) p[i] = i;
  Pcg64 g;
  seed_pair(g, phase_seed, skey[r0]);
  for (uint32_t i = B - 1; i >= 1; --i) {   // numpy Generator.permutation (Fisher-Yates)
    const uint32_t j = (uint32_t)g.interval(i);
    const uint32_t t = p[i]; p[i] = p[j]; p[j] = t;
  }
  const uint32_t q = quota[b];
  uint32_t t = 0, nr = 0;
  for (uint32_t i = 0; i < B; ++i) {
    const uint32_t o = s0 + p[i];
    uint32_t lo = r0, hi = r1 - 1;           // last run with cum[run] <= o
    while (lo < hi) {
      const uint32_t mid = (lo + hi + 1) >> 1;
      if (cum[mid] <= o) lo = mid; else hi = mid - 1;
    }
    const uint32_t m = rstart[sval[lo]] + (o - cum[lo]);
    if (verdict[m] == 0) {
      slot[qoff[b] + t] = m;
      if (++t == q) break;
    } else {
      rej[s0 + nr] = m;
      ++nr;
    }
  }
  taken[b] = t;
  rejn[b] = nr;
}

// Small buckets: one thread each, the permutation in global memory (the
// bucket's slice of `perm`).

__global__ void k4_walk(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ sval,
                        const uint32_t* __restrict__ rstart, const uint32_t* __restrict__ cum,
                        const uint32_t* __restrict__ bstart, const uint32_t* __restrict__ nb_dev,
                        const uint32_t* __restrict__ qoff, const uint32_t* __restrict__ quota,
                        const uint8_t* __restrict__ verdict, uint64_t phase_seed, uint32_t* __restrict__ perm,
                        int64_t* __restrict__ slot, uint32_t* __restrict__ taken, int64_t* __restrict__ rej,
                        uint32_t* __restrict__ rejn) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= (int64_t)*nb_dev) return;
  const uint32_t s0 = cum[bstart[b]], B = cum[bstart[b + 1]] - s0;
  if (B >= kBigBucket) return;   // k4_walk_big
  walk_bucket(b, perm + s0, skey, sval, rstart, cum, bstart, qoff, quota, verdict, phase_seed, false, slot, taken,
              rej, rejn);
}

// Big buckets (random schedules of a small pipeline share a few structures:
// C4 has 16 buckets of ~16K): one CTA each.  The Fisher-Yates shuffle is
// sequential, so one thread runs it on a permutation in shared memory
// (initialised by the whole CTA).  The walk is then parallel: every thread
// maps its strided positions to candidates (run lookup: O(1) when every run
// of the bucket is one candidate, else a binary search) and their verdicts,
// and one thread scans the validity bitmask in draw order.  Buckets beyond
// the shared capacity take the one-thread path on their global slice.
constexpr int kWalkBits = kWalkSmemEntries / 32;

__global__ void __launch_bounds__(256) k4_walk_big(
    const uint64_t* __restrict__ skey, const uint32_t* __restrict__ sval, const uint32_t* __restrict__ rstart,
    const uint32_t* __restrict__ cum, const uint32_t* __restrict__ bstart, const uint32_t* __restrict__ nb_dev,
    const uint32_t* __restrict__ qoff, const uint32_t* __restrict__ quota, const uint8_t* __restrict__ verdict,
    uint64_t phase_seed, uint32_t* __restrict__ perm, int64_t* __restrict__ slot, uint32_t* __restrict__ taken,
    int64_t* __restrict__ rej, uint32_t* __restrict__ rejn, const uint32_t* __restrict__ big,
    const uint32_t* __restrict__ big_cnt) {
  extern __shared__ uint32_t ps[];
  __shared__ uint32_t vbits[kWalkBits];
  const int64_t nbig = *big_cnt;
  for (int64_t bi = blockIdx.x; bi < nbig; bi += gridDim.x) {
    const int64_t b = big[bi];
    const uint32_t r0 = bstart[b], r1 = bstart[b + 1];
    const uint32_t s0 = cum[r0], B = cum[r1] - s0;
    if (B > (uint32_t)kWalkSmemEntries) {
      if (threadIdx.x == 0)
        walk_bucket(b, perm + s0, skey, sval, rstart, cum, bstart, qoff, quota, verdict, phase_seed, false, slot,
                    taken, rej, rejn);
      __syncthreads();
      continue;
    }
    for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) ps[i] = i;
    for (uint32_t i = threadIdx.x; i < (B + 31) / 32; i += blockDim.x) vbits[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {   // numpy Generator.permutation (Fisher-Yates)
      Pcg64 g;
      seed_pair(g, phase_seed, skey[r0]);
      for (uint32_t i = B - 1; i >= 1; --i) {
        const uint32_t j = (uint32_t)g.interval(i);
        const uint32_t t = ps[i]; ps[i] = ps[j]; ps[j] = t;
      }
    }
    __syncthreads();
    const bool singles = (r1 - r0) == B;   // every run one candidate
    for (uint32_t i = threadIdx.x; i < B; i += blockDim.x) {
      const uint32_t o = s0 + ps[i];
      uint32_t lo;
      if (singles) {
        lo = r0 + ps[i];
      } else {
        lo = r0;
        uint32_t hi = r1 - 1;           // last run with cum[run] <= o
        while (lo < hi) {
          const uint32_t mid = (lo + hi + 1) >> 1;
          if (cum[mid] <= o) lo = mid; else hi = mid - 1;
        }
      }
      const uint32_t m = rstart[sval[lo]] + (o - cum[lo]);
      ps[i] = m;                         // position -> candidate
      if (verdict[m] == 0) atomicOr(&vbits[i >> 5], 1u << (i & 31));
    }
    __syncthreads();
    if (threadIdx.x == 0) {   // search.py:151-164: draw order until quota valid
      const uint32_t q = quota[b];
      uint32_t t = 0, nr = 0;
      for (uint32_t i = 0; i < B; ++i) {
        if ((vbits[i >> 5] >> (i & 31)) & 1u) {
          slot[qoff[b] + t] = ps[i];
          if (++t == q) break;
        } else {
          rej[s0 + nr] = ps[i];
          ++nr;
        }
      }
      taken[b] = t;
      rejn[b] = nr;
    }
    __syncthreads();
  }
}

__global__ void k4_gather(const uint32_t* __restrict__ nb_dev, const uint32_t* __restrict__ qoff,
                          const uint32_t* __restrict__ taken, const uint32_t* __restrict__ toff,
                          const int64_t* __restrict__ slot, int64_t* __restrict__ rep_idx,
                          const uint32_t* __restrict__ bstart, const uint32_t* __restrict__ cum,
                          const uint32_t* __restrict__ rejn, const uint32_t* __restrict__ roff,
                          const int64_t* __restrict__ rej, int64_t* __restrict__ rej_idx,
                          const uint32_t* __restrict__ tot_reps, const uint32_t* __restrict__ tot_rej,
                          int64_t* __restrict__ n_reps, int64_t* __restrict__ n_rejects) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b < (int64_t)*nb_dev) {
    for (uint32_t t = 0; t < taken[b]; ++t) rep_idx[toff[b] + t] = slot[qoff[b] + t];
    if (rej_idx) {
      const uint32_t s0 = cum[bstart[b]];
      for (uint32_t t = 0; t < rejn[b]; ++t) rej_idx[roff[b] + t] = rej[s0 + t];
    }
  }
  if (b == 0) {
    *n_reps = (int64_t)*tot_reps;
    *n_rejects = (int64_t)*tot_rej;
  }
}

// workspace carve-up for K4 (every array sized for the candidate count n)
struct SelWs {
  uint32_t *head, *runid, *rstart, *len, *cum, *bhead, *bid, *bstart, *quota, *qoff, *taken, *toff, *rejn,
      *roff, *perm, *sums, *hist, *cnt, *big;   // cnt: m, nb, total reps, total rejects, big buckets
  uint32_t *rval, *rval2;
  uint64_t *rkey, *rkey2;
  int64_t *slot, *rej;
};

static size_t carve(SelWs& w, void* base, int64_t n) {
  size_t o = 0;
  char* p = (char*)base;
  auto take = [&](size_t bytes) { char* r = p ? p + o : nullptr; o += align256(bytes); return r; };
  w.head = (uint32_t*)take(4 * n);
  w.runid = (uint32_t*)take(4 * n);
  w.rstart = (uint32_t*)take(4 * (n + 1));
  w.len = (uint32_t*)take(4 * n);
  w.cum = (uint32_t*)take(4 * (n + 1));
  w.bhead = (uint32_t*)take(4 * n);
  w.bid = (uint32_t*)take(4 * n);
  w.bstart = (uint32_t*)take(4 * (n + 1));
  w.quota = (uint32_t*)take(4 * n);
  w.qoff = (uint32_t*)take(4 * n);
  w.taken = (uint32_t*)take(4 * n);
  w.toff = (uint32_t*)take(4 * n);
  w.rejn = (uint32_t*)take(4 * n);
  w.roff = (uint32_t*)take(4 * n);
  w.perm = (uint32_t*)take(4 * n);
  w.rval = (uint32_t*)take(4 * n);
  w.rval2 = (uint32_t*)take(4 * n);
  w.rkey = (uint64_t*)take(8 * n);
  w.rkey2 = (uint64_t*)take(8 * n);
  w.slot = (int64_t*)take(8 * n);
  w.rej = (int64_t*)take(8 * n);
  w.hist = (uint32_t*)take(rs_hist_bytes(n));
  const size_t sb = std::max(rs_sums_bytes(n), align256(4 * (scan_tiles_of(n) + 1)));
  w.sums = (uint32_t*)take(sb);
  w.cnt = (uint32_t*)take(32);
  w.big = (uint32_t*)take(4 * (n / kBigBucket + 1));
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
  uint32_t *m_dev = w.cnt, *nb_dev = w.cnt + 1, *tot_reps = w.cnt + 2, *tot_rej = w.cnt + 3, *big_cnt = w.cnt + 4;
  k4_heads<<<G, T, 0, st>>>(hashes, n, w.head); g_launch_count++;
  scan_u32(w.head, w.runid, n, nullptr, false, w.sums, m_dev, st);
  k4_runs<<<G, T, 0, st>>>(hashes, n, w.runid, w.rkey, w.rval, w.rstart); g_launch_count++;
  radix_sort_pairs(w.rkey, w.rval, w.rkey2, w.rval2, n, m_dev, w.hist, w.sums, st);
  k4_sorted<<<G, T, 0, st>>>(w.rkey, w.rval, w.rstart, m_dev, n, w.len, w.bhead); g_launch_count++;
  scan_u32(w.len, w.cum, n, m_dev, false, w.sums, nullptr, st);
  scan_u32(w.bhead, w.bid, n, m_dev, false, w.sums, nullptr, st);
  k4_buckets<<<G, T, 0, st>>>(w.rkey, w.bid, m_dev, n, w.bstart, w.cum, nb_dev); g_launch_count++;
  cudaMemsetAsync(big_cnt, 0, 4, st);
  k4_quota<<<G, T, 0, st>>>(w.bstart, w.cum, nb_dev, w.quota, w.big, big_cnt); g_launch_count++;
  scan_u32(w.quota, w.qoff, n, nb_dev, false, w.sums, nullptr, st);
  k4_walk<<<G, 64, 0, st>>>(w.rkey, w.rval, w.rstart, w.cum, w.bstart, nb_dev, w.qoff, w.quota, verdict,
                            phase_seed, w.perm, w.slot, w.taken, w.rej, w.rejn); g_launch_count++;
  if (n >= (int64_t)kBigBucket) {   // a bucket of >= kBigBucket members is possible
    static bool attr = false;
    if (!attr) {
      if (cudaFuncSetAttribute(k4_walk_big, cudaFuncAttributeMaxDynamicSharedMemorySize, 4 * kWalkSmemEntries) !=
          cudaSuccess)
        return -3;
      attr = true;
    }
    const int64_t maxbig = n / kBigBucket;
    const unsigned gb = (unsigned)(maxbig < 296 ? maxbig : 296);
    k4_walk_big<<<gb, 256, 4 * kWalkSmemEntries, st>>>(w.rkey, w.rval, w.rstart, w.cum, w.bstart, nb_dev, w.qoff,
                                                       w.quota, verdict, phase_seed, w.perm, w.slot, w.taken, w.rej,
                                                       w.rejn, w.big, big_cnt);
    g_launch_count++;
  }
  scan_u32(w.taken, w.toff, n, nb_dev, false, w.sums, tot_reps, st);
  scan_u32(w.rejn, w.roff, n, nb_dev, false, w.sums, tot_rej, st);
  k4_gather<<<G, T, 0, st>>>(nb_dev, w.qoff, w.taken, w.toff, w.slot, rep_idx, w.bstart, w.cum, w.rejn, w.roff,
                             w.rej, rej_idx, tot_reps, tot_rej, n_reps, n_rejects); g_launch_count++;
  return 0;
}

// ------------------------------------------------------------ K5 kernels ---
// element count given on the host (nmax) or, when ndev is set, on the device
__device__ __forceinline__ int64_t count64(int64_t nmax, const int64_t* ndev) {
  if (!ndev) return nmax;
  const int64_t c = *ndev;
  return c < nmax ? (c < 0 ? 0 : c) : nmax;
}

__device__ __forceinline__ uint64_t sortable(double x) {
  if (x == 0.0) x = 0.0;   // -0.0 == 0.0 in the reference's sort
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ULL);
}
__device__ __forceinline__ double unsortable(uint64_t k) {
  const uint64_t b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFULL) : ~k;
  return __longlong_as_double((long long)b);
}

__global__ void keys_kernel(const double* __restrict__ costs, const uint64_t* __restrict__ ph,
                            const int64_t* __restrict__ rep, int64_t nmax, const int64_t* __restrict__ ndev,
                            const uint64_t* __restrict__ flagged, int64_t nflag, double penalty,
                            uint64_t* __restrict__ key, uint64_t* __restrict__ ckey, double* __restrict__ kval) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count64(nmax, ndev)) return;
  const int64_t src = rep ? rep[i] : i;   // rep: the representatives' candidate indices
  double c = costs[src];
  bool f = false;
  if (nflag > 0) {
    int64_t lo = 0, hi = nflag;
    const uint64_t h = ph[src];
    while (lo < hi) { int64_t mid = (lo + hi) >> 1; if (flagged[mid] < h) lo = mid + 1; else hi = mid; }
    f = lo < nflag && flagged[lo] == h;
  }
  double k = f ? c * penalty : c;   // apply_pass_penalty (search.py:76-87)
  kval[i] = k;
  key[i] = sortable(k);
  ckey[i] = sortable(c);
}

// Gumbel noise on log-cost (search.py:185-192): the reference draws
// rng.gumbel(size=n) from default_rng((phase_seed, 0x657870)), i.e. draw i
// uses the (i+1)-th PCG64 output unless an earlier draw hit the 2^-53
// rejection (U == 1).  Each thread jumps ahead to its chunk; a rejection
// anywhere raises `redo` and the sequential kernel below redraws the lot.
constexpr int kGumbelChunk = 32;
__device__ __forceinline__ double gumbel_key(double kv, double gum, double temperature) {
  const double k = kv > 1e-300 ? kv : 1e-300;
  return log(k) + gum * temperature;
}

__global__ void gumbel_parallel(double* __restrict__ kval, uint64_t* __restrict__ key, int64_t nmax,
                                const int64_t* __restrict__ ndev, double temperature, uint64_t phase_seed,
                                uint32_t* __restrict__ redo) {
  const int64_t n = count64(nmax, ndev);
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t i0 = c * kGumbelChunk;
  if (i0 >= n) return;
  Pcg64 g;
  seed_pair(g, phase_seed, 0x657870ULL);
  pcg_advance(g, (uint64_t)i0);
  const int64_t i1 = i0 + kGumbelChunk < n ? i0 + kGumbelChunk : n;
  for (int64_t i = i0; i < i1; ++i) {
    const double u = 1.0 - g.next_double();
    if (!(u < 1.0)) { atomicExch(redo, 1u); return; }
    const double v = gumbel_key(kval[i], -log(-log(u)), temperature);
    key[i] = sortable(v);
  }
}

__global__ void gumbel_serial(const double* __restrict__ kval, uint64_t* __restrict__ key, int64_t nmax,
                              const int64_t* __restrict__ ndev, double temperature, uint64_t phase_seed,
                              const uint32_t* __restrict__ redo) {
  if (threadIdx.x != 0 || blockIdx.x != 0 || *redo == 0) return;
  const int64_t n = count64(nmax, ndev);
  Pcg64 g;
  seed_pair(g, phase_seed, 0x657870ULL);
  for (int64_t i = 0; i < n; ++i) {
    double u;
    do { u = 1.0 - g.next_double(); } while (!(u < 1.0));
    key[i] = sortable(gumbel_key(kval[i], -log(-log(u)), temperature));
  }
}

// Single-CTA stable radix select: the key of stable rank `target` and how
// many keys are strictly smaller.
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
    if (threadIdx.x < 32) {   // warp 0: find the digit holding rank s_rank
      const int lane = threadIdx.x;
      unsigned c8[8];
      unsigned tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { c8[j] = hist[lane * 8 + j]; tot += c8[j]; }
      unsigned incl = tot;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int64_t r = s_rank;
      const int64_t excl = (int64_t)(incl - tot);
      const bool mine = excl <= r && r < (int64_t)incl;
      const unsigned who = __ballot_sync(0xffffffffu, mine);
      __syncwarp();   // every lane has read s_rank before the owner rewrites it
      if (lane == __ffs(who) - 1) {
        int64_t acc = excl;
        int d = lane * 8;
        for (int j = 0; j < 8; ++j, ++d) {
          if (acc + c8[j] > r) break;
          acc += c8[j];
        }
        s_rank = r - acc;
        s_less += acc;
        s_prefix = pre | ((uint64_t)d << shift);
      }
    }
    __syncthreads();
  }
  kstar = s_prefix;
  less = s_less;
  __syncthreads();
}

// Block-wide bitonic sort of P (power of two) u64 keys + u32 payloads in
// shared memory, ascending by (key, payload).
template <int NT>
__device__ void bitonic_kp(uint64_t* sk, uint32_t* sp, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += NT) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = sk[i] > sk[j] || (sk[i] == sk[j] && sp[i] > sp[j]);
          if (gt == up) {
            const uint64_t tk = sk[i]; sk[i] = sk[j]; sk[j] = tk;
            const uint32_t tp = sp[i]; sp[i] = sp[j]; sp[j] = tp;
          }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ bool band_break(double a, double b, double band) {   // a <= b, adjacent
  return (b - a) > band * fmax(fabs(a), fabs(b));
}

// The cut (search.py:193, 196-200) with the tie band.  Keys are ordered by
// (band group, rep position), where a band group is a maximal run of keys
// (in value order) whose adjacent gaps are within `band` (relative) —
// exact ties are the zero-width case, so band 0 is the reference's stable
// sort.  Only the group structure around one rank matters:
//   CTA 0 (top-k): every key <= the k-th key + margin, i.e. all keys that
//     can precede or share a group with rank k-1;
//   CTA 1 (bottom half, unpenalized costs): the keys within a margin of
//     rank n/2; everything below the window is in the top half, everything
//     above it in the bottom half.
// The window is widened until no band group straddles its edges (a radix
// select, one counting/collecting pass per try), then sorted in shared
// memory by value, split into groups, and re-sorted by (group, position).
constexpr int kWinNT = 1024;
constexpr int kWinCap = 16384;
constexpr int kWinSmem = kWinCap * (8 + 4);

__global__ void __launch_bounds__(kWinNT) cut_kernel(const uint64_t* __restrict__ key, const uint64_t* __restrict__ ckey,
                                                     int64_t nmax, const int64_t* __restrict__ ndev, int64_t k,
                                                     double band, int64_t* __restrict__ out_pos,
                                                     int64_t* __restrict__ n_out, uint8_t* __restrict__ bottom,
                                                     uint32_t* __restrict__ status) {
  const int64_t n = count64(nmax, ndev);
  if (k > n) k = n;
  extern __shared__ __align__(16) unsigned char win_smem[];
  uint64_t* wk = (uint64_t*)win_smem;
  uint32_t* wp = (uint32_t*)(wk + kWinCap);
  __shared__ int s_cnt, s_ok;
  __shared__ unsigned long long s_clo, s_maxb, s_mina, s_wmin, s_wmax;
  __shared__ uint32_t ws[32];
  __shared__ uint32_t tot;
  const bool top = blockIdx.x == 0;
  if (!top && !bottom) return;
  if (top && k < 1) {   // empty representative set (device count 0)
    if (threadIdx.x == 0) *n_out = 0;
    return;
  }
  const uint64_t* kk = top ? key : ckey;
  if (!top && n <= 1) {
    for (int64_t i = threadIdx.x; i < n; i += kWinNT) bottom[i] = 0;
    return;
  }
  const int64_t r = top ? k - 1 : n / 2;
  uint64_t kstar;
  int64_t less;
  radix_select<kWinNT>(kk, n, r, kstar, less);
  const double V = unsortable(kstar);
  double W = 4.0;
  uint64_t klo = 0, khi = ~0ull;
  for (int it = 0;; ++it) {
    const double d = W * band * fabs(V);
    klo = top ? 0ull : sortable(V - d);
    khi = sortable(V + d);
    if (kstar < klo) klo = kstar;
    if (kstar > khi) khi = kstar;
    if (threadIdx.x == 0) { s_cnt = 0; s_clo = 0; s_maxb = 0; s_mina = ~0ull; s_wmin = ~0ull; s_wmax = 0; }
    __syncthreads();
    unsigned long long clo = 0, maxb = 0, mina = ~0ull, wmin = ~0ull, wmax = 0;
    for (int64_t i = threadIdx.x; i < n; i += kWinNT) {
      const uint64_t x = kk[i];
      if (x < klo) { ++clo; maxb = x > maxb ? x : maxb; }
      else if (x > khi) { mina = x < mina ? x : mina; }
      else {
        wmin = x < wmin ? x : wmin;
        wmax = x > wmax ? x : wmax;
        const int s = atomicAdd(&s_cnt, 1);
        if (s < kWinCap) { wk[s] = x; wp[s] = (uint32_t)i; }
      }
    }
    atomicAdd(&s_clo, clo);
    if (clo) atomicMax(&s_maxb, maxb);
    if (mina != ~0ull) atomicMin(&s_mina, mina);
    atomicMin(&s_wmin, wmin);
    atomicMax(&s_wmax, wmax);
    __syncthreads();
    if (threadIdx.x == 0) {
      bool ok = true;
      if (s_clo && !band_break(unsortable(s_maxb), unsortable(s_wmin), band)) ok = false;
      if (s_mina != ~0ull && !band_break(unsortable(s_wmax), unsortable(s_mina), band)) ok = false;
      s_ok = s_cnt > kWinCap ? -1 : (ok ? 1 : 0);
    }
    __syncthreads();
    if (s_ok != 0) break;
    if (it >= 16) { if (threadIdx.x == 0) s_ok = -1; __syncthreads(); break; }
    W *= 16.0;
    __syncthreads();
  }
  if (s_ok < 0) {   // a tie group wider than the shared-memory window
    if (threadIdx.x == 0) atomicOr(status, top ? 1u : 2u);
    return;
  }
  const int cnt = s_cnt;
  int P = 1;
  while (P < cnt) P <<= 1;
  for (int i = cnt + threadIdx.x; i < P; i += kWinNT) { wk[i] = ~0ull; wp[i] = 0xFFFFFFFFu; }
  __syncthreads();
  bitonic_kp<kWinNT>(wk, wp, P);
  // group ids: inclusive scan of the band breaks (each thread owns a
  // contiguous chunk of the sorted window)
  constexpr int kPer = kWinCap / kWinNT;
  const int j0 = threadIdx.x * kPer;
  uint32_t brk[kPer];
  uint32_t s = 0;
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = j0 + q;
    brk[q] = (j > 0 && j < cnt && band_break(unsortable(wk[j - 1]), unsortable(wk[j]), band)) ? 1u : 0u;
    s += brk[q];
  }
  uint32_t gid = block_scan_excl(s, ws, &tot);   // ends with a barrier: all reads of wk are done
#pragma unroll
  for (int q = 0; q < kPer; ++q) {
    const int j = j0 + q;
    gid += brk[q];
    if (j < cnt) wk[j] = ((uint64_t)gid << 32) | wp[j];
  }
  __syncthreads();
  bitonic_kp<kWinNT>(wk, wp, P);
  if (top) {
    const int64_t kk_ = k < n ? k : n;
    for (int j = threadIdx.x; j < kk_; j += kWinNT) out_pos[j] = (int64_t)(wk[j] & 0xFFFFFFFFull);
    if (threadIdx.x == 0) *n_out = kk_;
    return;
  }
  const int64_t clo = (int64_t)s_clo;
  for (int64_t i = threadIdx.x; i < n; i += kWinNT) {
    const uint64_t x = kk[i];
    if (x < klo) bottom[i] = 0;
    else if (x > khi) bottom[i] = 1;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < cnt; j += kWinNT)
    bottom[wk[j] & 0xFFFFFFFFull] = (clo + j >= r) ? 1 : 0;
}

__global__ void cut_status(const uint32_t* __restrict__ status, int64_t* __restrict__ n_out) {
  if (threadIdx.x == 0 && *status) *n_out = -(int64_t)*status;
}

int64_t topk_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  return (int64_t)(align256(8 * n) * 3 + align256(16));
}

int beam_topk(const double* costs, const uint64_t* ph, const int64_t* rep, int64_t n, const int64_t* ndev,
              const uint64_t* flagged, int64_t nflag, double penalty, double temperature, uint64_t phase_seed,
              int64_t k, double band, void* ws, int64_t ws_bytes, int64_t* out_pos, int64_t* n_out, uint8_t* bottom,
              cudaStream_t st) {
  if (n <= 0) { cudaMemsetAsync(n_out, 0, 8, st); return 0; }
  if (topk_workspace_bytes(n) > ws_bytes) return -2;
  if (n >= (int64_t)0xFFFFFFFF) return -3;
  if (k > n) k = n;
  if (k < 1 || k > kWinCap || !(band >= 0)) return -4;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(cut_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kWinSmem) != cudaSuccess)
      return -5;
    attr = true;
  }
  char* p = (char*)ws;
  uint64_t* key = (uint64_t*)p; p += align256(8 * n);
  uint64_t* ckey = (uint64_t*)p; p += align256(8 * n);
  double* kval = (double*)p; p += align256(8 * n);
  uint32_t* status = (uint32_t*)p;
  cudaMemsetAsync(status, 0, 8, st);
  const unsigned G = (unsigned)((n + 255) / 256);
  keys_kernel<<<G, 256, 0, st>>>(costs, ph, rep, n, ndev, flagged, nflag, penalty, key, ckey, kval); g_launch_count++;
  if (temperature > 0) {
    const int64_t chunks = (n + kGumbelChunk - 1) / kGumbelChunk;
    gumbel_parallel<<<(unsigned)((chunks + 127) / 128), 128, 0, st>>>(kval, key, n, ndev, temperature, phase_seed,
                                                                       status + 1);
    gumbel_serial<<<1, 32, 0, st>>>(kval, key, n, ndev, temperature, phase_seed, status + 1);
    g_launch_count += 2;
  }
  cut_kernel<<<bottom ? 2 : 1, kWinNT, kWinSmem, st>>>(key, ckey, n, ndev, k, band, out_pos, n_out, bottom, status);
  cut_status<<<1, 32, 0, st>>>(status, n_out);
  g_launch_count += 2;
  return 0;
}

}  // namespace gs
