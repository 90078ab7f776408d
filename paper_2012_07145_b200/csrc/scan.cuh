// Device-wide and block-wide prefix sums of u32 counts, shared by K1's run
// preparation and K4's bucketing (no CUB on the step's launch list).
//
// scan_u32 is a three-launch reduce-then-scan: per-tile sums, one CTA scans
// the tile sums (writing the grand total to a device word), and a down-sweep
// that rescans each tile from its base.  The element count may live on the
// device (`dcount`, clamped to the host bound `nmax`), so a scan whose length
// an earlier kernel produced needs no host round trip.  In-place (in == out)
// is allowed: every element is read before it is written by the same thread.
#pragma once
#include "gs_internal.cuh"

namespace gs {

inline size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

__device__ __forceinline__ int64_t count_of(int64_t nmax, const uint32_t* dcount) {
  if (!dcount) return nmax;
  const int64_t c = (int64_t)*dcount;
  return c < nmax ? c : nmax;
}

constexpr int kScanNT = 1024;
constexpr int kScanIPT = 8;
constexpr int kScanTile = kScanNT * kScanIPT;

inline int64_t scan_tiles_of(int64_t n) { return n < 1 ? 1 : (n + kScanTile - 1) / kScanTile; }

// Block-wide exclusive scan of one u32 per thread (blockDim a multiple of 32,
// `ws` 32 shared words).  *tot receives the block total.  Ends with a
// barrier, so shared data read before the call may be overwritten after it.
__device__ __forceinline__ uint32_t block_scan_excl(uint32_t v, uint32_t* ws, uint32_t* tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = (int)(blockDim.x >> 5);
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[w] = x;
  __syncthreads();
  if (w == 0) {
    const uint32_t s = lane < nw ? ws[lane] : 0u;
    uint32_t t = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) ws[lane] = t - s;
    if (lane == 31) *tot = t;
  }
  __syncthreads();
  const uint32_t r = ws[w] + x - v;
  __syncthreads();
  return r;
}

static __global__ void __launch_bounds__(kScanNT) scan_reduce_kernel(const uint32_t* __restrict__ in, int64_t nmax,
                                                                     const uint32_t* __restrict__ dcount,
                                                                     uint32_t* __restrict__ sums) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t tot;
  const int64_t n = count_of(nmax, dcount);
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  uint32_t s = 0;
  if (t0 < n) {
    for (int j = 0; j < kScanIPT; ++j) {   // coalesced: round j covers [t0 + j*NT, t0 + (j+1)*NT)
      const int64_t i = t0 + (int64_t)j * kScanNT + threadIdx.x;
      if (i < n) s += in[i];
    }
  }
  block_scan_excl(s, ws, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// one CTA: exclusive scan of the tile sums in place; sums[tiles] and *total
// receive the grand total
static __global__ void __launch_bounds__(kScanNT) scan_sums_kernel(uint32_t* __restrict__ sums, int64_t tiles,
                                                                   uint32_t* __restrict__ total) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t tot;
  uint32_t carry = 0;
  for (int64_t b = 0; b < tiles; b += kScanNT) {
    const int64_t i = b + threadIdx.x;
    const uint32_t v = i < tiles ? sums[i] : 0u;
    const uint32_t e = block_scan_excl(v, ws, &tot);
    if (i < tiles) sums[i] = carry + e;
    carry += tot;
  }
  if (threadIdx.x == 0) {
    sums[tiles] = carry;
    if (total) *total = carry;
  }
}

// down-sweep: thread t owns the kScanIPT consecutive elements
// [t0 + t*IPT, t0 + (t+1)*IPT) of its tile
static __global__ void __launch_bounds__(kScanNT) scan_down_kernel(const uint32_t* in, uint32_t* out, int64_t nmax,
                                                                   const uint32_t* __restrict__ dcount,
                                                                   const uint32_t* __restrict__ sums, int inclusive) {
  __shared__ uint32_t ws[32];
  __shared__ uint32_t tot;
  const int64_t n = count_of(nmax, dcount);
  const int64_t t0 = (int64_t)blockIdx.x * kScanTile;
  if (t0 >= n) return;   // uniform per block
  const int64_t i0 = t0 + (int64_t)threadIdx.x * kScanIPT;
  uint32_t v[kScanIPT];
  uint32_t s = 0;
#pragma unroll
  for (int j = 0; j < kScanIPT; ++j) {
    v[j] = i0 + j < n ? in[i0 + j] : 0u;
    s += v[j];
  }
  uint32_t run = sums[blockIdx.x] + block_scan_excl(s, ws, &tot);
#pragma unroll
  for (int j = 0; j < kScanIPT; ++j) {
    if (i0 + j < n) out[i0 + j] = inclusive ? run + v[j] : run;
    run += v[j];
  }
}

// out[i] = sum of in[0..i) (exclusive) or in[0..i] (inclusive) for
// i < count_of(nmax, dcount); `sums` holds scan_tiles_of(nmax) + 1 words;
// `total` (device, may be null) receives the sum of all counted elements.
static inline void scan_u32(const uint32_t* in, uint32_t* out, int64_t nmax, const uint32_t* dcount, bool inclusive,
                            uint32_t* sums, uint32_t* total, cudaStream_t st) {
  const int64_t tiles = scan_tiles_of(nmax);
  scan_reduce_kernel<<<(unsigned)tiles, kScanNT, 0, st>>>(in, nmax, dcount, sums);
  scan_sums_kernel<<<1, kScanNT, 0, st>>>(sums, tiles, total);
  scan_down_kernel<<<(unsigned)tiles, kScanNT, 0, st>>>(in, out, nmax, dcount, sums, inclusive ? 1 : 0);
  g_launch_count += 3;
}

}  // namespace gs
