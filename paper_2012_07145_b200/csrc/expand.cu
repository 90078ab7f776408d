// Beam-step expansion on the device: every phase-2
// tiling of each parent's step root, in the reference's enumeration order
// (search.py:223-235 `_phase2_candidates`; options.py:144-183
// `enumerate_serial_tilings` / `enumerate_thread_tilings`, products with
// dim 0 varying slowest).  The host then uploads only the beam (parents),
// not the expanded candidate records.
#include "gs_internal.cuh"
#include "scan.cuh"

namespace gs {

constexpr int kExpandWarps = 2;
constexpr int kMaxTilings = 4096;   // per parent (one warp's list in shared memory)

// sorted, de-duplicated serial options of one extent; returns count
__device__ int serial_opts(const GsTilingMenus& m, int e, int* o) {
  int n = 0;
  auto add = [&](int v) {
    for (int i = 0; i < n; ++i) if (o[i] == v) return;
    int j = n++;
    while (j > 0 && o[j - 1] > v) { o[j] = o[j - 1]; --j; }
    o[j] = v;
  };
  for (int i = 0; i < m.n_serial_powers; ++i) if (m.serial_powers[i] <= e) add(m.serial_powers[i]);
  for (int i = 0; i < m.n_odd_serial; ++i) {
    const int v = m.odd_serial[i];
    if (v <= e && e % v == 0 && (e / v) % m.warp_size == 0) add(v);
  }
  if (n == 0) o[n++] = 1;
  return n;
}

// sorted, de-duplicated thread options of one post-serial extent
__device__ int thread_opts(const GsTilingMenus& m, int e, bool inner, int* o) {
  int n = 0;
  const int* menu = inner ? m.innermost_thread : m.outer_thread;
  const int cnt = inner ? m.n_innermost : m.n_outer;
  for (int i = 0; i < cnt; ++i) {
    const int v = menu[i] < e ? menu[i] : e;
    bool dup = false;
    for (int k = 0; k < n; ++k) dup |= o[k] == v;
    if (dup) continue;
    int j = n++;
    while (j > 0 && o[j - 1] > v) { o[j] = o[j - 1]; --j; }
    o[j] = v;
  }
  return n;
}

// Enumerate the tilings of a func (one thread).  emit(serial[], thread[])
// is called in reference order; returns the count.
template <typename F>
__device__ int64_t enum_tilings(const GsTilingMenus& m, const GsFunc& fn, F&& emit) {
  const int nd = fn.ndim;
  int so[GS_MAX_NDIM][16], sn[GS_MAX_NDIM];
  for (int d = 0; d < nd; ++d) sn[d] = serial_opts(m, fn.extent[d], so[d]);
  int64_t count = 0;
  int idx[GS_MAX_NDIM] = {0, 0, 0, 0};
  for (;;) {
    int sv[GS_MAX_NDIM] = {1, 1, 1, 1};
    int64_t prod = 1;
    for (int d = 0; d < nd; ++d) { sv[d] = so[d][idx[d]]; prod *= sv[d]; }
    if (prod <= m.unroll_budget) {
      int post[GS_MAX_NDIM], inner = 0;
      for (int d = 0; d < nd; ++d) post[d] = (fn.extent[d] + sv[d] - 1) / sv[d];
      inner = -1;
      for (int d = 0; d < nd; ++d) if (post[d] >= 16) { inner = d; break; }
      if (inner < 0) inner = 0;
      int to[GS_MAX_NDIM][16], tn[GS_MAX_NDIM];
      for (int d = 0; d < nd; ++d) tn[d] = thread_opts(m, post[d], d == inner, to[d]);
      int tj[GS_MAX_NDIM] = {0, 0, 0, 0};
      for (;;) {
        int tv[GS_MAX_NDIM] = {1, 1, 1, 1};
        for (int d = 0; d < nd; ++d) tv[d] = to[d][tj[d]];
        emit(sv, tv);
        ++count;
        int d = nd - 1;   // last dim fastest
        while (d >= 0 && ++tj[d] == tn[d]) { tj[d] = 0; --d; }
        if (d < 0) break;
      }
    }
    int d = nd - 1;
    while (d >= 0 && ++idx[d] == sn[d]) { idx[d] = 0; --d; }
    if (d < 0) break;
  }
  return count;
}

__global__ void expand_count_kernel(const GsFunc* __restrict__ funcs, const GsDecision* __restrict__ parents,
                                    int64_t n, int S, const int32_t* __restrict__ step, GsTilingMenus m,
                                    uint32_t* __restrict__ counts, int* __restrict__ gerr) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int s = step[p];
  const int f = s >= 0 && s < S ? parents[p * S + s].func : 0xFFFF;
  if (f == 0xFFFF || parents[p * S + s].kind != GS_ROOT) { counts[p] = 0; atomicOr(gerr, 32); return; }
  const int64_t c = enum_tilings(m, funcs[f], [](const int*, const int*) {});
  if (c > kMaxTilings) atomicOr(gerr, 16);
  counts[p] = (uint32_t)(c > kMaxTilings ? 0 : c);   // over-long lists are skipped (and reported)
}

__global__ void __launch_bounds__(kExpandWarps * 32) expand_write_kernel(
    const GsFunc* __restrict__ funcs, const GsDecision* __restrict__ parents, int64_t n, int S,
    const int32_t* __restrict__ step, GsTilingMenus m, const int64_t* __restrict__ offsets,
    GsDecision* __restrict__ out, int64_t out_cap, int32_t* __restrict__ owner, int* __restrict__ gerr) {
  extern __shared__ __align__(16) uint8_t smx[];
  uint8_t (*til)[kMaxTilings][8] = reinterpret_cast<uint8_t (*)[kMaxTilings][8]>(smx);
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kExpandWarps;
  for (int64_t p = (int64_t)blockIdx.x * kExpandWarps + wib; p < n; p += nwarps) {
    const int64_t base = offsets[p], cnt = offsets[p + 1] - base;
    if (cnt <= 0 || cnt > kMaxTilings) continue;
    if (base + cnt > out_cap) {   // the caller's buffer is smaller than the step: write nothing past it
      if (lane == 0) atomicOr(gerr, 16);
      continue;
    }
    const int s = step[p];
    const GsDecision* par = parents + p * S;
    if (lane == 0) {
      int k = 0;
      enum_tilings(m, funcs[par[s].func], [&](const int* sv, const int* tv) {
        for (int d = 0; d < GS_MAX_NDIM; ++d) { til[wib][k][d] = (uint8_t)sv[d]; til[wib][k][4 + d] = (uint8_t)tv[d]; }
        ++k;
      });
    }
    __syncwarp();
    const uint4* src = reinterpret_cast<const uint4*>(par);
    const int nd = funcs[par[s].func].ndim;
    for (int64_t t = 0; t < cnt; ++t) {
      uint4* dst = reinterpret_cast<uint4*>(out + (base + t) * S);
      for (int i = lane; i < S; i += 32) {
        uint4 r = __ldg(src + i);
        if (i == s) {
          GsDecision d = *reinterpret_cast<const GsDecision*>(&r);
          d.flags = 3;
          for (int k = 0; k < nd; ++k) { d.serial[k] = til[wib][t][k]; d.thread[k] = til[wib][t][4 + k]; }
          r = *reinterpret_cast<const uint4*>(&d);
        }
        dst[i] = r;
      }
      if (owner && lane == 0) owner[base + t] = (int32_t)p;
    }
    __syncwarp();
  }
}

// offsets[0] = 0, offsets[p + 1] = inclusive prefix of the (u32) counts
__global__ void expand_offsets_kernel(const uint32_t* __restrict__ incl, int64_t n, int64_t* __restrict__ offsets) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p == 0) offsets[0] = 0;
  if (p < n) offsets[p + 1] = (int64_t)incl[p];
}

// counts | inclusive scan | scan tile sums
int64_t expand_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  return (int64_t)(2 * align256(4 * n) + align256(4 * (scan_tiles_of(n) + 1)));
}

int launch_expand(const GsFunc* funcs, const GsDecision* parents, int64_t n, int S, const int32_t* step,
                  const GsTilingMenus& m, int64_t* offsets, void* ws, int64_t ws_bytes, GsDecision* out,
                  int64_t out_cap, int32_t* owner, int* gerr, int num_sms, cudaStream_t st) {
  if (n <= 0) { cudaMemsetAsync(offsets, 0, sizeof(int64_t), st); return 0; }
  if (n > (int64_t)1 << 20) return -1;   // keeps the u32 scan exact: n * kMaxTilings < 2^32
  if (expand_workspace_bytes(n) > ws_bytes) return -2;
  uint8_t* w = static_cast<uint8_t*>(ws);
  uint32_t* counts = reinterpret_cast<uint32_t*>(w);
  uint32_t* incl = reinterpret_cast<uint32_t*>(w + align256(4 * n));
  uint32_t* sums = reinterpret_cast<uint32_t*>(w + 2 * align256(4 * n));
  expand_count_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(funcs, parents, n, S, step, m, counts, gerr);
  scan_u32(counts, incl, n, nullptr, true, sums, nullptr, st);
  expand_offsets_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st>>>(incl, n, offsets);
  g_launch_count += 2;
  if (out) {
    const int64_t want = (n + kExpandWarps - 1) / kExpandWarps;
    const int grid = (int)(want < (int64_t)num_sms * 16 ? want : (int64_t)num_sms * 16);
    const int smem = kExpandWarps * kMaxTilings * 8;
    cudaFuncSetAttribute(expand_write_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    expand_write_kernel<<<grid, kExpandWarps * 32, smem, st>>>(funcs, parents, n, S, step, m, offsets, out, out_cap,
                                                               owner, gerr);
    g_launch_count++;
  }
  return 0;
}

}  // namespace gs
