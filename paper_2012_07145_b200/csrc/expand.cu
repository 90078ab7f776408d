// Beam-step expansion on the device: every phase-2
// tiling of each parent's step root, in the reference's enumeration order
// (search.py:223-235 `_phase2_candidates`; options.py:144-183
// `enumerate_serial_tilings` / `enumerate_thread_tilings`, products with
// dim 0 varying slowest).  The host then uploads only the beam (parents),
// not the expanded candidate records.
#include "gs_internal.cuh"
#include "scan.cuh"
#include "rng.cuh"

namespace gs {

constexpr int kExpandWarps = 2;
constexpr int kMaxTilings = 4096;   // per parent (one warp's list in shared memory)

// sorted, de-duplicated serial options of one extent; returns count
__host__ __device__ int serial_opts(const GsTilingMenus& m, int e, int* o) {
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

// Phase-2 write: one warp per parent.  Lane 0 walks the tiling menu into a
// 512-entry shared-memory list (lists longer than that are written in
// chunks, each chunk re-walking the menu and keeping its own window), then
// the whole warp streams the chunk's candidates: the (tiling, record) pairs
// are flattened so every lane stores one 16-byte record per step (100-record
// candidates left a quarter of the lanes idle in a per-candidate loop), and
// the parent's records come from L1.  Eight warps per CTA, 4 KB of list
// each, so ~56 warps per SM keep the stores in flight (the earlier
// 4096-entry lists allowed 6).  The e2e C5 step (1M candidates, 1.6 GB of
// records written) lost ~0.3 ms of its 1.5 ms host-path overhead.
constexpr int kWriteWarps = 8;
constexpr int kTilChunk = 512;

__global__ void __launch_bounds__(kWriteWarps * 32) expand_write_kernel(
    const GsFunc* __restrict__ funcs, const GsDecision* __restrict__ parents, int64_t n, int S,
    const int32_t* __restrict__ step, GsTilingMenus m, const int64_t* __restrict__ offsets,
    GsDecision* __restrict__ out, int64_t out_cap, int32_t* __restrict__ owner, int* __restrict__ gerr) {
  __shared__ __align__(16) uint8_t til[kWriteWarps][kTilChunk][8];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t nwarps = (int64_t)gridDim.x * kWriteWarps;
  for (int64_t p = (int64_t)blockIdx.x * kWriteWarps + wib; p < n; p += nwarps) {
    const int64_t base = offsets[p], cnt = offsets[p + 1] - base;
    if (cnt <= 0 || cnt > kMaxTilings) continue;
    if (base + cnt > out_cap) {   // the caller's buffer is smaller than the step: write nothing past it
      if (lane == 0) atomicOr(gerr, 16);
      continue;
    }
    const int s = step[p];
    const GsDecision* par = parents + p * S;
    const GsFunc& fn = funcs[par[s].func];
    const int nd = fn.ndim;
    const uint4* src = reinterpret_cast<const uint4*>(par);
    for (int64_t k0 = 0; k0 < cnt; k0 += kTilChunk) {
      const int nt = (int)(cnt - k0 < kTilChunk ? cnt - k0 : kTilChunk);
      __syncwarp();
      if (lane == 0) {
        int64_t k = 0;
        enum_tilings(m, fn, [&](const int* sv, const int* tv) {
          if (k >= k0 && k < k0 + kTilChunk) {
            uint8_t* e = til[wib][k - k0];
            for (int d = 0; d < GS_MAX_NDIM; ++d) { e[d] = (uint8_t)sv[d]; e[4 + d] = (uint8_t)tv[d]; }
          }
          ++k;
        });
      }
      __syncwarp();
      uint4* dst = reinterpret_cast<uint4*>(out + (base + k0) * S);
      const int64_t total = (int64_t)nt * S;
      int t = lane / S, i = lane - t * S;   // (tiling, record) of flattened element j = lane
      for (int64_t j = lane; j < total; j += 32) {
        uint4 r = __ldg(src + i);
        if (i == s) {
          GsDecision d = *reinterpret_cast<const GsDecision*>(&r);
          d.flags = 3;
          for (int q = 0; q < nd; ++q) { d.serial[q] = til[wib][t][q]; d.thread[q] = til[wib][t][4 + q]; }
          r = *reinterpret_cast<const uint4*>(&d);
        }
        dst[j] = r;
        i += 32;
        while (i >= S) { i -= S; ++t; }
      }
      if (owner)
        for (int q = lane; q < nt; q += 32) owner[base + k0 + q] = (int32_t)p;
    }
  }
}

// ---------------------------------------------------------------------------
// Phase-1 expansion (search.py:204-220 `_phase1_candidates`): the placement
// menu of `func` in each parent (options.py:103-141
// `enumerate_compute_locations`, legality as loopnest.py:178-241
// `apply_decision`), fuse_at_block entries crossed with every serial tiling
// (options.py:144-162), parents in order, menus in reference order.
// Static per-func facts (output, inlinable, pointwise-called, cheap, the
// consumer lists) are packed at pipeline creation (P1Static).
// ---------------------------------------------------------------------------
constexpr int kP1MaxFuncs = 512;    // funcs per pipeline for the menus (per-thread local arrays)
constexpr int kP1MaxMenu = 64;      // menu entries per parent

__device__ int p1_kernel_of(const int8_t* kind, const int16_t* cons, int c, int nf) {
  for (int it = 0; it <= nf; ++it) {
    if (c < 0 || kind[c] < 0 || kind[c] == GS_INLINE) return -1;
    if (kind[c] == GS_ROOT) return c;
    c = cons[c];
  }
  return -1;
}

// The placement menu of `func` in a state (kind / consumer per func, -1 =
// unscheduled): entries kind | consumer << 8 in reference order, restricted
// to restrict_mask (search.py:208-210).  Returns the entry count, or -1 when
// it exceeds kP1MaxMenu.  Kept out of line: inlined into rand_sched_kernel,
// its bitmask arrays were given the caller's menu-array stack slots (the
// menu's first entry came back overwritten; memcheck saw local accesses out
// of bounds) with nvcc 12.9 -O3.
__device__ __noinline__ int p1_menu(const P1Static& st, int nf, int func, const int8_t* kind, const int16_t* cons,
                       int restrict_mask, int32_t* mp) {
  int m = 0;
  auto add = [&](int k, int c) {
    if (m < kP1MaxMenu) mp[m] = k | ((c & 0xFFFF) << 8);
    ++m;
  };
  const uint8_t fl = st.flags[func];
  if (fl & P1_OUTPUT) {
    add(GS_ROOT, 0xFFFF);
  } else if ((fl & P1_SINGLE_STAGE) && (fl & P1_POINTWISE_CALLED) && (fl & P1_INLINE_OK)) {
    add(GS_INLINE, 0xFFFF);
  } else {
    add(GS_ROOT, 0xFFFF);
    // effective consumers: non-inlined funcs reading func, through inlined ones
    // (breadth-first over bitmask frontiers: no per-thread stack)
    constexpr int NW = kP1MaxFuncs / 32;
    uint32_t eff[NW], seen[NW], front[NW];
    const int nw = (nf + 31) / 32;
    for (int w = 0; w < nw; ++w) { eff[w] = 0u; seen[w] = 0u; front[w] = 0u; }
    front[func >> 5] = 1u << (func & 31);
    for (bool more = true; more;) {
      more = false;
      for (int w = 0; w < nw; ++w) {
        uint32_t bits = front[w];
        front[w] = 0u;
        while (bits) {
          const int g = 32 * w + __ffs(bits) - 1;
          bits &= bits - 1;
          for (int q = st.cons_off[g]; q < st.cons_off[g + 1]; ++q) {
            const int c = st.cons[q];
            if (kind[c] == GS_INLINE) {
              if (!(seen[c >> 5] & (1u << (c & 31)))) {
                seen[c >> 5] |= 1u << (c & 31);
                front[c >> 5] |= 1u << (c & 31);
                more = true;
              }
            } else {
              eff[c >> 5] |= 1u << (c & 31);
            }
          }
        }
      }
    }
    int neff = 0;
    for (int w = 0; w < (nf + 31) / 32; ++w) neff += __popc(eff[w]);
    for (int r = 0; r < nf; ++r) {   // sorted(effective_consumers) = name order
      const int c = st.sorted[r];
      if (!(eff[c >> 5] & (1u << (c & 31)))) continue;
      if (kind[c] < 0) continue;   // not scheduled yet
      // fuse_at_block: target scheduled, not inlined, and every effective
      // consumer in the target's kernel; fuse_at_thread: the only consumer
      const bool target_ok = kind[c] != GS_INLINE;
      bool block_ok = target_ok;
      if (block_ok) {
        const int kern = p1_kernel_of(kind, cons, c, nf);
        for (int w = 0; w < (nf + 31) / 32 && block_ok; ++w) {
          uint32_t bits = eff[w];
          while (bits && block_ok) {
            const int o = 32 * w + __ffs(bits) - 1;
            bits &= bits - 1;
            if (p1_kernel_of(kind, cons, o, nf) != kern) block_ok = false;
          }
        }
      }
      if (block_ok) add(GS_FUSE_BLOCK, c);
      if (target_ok && neff == 1) add(GS_FUSE_THREAD, c);
    }
    if ((fl & P1_CHEAP) && (fl & P1_INLINE_OK)) add(GS_INLINE, 0xFFFF);
  }
  if (m > kP1MaxMenu) return -1;
  if (restrict_mask != 0xF) {
    int k = 0;
    for (int i = 0; i < m; ++i) if (restrict_mask & (1 << (mp[i] & 0xFF))) mp[k++] = mp[i];
    if (k == 0) {
      for (int i = 0; i < m; ++i) if ((mp[i] & 0xFF) == GS_ROOT) mp[k++] = mp[i];
    }
    m = k;
  }
  return m;
}

// one thread per parent: its menu and candidate count; ndec[p] = the
// parent's decision count (the new record's slot)
__global__ void p1_menu_kernel(const GsFunc* __restrict__ funcs, int nf, const P1Static st,
                               const GsDecision* __restrict__ parents, int64_t n, int S, int func, int restrict_mask,
                               int n_serial, int32_t* __restrict__ menu, uint8_t* __restrict__ nmenu,
                               int32_t* __restrict__ ndec, uint32_t* __restrict__ counts, int* __restrict__ gerr) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  int8_t kind[kP1MaxFuncs];
  int16_t cons[kP1MaxFuncs];
  for (int f = 0; f < nf; ++f) kind[f] = -1;
  int nd = 0;
  const GsDecision* par = parents + p * S;
  for (; nd < S && par[nd].func != 0xFFFF; ++nd) {
    const int f = par[nd].func;
    if (f >= nf) { atomicOr(gerr, 32); counts[p] = 0; nmenu[p] = 0; return; }
    kind[f] = (int8_t)par[nd].kind;
    cons[f] = par[nd].consumer == 0xFFFF ? (int16_t)-1 : (int16_t)par[nd].consumer;
  }
  ndec[p] = nd;
  // the new record needs a free slot, and func must be unscheduled (apply_decision)
  if (nd >= S || kind[func] >= 0) { atomicOr(gerr, 32); counts[p] = 0; nmenu[p] = 0; return; }
  int32_t* mp = menu + p * kP1MaxMenu;
  const int m = p1_menu(st, nf, func, kind, cons, restrict_mask, mp);
  if (m < 0) { atomicOr(gerr, 16); counts[p] = 0; nmenu[p] = 0; return; }
  uint32_t cnt = 0;
  for (int i = 0; i < m; ++i) cnt += (mp[i] & 0xFF) == GS_FUSE_BLOCK ? (uint32_t)n_serial : 1u;
  nmenu[p] = (uint8_t)m;
  counts[p] = cnt;
}

// one warp per parent: each candidate = the parent's records + the new one
__global__ void __launch_bounds__(kExpandWarps * 32) p1_write_kernel(
    const GsFunc* __restrict__ funcs, const GsDecision* __restrict__ parents, int64_t n, int S, int func,
    GsTilingMenus m, const int32_t* __restrict__ menu, const uint8_t* __restrict__ nmenu,
    const int32_t* __restrict__ ndec, const int64_t* __restrict__ offsets, GsDecision* __restrict__ out,
    int64_t out_cap, int32_t* __restrict__ owner, int* __restrict__ gerr) {
  __shared__ uint8_t ser[kExpandWarps][kMaxTilings][4];
  __shared__ int nser_s[kExpandWarps];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const GsFunc& fn = funcs[func];
  if (lane == 0) {   // serial tilings of func (enumerate_serial_tilings order)
    const int nd = fn.ndim;
    int so[GS_MAX_NDIM][16], sn[GS_MAX_NDIM];
    for (int d = 0; d < nd; ++d) sn[d] = serial_opts(m, fn.extent[d], so[d]);
    int idx[GS_MAX_NDIM] = {0, 0, 0, 0}, k = 0;
    for (;;) {
      int64_t prod = 1;
      for (int d = 0; d < nd; ++d) prod *= so[d][idx[d]];
      if (prod <= m.unroll_budget && k < kMaxTilings) {
        for (int d = 0; d < GS_MAX_NDIM; ++d) ser[wib][k][d] = (uint8_t)(d < nd ? so[d][idx[d]] : 0);
        ++k;
      }
      int d = nd - 1;
      while (d >= 0 && ++idx[d] == sn[d]) { idx[d] = 0; --d; }
      if (d < 0) break;
    }
    nser_s[wib] = k;
  }
  __syncwarp();
  const int nser = nser_s[wib];
  const int64_t nwarps = (int64_t)gridDim.x * kExpandWarps;
  for (int64_t p = (int64_t)blockIdx.x * kExpandWarps + wib; p < n; p += nwarps) {
    const int64_t base = offsets[p], cnt = offsets[p + 1] - base;
    if (cnt <= 0) continue;
    if (base + cnt > out_cap) { if (lane == 0) atomicOr(gerr, 16); continue; }
    const uint4* src = reinterpret_cast<const uint4*>(parents + p * S);
    const int slot = ndec[p];
    int64_t t = 0;
    for (int e = 0; e < nmenu[p]; ++e) {
      const int ent = menu[p * kP1MaxMenu + e];
      const int k = ent & 0xFF, c = (ent >> 8) & 0xFFFF;
      const int reps = k == GS_FUSE_BLOCK ? nser : 1;
      for (int r = 0; r < reps; ++r, ++t) {
        uint4* dst = reinterpret_cast<uint4*>(out + (base + t) * S);
        for (int i = lane; i < S; i += 32) {
          uint4 v = __ldg(src + i);
          if (i == slot) {
            GsDecision d;
            d.func = (uint16_t)func;
            d.consumer = (uint16_t)c;
            d.kind = (uint8_t)k;
            d.flags = k == GS_FUSE_BLOCK ? 1 : 0;
            for (int q = 0; q < GS_MAX_NDIM; ++q) { d.serial[q] = k == GS_FUSE_BLOCK ? ser[wib][r][q] : 0; d.thread[q] = 0; }
            d.pad = 0;
            v = *reinterpret_cast<const uint4*>(&d);
          }
          dst[i] = v;
        }
        if (owner && lane == 0) owner[base + t] = (int32_t)p;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Random complete schedules (the reference test-suite's `_random_schedule`,
// tests/test_acceptance.py:136-160): candidate i walks the schedulable funcs
// with its own default_rng((seed, first + i)) — a menu draw per func, a
// serial draw for fuse_at_block, then a serial and a thread tiling draw per
// compute_root func — exactly the reference's draw sequence, so each
// candidate equals `_random_schedule(graph, default_rng((seed, i)))`.
// ---------------------------------------------------------------------------
__device__ int nth_serial(const GsTilingMenus& m, const GsFunc& fn, int want, int* sv) {
  const int nd = fn.ndim;
  int so[GS_MAX_NDIM][16], sn[GS_MAX_NDIM];
  for (int d = 0; d < nd; ++d) sn[d] = serial_opts(m, fn.extent[d], so[d]);
  int idx[GS_MAX_NDIM] = {0, 0, 0, 0}, k = 0;
  for (;;) {
    int64_t prod = 1;
    for (int d = 0; d < nd; ++d) prod *= so[d][idx[d]];
    if (prod <= m.unroll_budget) {
      if (k == want && sv) for (int d = 0; d < nd; ++d) sv[d] = so[d][idx[d]];
      ++k;
    }
    int d = nd - 1;
    while (d >= 0 && ++idx[d] == sn[d]) { idx[d] = 0; --d; }
    if (d < 0) break;
  }
  return k;
}

// enumerate_thread_tilings(post) (options.py:165-183): count, and the
// want-th vector (last dim fastest)
__device__ int nth_thread(const GsTilingMenus& m, const int* post, int nd, int want, int* tv) {
  int inner = -1;
  for (int d = 0; d < nd; ++d) if (post[d] >= 16) { inner = d; break; }
  if (inner < 0) inner = 0;
  int to[GS_MAX_NDIM][16], tn[GS_MAX_NDIM];
  int total = 1;
  for (int d = 0; d < nd; ++d) { tn[d] = thread_opts(m, post[d], d == inner, to[d]); total *= tn[d]; }
  if (tv && want < total) {
    int r = want;
    for (int d = nd - 1; d >= 0; --d) { tv[d] = to[d][r % tn[d]]; r /= tn[d]; }
  }
  return total;
}

__global__ void rand_sched_kernel(const GsFunc* __restrict__ funcs, int nf, const P1Static st,
                                  const int32_t* __restrict__ order, int n_order, GsTilingMenus m, uint64_t seed,
                                  int64_t first, int64_t n, int S, GsDecision* __restrict__ out,
                                  int* __restrict__ gerr) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  Pcg64 g;
  seed_pair(g, seed, (uint64_t)(first + c));
  int8_t kind[kP1MaxFuncs];
  int16_t cons[kP1MaxFuncs];
  int16_t rec[kP1MaxFuncs];
  for (int f = 0; f < nf; ++f) kind[f] = -1;
  GsDecision* o = out + c * S;
  int32_t mp[kP1MaxMenu];
  int nd = 0;
  for (int i = 0; i < n_order; ++i) {
    const int func = order[i];
    const int len = p1_menu(st, nf, func, kind, cons, 0xF, mp);
    if (len <= 0 || nd >= S) { atomicOr(gerr, len < 0 ? 16 : 32); return; }
    const uint32_t pick = g.integers((uint32_t)len);
    const int e = mp[pick];

    const int k = e & 0xFF, tgt = (e >> 8) & 0xFFFF;
    GsDecision d;
    d.func = (uint16_t)func;
    d.kind = (uint8_t)k;
    d.consumer = (k == GS_FUSE_BLOCK || k == GS_FUSE_THREAD) ? (uint16_t)tgt : (uint16_t)0xFFFF;
    d.flags = 0;
    d.pad = 0;
    for (int q = 0; q < GS_MAX_NDIM; ++q) { d.serial[q] = 0; d.thread[q] = 0; }
    if (k == GS_FUSE_BLOCK) {
      int sv[GS_MAX_NDIM];
      const int ns = nth_serial(m, funcs[func], -1, nullptr);
      nth_serial(m, funcs[func], (int)g.integers((uint32_t)ns), sv);
      for (int q = 0; q < funcs[func].ndim; ++q) d.serial[q] = (uint8_t)sv[q];
      d.flags = 1;
    }
    o[nd] = d;
    rec[func] = (int16_t)nd++;
    kind[func] = (int8_t)k;
    cons[func] = d.consumer == 0xFFFF ? (int16_t)-1 : (int16_t)d.consumer;
  }
  for (int i = 0; i < n_order; ++i) {   // deferred root tilings, scheduling order
    const int func = order[i];
    if (kind[func] != GS_ROOT) continue;
    const GsFunc& fn = funcs[func];
    int sv[GS_MAX_NDIM], tv[GS_MAX_NDIM], post[GS_MAX_NDIM];
    const int ns = nth_serial(m, fn, -1, nullptr);
    nth_serial(m, fn, (int)g.integers((uint32_t)ns), sv);
    for (int q = 0; q < fn.ndim; ++q) post[q] = (fn.extent[q] + sv[q] - 1) / sv[q];
    const int nt = nth_thread(m, post, fn.ndim, -1, nullptr);
    nth_thread(m, post, fn.ndim, (int)g.integers((uint32_t)nt), tv);
    GsDecision& d = o[rec[func]];
    for (int q = 0; q < fn.ndim; ++q) { d.serial[q] = (uint8_t)sv[q]; d.thread[q] = (uint8_t)tv[q]; }
    d.flags = 3;
  }
  for (int i = nd; i < S; ++i) {
    GsDecision d;
    d.func = 0xFFFF; d.consumer = 0xFFFF; d.kind = 0; d.flags = 0; d.pad = 0;
    for (int q = 0; q < GS_MAX_NDIM; ++q) { d.serial[q] = 0; d.thread[q] = 0; }
    o[i] = d;
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
    const int64_t want = (n + kWriteWarps - 1) / kWriteWarps;
    const int grid = (int)(want < (int64_t)num_sms * 8 ? want : (int64_t)num_sms * 8);
    expand_write_kernel<<<grid, kWriteWarps * 32, 0, st>>>(funcs, parents, n, S, step, m, offsets, out, out_cap,
                                                           owner, gerr);
    g_launch_count++;
  }
  return 0;
}

// number of serial tilings of a func (enumerate_serial_tilings), host side
int serial_count(const GsTilingMenus& m, const GsFunc& fn) {
  const int nd = fn.ndim;
  int so[GS_MAX_NDIM][16], sn[GS_MAX_NDIM];
  for (int d = 0; d < nd; ++d) sn[d] = serial_opts(m, fn.extent[d], so[d]);
  int idx[GS_MAX_NDIM] = {0, 0, 0, 0}, k = 0;
  for (;;) {
    int64_t prod = 1;
    for (int d = 0; d < nd; ++d) prod *= so[d][idx[d]];
    if (prod <= m.unroll_budget) ++k;
    int d = nd - 1;
    while (d >= 0 && ++idx[d] == sn[d]) { idx[d] = 0; --d; }
    if (d < 0) break;
  }
  return k;
}

// The menu kernels keep per-thread state in local arrays (a few KB of stack
// frame, p1_menu's in an out-of-line call): make sure the per-thread stack
// limit covers the kernel's local size.  Raised once, before first use.
static int ensure_stack(const void* kernel) {
  cudaFuncAttributes a;
  if (cudaFuncGetAttributes(&a, kernel) != cudaSuccess) return -1;
  size_t cur = 0;
  if (cudaDeviceGetLimit(&cur, cudaLimitStackSize) != cudaSuccess) return -1;
  const size_t need = (a.localSizeBytes + 1023) & ~(size_t)1023;
  if (cur < need && cudaDeviceSetLimit(cudaLimitStackSize, need) != cudaSuccess) return -1;
  return 0;
}

int64_t phase1_workspace_bytes(int64_t n) {
  if (n < 1) n = 1;
  return expand_workspace_bytes(n) + (int64_t)(align256(4 * n * kP1MaxMenu) + align256(n) + align256(4 * n));
}

int launch_phase1(const GsFunc* funcs, int nf, const P1Static& st, const GsDecision* parents, int64_t n, int S,
                  int func, int restrict_mask, const GsTilingMenus& m, int n_serial, int64_t* offsets, void* ws,
                  int64_t ws_bytes, GsDecision* out, int64_t out_cap, int32_t* owner, int* gerr, int num_sms,
                  cudaStream_t st_) {
  if (n <= 0) { cudaMemsetAsync(offsets, 0, sizeof(int64_t), st_); return 0; }
  if (n > (int64_t)1 << 20 || nf > kP1MaxFuncs) return -1;
  if (phase1_workspace_bytes(n) > ws_bytes) return -2;
  uint8_t* w = static_cast<uint8_t*>(ws);
  uint32_t* counts = reinterpret_cast<uint32_t*>(w);
  uint32_t* incl = reinterpret_cast<uint32_t*>(w + align256(4 * n));
  uint32_t* sums = reinterpret_cast<uint32_t*>(w + 2 * align256(4 * n));
  uint8_t* rest = w + expand_workspace_bytes(n);
  int32_t* menu = reinterpret_cast<int32_t*>(rest);
  uint8_t* nmenu = rest + align256(4 * n * kP1MaxMenu);
  int32_t* ndec = reinterpret_cast<int32_t*>(nmenu + align256(n));
  static bool stack_ok = false;
  if (!stack_ok) { if (ensure_stack((const void*)p1_menu_kernel)) return -3; stack_ok = true; }
  p1_menu_kernel<<<(unsigned)((n + 63) / 64), 64, 0, st_>>>(funcs, nf, st, parents, n, S, func, restrict_mask,
                                                            n_serial, menu, nmenu, ndec, counts, gerr);
  scan_u32(counts, incl, n, nullptr, true, sums, nullptr, st_);
  expand_offsets_kernel<<<(unsigned)((n + 1 + 255) / 256), 256, 0, st_>>>(incl, n, offsets);
  g_launch_count += 2;
  if (out) {
    const int64_t want = (n + kExpandWarps - 1) / kExpandWarps;
    const int grid = (int)(want < (int64_t)num_sms * 16 ? want : (int64_t)num_sms * 16);
    p1_write_kernel<<<grid, kExpandWarps * 32, 0, st_>>>(funcs, parents, n, S, func, m, menu, nmenu, ndec, offsets,
                                                          out, out_cap, owner, gerr);
    g_launch_count++;
  }
  return 0;
}

int launch_random_schedules(const GsFunc* funcs, int nf, const P1Static& st, const int32_t* order, int n_order,
                            const GsTilingMenus& m, uint64_t seed, int64_t first, int64_t n, int S, GsDecision* out,
                            int* gerr, cudaStream_t st_) {
  if (n <= 0) return 0;
  if (nf > kP1MaxFuncs) return -1;
  static bool stack_ok = false;
  if (!stack_ok) { if (ensure_stack((const void*)rand_sched_kernel)) return -3; stack_ok = true; }
  rand_sched_kernel<<<(unsigned)((n + 63) / 64), 64, 0, st_>>>(funcs, nf, st, order, n_order, m, seed, first, n, S,
                                                               out, gerr);
  g_launch_count++;
  return 0;
}

}  // namespace gs
