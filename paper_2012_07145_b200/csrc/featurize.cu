// K1 — per-candidate resolve + 56 schedule features per stage row + prune
// (reference featurize.py:275-617, resolve.py:207-425, options.py:200-255).
//
// One CTA per SM (up to 12 warps); every warp is a scorer with its own slice
// of shared memory (capacity-sized arrays optionally in an L1-cached global
// scratch: spill levels), taking work from a global counter:
//   * the candidate-independent pipeline descriptor is staged ONCE per CTA
//     into shared memory with a bulk async copy (TMA `cp.async.bulk`, SASS
//     UBLKCP) completing on an mbarrier;
//   * per candidate the warp loads its 16-byte decision records with 128-bit
//     loads, diffs them against the previous candidate it scored (siblings
//     of a beam step share their decision structure), re-resolves only the
//     funcs whose dependency mask meets the changed records, computes the
//     prune verdict warp-parallel, and recomputes only the feature rows whose
//     own / host / kernel / producer-layout records changed (the rest are
//     bit-identical copies, or — reuse mode 2 — not written at all);
//   * the CTA's warps run in lockstep: phase A (records, diff, resolve,
//     prune, row flags) for every warp's candidate, a CTA barrier, then the
//     feature rows, and a barrier again, so the SM streams one phase's code
//     at a time;
//   * large batches of long sibling runs use a two-phase schedule: run heads
//     first (each saves the persistent prefix of its warp state to its run's
//     slot in HBM), then 5-candidate sibling slices, claimed 12 at a time per
//     CTA, that resume from their head's state, so a run splits across warps
//     without re-resolving; the sibling launch pools the CTA's dirty rows in
//     row-major order (row q of every warp's candidate, then q + 1), each
//     taken by the next free warp;
//   * warp-instruction transaction counts (featurize.py:173-196, 508-571)
//     use the residue invariance of the counts (global: address constant mod
//     32 B; shared: mod the 4 B bank width): residue histograms in registers,
//     interval sums over one prefix scan for monotonic warps, one evaluation
//     per shift class for regular thread tiles, and __match_any_sync /
//     __ballot_sync for the rest.
// See DESIGN.md "K1 featurize" for the roofline reading.
#include "gs_internal.cuh"
#include "scan.cuh"
#include <cstddef>
#include <cuda/std/cstdint>

namespace gs {

struct Frame { int16_t owner, root; int32_t cur, end; int16_t plen, pad; int64_t vol; };

struct ICall { int16_t root, iname, stage, pad; int64_t vol; };   // per (root stage, inline func)

// Per-warp row scratch.  The generic counters (machines other than 32 B
// transactions / 32 x 4 B banks) need residue tables of up to kMaxM entries;
// they sit at the end and are allocated only for such machines, which keeps
// the default machine's warp slice small enough for ten scorer warps.
struct WarpScr {
  double feat[GS_NUM_FEATURES];
  unsigned long long H[32], S[32];      // residue_hist scratch (Q <= 32)
  unsigned long long acc[4][3][2];      // box x tier x (bytes, lines)
  int16_t rl[kRowReads];
  int8_t grp[kRowReads];
  int8_t gtier[kRowReads];
  int16_t gprod[kRowReads];
  int ngroups;
  int nr;
  // generic machines only
  unsigned long long GH[kMaxM], GS[kMaxM], T[kMaxM];
  int16_t nz[kMaxM];
};
constexpr int kScrDefaultBytes = (int)offsetof(WarpScr, GH);

struct Misc {
  int ndec, nreads, npath, nrows, nicall, err, verdict, same_struct, prev_valid, ndirty, ngeo, incr;
  int64_t ni;          // structure: sum of scheduled funcs' domain volumes (prune rule 1)
};

constexpr int kMaxMaskWords = 8;   // incremental resolve for pipelines of <= 256 funcs

template <int ND>
struct K1 {
  const GsFunc* F;
  const GsStage* ST;
  const GsAccess* A;
  const PipeDev* P;
  GsDecision* dec;   // current decision records
  int16_t* didx;
  CF<ND>* cf;        // current geometry
  RRead* rd;
  int16_t* path;
  int32_t* rdb;      // [2*ns]: begin,end of reads per global stage
  int32_t* rows;
  Frame* stack;
  int64_t* volacc;
  int16_t* touched;
  ICall* icall;
  int32_t* srcb;     // [nf+1] CSR: reads by producer
  int16_t* srcl;     // [rcap]
  int32_t* rdepb;    // [R+1] CSR: funcs (besides host/kernel) a row depends on
  int16_t* rdep;     // [rcap + nf]
  uint8_t* dirty;    // [nf]
  int16_t* rowlist;  // [R] rows to recompute this candidate
  // incremental resolve (structure-time metadata + per-candidate flags)
  int16_t* kern;     // [nf] kernel owner of each non-inline func (kernel_of)
  uint32_t* dm;      // [nf][mw] funcs whose decision records f's geometry depends on
  uint32_t* cmask;   // [mw] funcs whose decision record changed vs the previous candidate
  int32_t* kmb;      // [nf+1] CSR: fused members of each kernel owner
  int16_t* kml;      // [nf]
  int32_t* icb;      // [nf+1] CSR: icall entries per inline func (icall order)
  int16_t* icl;      // [pcap]
  int16_t* dlist;    // [nf] decision indices whose geometry is recomputed
  uint8_t* gdirty;   // [nf] geometry recomputed this candidate
  uint8_t* kdirty;   // [nf] kernel aggregates recomputed this candidate
  Misc* misc;
  int mw;            // mask words (0 = incremental resolve off)
  bool track;        // k.cf holds the previous candidate's geometry: flag changed records
  int rcap, pcap;
  int* gerr;
};

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

__device__ __forceinline__ int64_t wmin64(int64_t v) {
  for (int o = 16; o; o >>= 1) { int64_t u = __shfl_xor_sync(0xffffffffu, v, o); v = u < v ? u : v; }
  return v;
}
__device__ __forceinline__ int64_t wmax64(int64_t v) {
  for (int o = 16; o; o >>= 1) { int64_t u = __shfl_xor_sync(0xffffffffu, v, o); v = u > v ? u : v; }
  return v;
}

__device__ __noinline__ int64_t div64_slow(int64_t a, int64_t b) { return a / b; }
// a / b for a >= 0, b > 0: 32-bit division when both fit (all real extents)
__device__ __forceinline__ int64_t udiv(int64_t a, int64_t b) {
  if (((uint64_t)a | (uint64_t)b) <= 0x7FFFFFFFull) return (int64_t)((uint32_t)a / (uint32_t)b);
  return div64_slow(a, b);
}

template <int ND>
__device__ __forceinline__ int64_t prod_ext(const CF<ND>& c) {
  int64_t p = 1;
#pragma unroll
  for (int d = 0; d < ND; ++d) p *= c.ext[d];
  return p;
}
template <int ND>
__device__ __forceinline__ int64_t alloc_of(const CF<ND>& c) {
  if (c.tier == T_NONE) return 0;
  int64_t p = 1;
#pragma unroll
  for (int d = 0; d < ND; ++d) p *= (int64_t)c.rhi[d] - c.rlo[d] + 1;
  return p;
}
template <int ND>
__device__ __forceinline__ void block_box(const CF<ND>& c, int32_t* lo, int32_t* hi) {
  // resolve.py:112-122
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    if (c.kind == K_ROOT) { lo[d] = 0; hi[d] = c.ctx[d] * c.coeff[d] - 1; }   // thread*serial
    else if (c.kind == K_BLOCK) { lo[d] = c.rlo[d]; hi[d] = c.rhi[d]; }
    else { lo[d] = c.base[d]; hi[d] = c.base[d] + (c.ctx[d] - 1) * c.coeff[d] + c.ext[d] - 1; }
  }
}

// chain box of [lo,hi] through a path of accesses, dimension d
__device__ __forceinline__ void chain_iv(const GsAccess* A, const int16_t* p, int plen, int d,
                                         int64_t& a, int64_t& b) {
  #pragma unroll 1
  for (int k = 0; k < plen; ++k) {
    const GsAccess& x = A[p[k]];
    a = a * x.s[d] + x.lo[d];
    b = b * x.s[d] + x.hi[d];
  }
}

// ---------------------------------------------------------------------------
// resolve (warp 0), split in two:
//   structure — depends only on (func, kind, consumer) of each decision:
//               expanded reads + chain paths, rows, inline call volumes per
//               (root stage, inline func), producer->reads and row-dependency
//               CSRs; rebuilt only when the structure changes;
//   geometry  — per-func padded-tile geometry (needs tilings), kernel
//               aggregates, inline totals / primaries.
// ---------------------------------------------------------------------------
template <int ND>
__device__ int8_t tier_of_producer(const K1<ND>& k, int p) {
  int di = k.didx[p];
  if (di < 0 || k.F[p].is_external) return T_GLOBAL;
  int kind = k.dec[di].kind;
  return kind == GS_ROOT ? T_GLOBAL : kind == GS_FUSE_BLOCK ? T_SHARED : T_REGISTER;
}

// Depth-first inline substitution of one stage (resolve.py:167-200): emits
// the reads and accumulates inline call volumes (volacc, first-touch order).
template <int ND>
__device__ void expand_stage(K1<ND>& k, int root, int gstage, int& ntouched) {
  Misc& m = *k.misc;
  int16_t* pfx = k.touched + k.P->nf;   // path prefix buffer (nf + 1 entries)
  const GsStage& st = k.ST[gstage];
  k.stack[0] = Frame{(int16_t)root, (int16_t)root, st.access_begin, st.access_begin + st.n_access, 0, 0, 1};
  int sp = 1;
  while (sp > 0) {
    Frame& fr = k.stack[sp - 1];
    if (fr.cur == fr.end) { --sp; continue; }
    int a = fr.cur++;
    pfx[fr.plen] = (int16_t)a;
    int p = k.A[a].producer;
    int di = k.didx[p];
    if (di >= 0 && k.dec[di].kind == GS_INLINE) {
      int64_t vol = fr.vol * (int64_t)k.A[a].window;
      if (k.volacc[p] == 0) k.touched[ntouched++] = (int16_t)p;
      k.volacc[p] += vol;
      if (sp >= k.P->nf + 1) { m.err |= E_STACK; return; }
      const GsStage& is = k.ST[k.F[p].stage_begin];
      k.stack[sp] = Frame{(int16_t)p, fr.root, is.access_begin, is.access_begin + is.n_access,
                          (int16_t)(fr.plen + 1), 0, vol};
      ++sp;
    } else {
      int plen = fr.plen + 1;
      if (m.nreads >= k.rcap) { m.err |= E_READS; return; }
      if (m.npath + plen > k.pcap || plen > 255) { m.err |= E_PATHS; return; }
      RRead r;
      r.owner = fr.owner; r.producer = (int16_t)p; r.root = fr.root; r.tier = tier_of_producer(k, p);
      r.pad = 0;
      r.plen = (uint8_t)plen; r.pbeg = (uint16_t)m.npath;
      for (int i = 0; i < plen; ++i) k.path[m.npath + i] = pfx[i];
      m.npath += plen;
      k.rd[m.nreads++] = r;
    }
  }
}

// lane 0
template <int ND>
__device__ __noinline__ void resolve_structure(K1<ND>& k) {
  Misc& m = *k.misc;
  const int nf = k.P->nf;
  m.nreads = 0; m.npath = 0; m.nicall = 0;
  for (int f = 0; f < nf; ++f) k.volacc[f] = 0;
  for (int i = 0; i < m.ndec && !m.err; ++i) {
    const GsDecision& d = k.dec[i];
    if (d.kind == GS_INLINE) continue;
    const GsFunc& fn = k.F[d.func];
    for (int s = 0; s < fn.n_stages && !m.err; ++s) {
      int gsid = fn.stage_begin + s;
      int nt = 0;
      k.rdb[2 * gsid] = m.nreads;
      expand_stage(k, d.func, gsid, nt);
      k.rdb[2 * gsid + 1] = m.nreads;
      for (int t = 0; t < nt; ++t) {
        int iname = k.touched[t];
        if (m.nicall >= k.pcap) { m.err |= E_PATHS; break; }
        k.icall[m.nicall++] = ICall{(int16_t)d.func, (int16_t)iname, (int16_t)s, 0, k.volacc[iname]};
        k.volacc[iname] = 0;
      }
    }
  }
  if (m.err) return;
  // reads grouped by producer, read order kept (CSR)
  for (int f = 0; f <= nf; ++f) k.srcb[f] = 0;
  for (int j = 0; j < m.nreads; ++j) k.srcb[k.rd[j].producer + 1]++;
  for (int f = 0; f < nf; ++f) k.srcb[f + 1] += k.srcb[f];
  for (int f = 0; f < nf; ++f) k.volacc[f] = k.srcb[f];   // fill cursors (reuse scratch)
  for (int j = 0; j < m.nreads; ++j) k.srcl[k.volacc[k.rd[j].producer]++] = (int16_t)j;
  for (int f = 0; f < nf; ++f) k.volacc[f] = 0;
  // rows: non-inline decision order (every stage), then inline (featurize.py:292-303)
  int nr = 0;
  for (int i = 0; i < m.ndec; ++i) {
    const GsDecision& d = k.dec[i];
    if (d.kind == GS_INLINE) continue;
    for (int s = 0; s < k.F[d.func].n_stages; ++s) k.rows[nr++] = (d.func << 8) | s;
  }
  for (int i = 0; i < m.ndec; ++i)
    if (k.dec[i].kind == GS_INLINE) k.rows[nr++] = (k.dec[i].func << 8);
  m.nrows = nr;
  // per-row dependencies besides its own func / host / kernel: producers of
  // the reads it owns and its fuse_at_thread children.  The children come
  // from a consumer CSR (kmb offsets, kml list, icb cursors: scratch here,
  // rebuilt as the kernel CSRs below), an inline row's reads from the root
  // stages it was expanded into (its icall entries), so the build is linear
  // in decisions + reads (it was rows x decisions and inline rows x reads:
  // half of the run-head launch).
  for (int f = 0; f <= nf; ++f) k.kmb[f] = 0;
  for (int i = 0; i < m.ndec; ++i)
    if (k.dec[i].kind == GS_FUSE_THREAD) k.kmb[k.dec[i].consumer + 1]++;
  for (int f = 0; f < nf; ++f) k.kmb[f + 1] += k.kmb[f];
  for (int f = 0; f < nf; ++f) k.icb[f] = k.kmb[f];
  for (int i = 0; i < m.ndec; ++i)
    if (k.dec[i].kind == GS_FUSE_THREAD) k.kml[k.icb[k.dec[i].consumer]++] = (int16_t)k.dec[i].func;
  int nd = 0;
  const int cap = k.rcap + nf;
  for (int r = 0; r < nr; ++r) {
    k.rdepb[r] = nd;
    const int f = k.rows[r] >> 8, si = k.rows[r] & 255;
    if (k.dec[k.didx[f]].kind == GS_INLINE) {
      for (int e = 0; e < m.nicall; ++e) {
        if (k.icall[e].iname != f) continue;
        const int g = k.F[k.icall[e].root].stage_begin + k.icall[e].stage;
        for (int j = k.rdb[2 * g]; j < k.rdb[2 * g + 1]; ++j)
          if (k.rd[j].owner == f && nd < cap) k.rdep[nd++] = k.rd[j].producer;
      }
    } else {
      const int g = k.F[f].stage_begin + si;
      for (int j = k.rdb[2 * g]; j < k.rdb[2 * g + 1]; ++j)
        if (k.rd[j].owner == f && nd < cap) k.rdep[nd++] = k.rd[j].producer;
      for (int q = k.kmb[f]; q < k.kmb[f + 1] && nd < cap; ++q) k.rdep[nd++] = k.kml[q];
    }
  }
  k.rdepb[nr] = nd;

  // prune rule 1 denominator: sum of scheduled funcs' domains (options.py:215-222)
  int64_t ni = 0;
  for (int i = 0; i < m.ndec; ++i) {
    const GsFunc& fn = k.F[k.dec[i].func];
    int64_t dom = 1;
    for (int dd = 0; dd < fn.ndim; ++dd) dom *= fn.extent[dd];
    ni += dom;
  }
  m.ni = ni;

  // ---- metadata for incremental sibling resolve --------------------------
  // kernel owner of every non-inline func: itself for roots, the owner of
  // its first fusion source's root otherwise (= cg0.kernel in geometry)
  for (int f = 0; f < nf; ++f) k.kern[f] = -1;
  for (int i = 0; i < m.ndec; ++i) {
    const GsDecision& d = k.dec[i];
    if (d.kind == GS_INLINE) continue;
    if (d.kind == GS_ROOT) { k.kern[d.func] = (int16_t)d.func; continue; }
    for (int q = k.srcb[d.func]; q < k.srcb[d.func + 1]; ++q)
      if (k.didx[k.rd[k.srcl[q]].root] < i) { k.kern[d.func] = k.kern[k.rd[k.srcl[q]].root]; break; }
  }
  // fused members per kernel owner (decision order)
  for (int f = 0; f <= nf; ++f) k.kmb[f] = 0;
  for (int i = 0; i < m.ndec; ++i) {
    const GsDecision& d = k.dec[i];
    if ((d.kind == GS_FUSE_BLOCK || d.kind == GS_FUSE_THREAD) && k.kern[d.func] >= 0) k.kmb[k.kern[d.func] + 1]++;
  }
  for (int f = 0; f < nf; ++f) k.kmb[f + 1] += k.kmb[f];
  for (int f = 0; f < nf; ++f) k.volacc[f] = k.kmb[f];
  for (int i = 0; i < m.ndec; ++i) {
    const GsDecision& d = k.dec[i];
    if ((d.kind == GS_FUSE_BLOCK || d.kind == GS_FUSE_THREAD) && k.kern[d.func] >= 0)
      k.kml[k.volacc[k.kern[d.func]]++] = (int16_t)d.func;
  }
  // icall entries per inline func, icall order kept (first max wins)
  for (int f = 0; f <= nf; ++f) k.icb[f] = 0;
  for (int e = 0; e < m.nicall; ++e) k.icb[k.icall[e].iname + 1]++;
  for (int f = 0; f < nf; ++f) k.icb[f + 1] += k.icb[f];
  for (int f = 0; f < nf; ++f) k.volacc[f] = k.icb[f];
  for (int e = 0; e < m.nicall; ++e) k.icl[k.volacc[k.icall[e].iname]++] = (int16_t)e;
  for (int f = 0; f < nf; ++f) k.volacc[f] = 0;
  // dependency masks: dm[f] = decision records f's geometry record depends
  // on (transitively), in resolve order; geometry only flows forward
  const int mw = k.mw;
  if (mw > 0) {
    uint32_t* dm = k.dm;
    for (int j = 0; j < nf * mw; ++j) dm[j] = 0;
    auto orm = [&](int dst, int src) { for (int w = 0; w < mw; ++w) dm[dst * mw + w] |= dm[src * mw + w]; };
    for (int i = 0; i < m.ndec; ++i) {
      const GsDecision& d = k.dec[i];
      if (d.kind == GS_INLINE) continue;
      const int f = d.func;
      dm[f * mw + (f >> 5)] |= 1u << (f & 31);
      if (d.kind == GS_ROOT) continue;
      for (int q = k.srcb[f]; q < k.srcb[f + 1]; ++q) {
        const int r = k.rd[k.srcl[q]].root;
        if (k.didx[r] < i) orm(f, r);
      }
      if (k.kern[f] >= 0) orm(f, k.kern[f]);
    }
    for (int f = 0; f < nf; ++f) {
      if (!(k.F[f].is_external || k.didx[f] < 0)) continue;
      for (int q = k.srcb[f]; q < k.srcb[f + 1]; ++q) orm(f, k.rd[k.srcl[q]].root);
    }
    for (int i = 0; i < m.ndec; ++i) {
      const GsDecision& d = k.dec[i];
      if (d.kind != GS_INLINE) continue;
      const int f = d.func;
      dm[f * mw + (f >> 5)] |= 1u << (f & 31);
      for (int q = k.icb[f]; q < k.icb[f + 1]; ++q) {
        const int r = k.icall[k.icl[q]].root;
        orm(f, r);
        if (k.kern[r] >= 0) orm(f, k.kern[r]);
      }
    }
  }
}

template <int ND>
__device__ __forceinline__ void zero_cf(CF<ND>& c) {
  int32_t* w = reinterpret_cast<int32_t*>(&c);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(CF<ND>) / 4); ++i) w[i] = 0;
}

// Store a func's geometry record (one lane).  When the buffer holds the
// previous candidate's geometry, a record that actually changes marks the
// func dirty: rows depending only on unchanged records are bit-identical.
// dirty bits: 1 = any field changed, 2 = the allocation layout (tier,
// realization region) changed — all a consumer's row reads of a producer
// or of a fuse_at_thread child (strides, allocation bytes); 4 = the
// kernel-owner aggregates (blocks, threads per block, shared bytes) — all
// a row reads of its host's kernel record.
template <int ND>
__device__ __forceinline__ void cf_store(K1<ND>& k, int f, const CF<ND>& c) {
  static_assert(sizeof(CF<ND>) % 16 == 0, "CF records are copied as 16-byte vectors");
  constexpr int NV = (int)(sizeof(CF<ND>) / 16);
  int4* dst = reinterpret_cast<int4*>(&k.cf[f]);
  const int4* src = reinterpret_cast<const int4*>(&c);
  if (k.track) {
    const CF<ND>& o = k.cf[f];
    bool l = o.tier != c.tier;
#pragma unroll
    for (int dd = 0; dd < ND; ++dd) l |= o.rlo[dd] != c.rlo[dd] || o.rhi[dd] != c.rhi[dd];
    bool d = false;
#pragma unroll
    for (int w = 0; w < NV; ++w) {
      const int4 a = dst[w], b = src[w];
      d |= a.x != b.x || a.y != b.y || a.z != b.z || a.w != b.w;
    }
    const bool ag = o.n_blocks != c.n_blocks || o.k_threads != c.k_threads || o.k_shared != c.k_shared;
    k.dirty[f] |= (uint8_t)(d | (l << 1) | (ag << 2));
  }
#pragma unroll
  for (int w = 0; w < NV; ++w) dst[w] = src[w];
}

// Geometry of the non-inline decision i (resolve.py:232-333); warp-wide.
// Kernel aggregates (threads per block = max, shared bytes = sum over the
// kernel's members) are NOT accumulated here but by kernel_aggregates():
// no member's geometry reads them, so the result is the same and a
// sibling that changes one member recomputes only its kernel's sums.
template <int ND>
__device__ __forceinline__ bool geometry_one(K1<ND>& k, int i) {
  const int lane = lane_id();
  Misc& m = *k.misc;
  const GsDecision d = k.dec[i];
  const int f = d.func;
  const GsFunc& fn = k.F[f];
  CF<ND> c;
  zero_cf(c);
  c.consumer = (d.kind == GS_ROOT) ? -1 : (int16_t)d.consumer;
  c.serial_prod = 1;
  if (d.kind == GS_ROOT) {
    int32_t ser[ND], thr[ND];
    const bool tiled = (d.flags & 3) == 3;
    int inner = 0;
    if (!tiled) {  // provisional tiling (resolve.py:159-164)
      inner = -1;
      for (int dd = 0; dd < fn.ndim; ++dd) if (fn.extent[dd] >= 16) { inner = dd; break; }
      if (inner < 0) inner = 0;
    }
    int64_t nb = 1, nt = 1, sp = 1;
#pragma unroll
    for (int dd = 0; dd < ND; ++dd) {
      int e = dd < fn.ndim ? fn.extent[dd] : 1;
      ser[dd] = tiled && dd < fn.ndim ? d.serial[dd] : 1;
      thr[dd] = tiled ? (dd < fn.ndim ? d.thread[dd] : 1) : (dd == inner ? (e < 32 ? e : 32) : 1);
      int64_t st = (int64_t)ser[dd] * thr[dd];
      int64_t b = udiv(e + st - 1, st);
      if (b < 1) b = 1;
      nb *= b; nt *= thr[dd]; sp *= ser[dd];
      c.rlo[dd] = 0; c.rhi[dd] = (int32_t)(b * st - 1);
      c.tlo[dd] = c.rlo[dd]; c.thi[dd] = c.rhi[dd];
      c.ctx[dd] = thr[dd]; c.base[dd] = 0; c.coeff[dd] = ser[dd]; c.ext[dd] = ser[dd];
    }
    c.kind = K_ROOT; c.tier = T_GLOBAL; c.kernel = (int16_t)f; c.realizations = 1;
    c.n_threads = (int32_t)nt; c.unrolled = sp < 16; c.has_serial = 1; c.serial_prod = (int32_t)sp;
    c.n_blocks = nb;
    // aggregates are kernel_aggregates()' business; keep the stored ones so
    // the change test sees only this func's own geometry
    c.k_threads = k.track ? k.cf[f].k_threads : (int32_t)nt;
    c.k_shared = k.track ? k.cf[f].k_shared : 0;
    __syncwarp();
    if (lane == 0) cf_store(k, f, c);
    __syncwarp();
    return true;
  }
  // fusion sources: reads of f issued by funcs resolved before it (resolve.py:379-393)
  const int sb = k.srcb[f], se = k.srcb[f + 1];
  int first = -1;
  for (int q = sb; q < se; ++q)
    if (k.didx[k.rd[k.srcl[q]].root] < i) { first = k.srcl[q]; break; }
  if (first < 0) { if (lane == 0) m.err |= E_SCHEDULE; __syncwarp(); return false; }
  const CF<ND> cg0 = k.cf[k.rd[first].root];
  int64_t lo[ND], hi[ND], tlo[ND], thi[ND], ts0[ND];
#pragma unroll
  for (int dd = 0; dd < ND; ++dd) { lo[dd] = tlo[dd] = INT64_MAX; hi[dd] = thi[dd] = INT64_MIN; ts0[dd] = 1; }
  {
    const RRead& r0 = k.rd[first];
    #pragma unroll 1
    for (int q = 0; q < r0.plen; ++q)
#pragma unroll
      for (int dd = 0; dd < ND; ++dd) ts0[dd] *= k.A[k.path[r0.pbeg + q]].s[dd];
  }
  for (int q0 = sb; q0 < se; q0 += 32) {
    const int q = q0 + lane;
    if (q < se) {
      const RRead& r = k.rd[k.srcl[q]];
      if (k.didx[r.root] < i) {
        const CF<ND>& cg = (d.kind == GS_FUSE_THREAD) ? cg0 : k.cf[r.root];
        int32_t blo[ND], bhi[ND];
        if (d.kind == GS_FUSE_BLOCK) block_box(cg, blo, bhi);
        else {
#pragma unroll
          for (int dd = 0; dd < ND; ++dd) { blo[dd] = cg.base[dd]; bhi[dd] = cg.base[dd] + cg.ext[dd] - 1; }
        }
#pragma unroll
        for (int dd = 0; dd < ND; ++dd) {
          int64_t a = blo[dd], b = bhi[dd];
          chain_iv(k.A, k.path + r.pbeg, r.plen, dd, a, b);
          lo[dd] = a < lo[dd] ? a : lo[dd]; hi[dd] = b > hi[dd] ? b : hi[dd];
          int64_t ta = cg.tlo[dd], tb = cg.thi[dd];
          chain_iv(k.A, k.path + r.pbeg, r.plen, dd, ta, tb);
          tlo[dd] = ta < tlo[dd] ? ta : tlo[dd]; thi[dd] = tb > thi[dd] ? tb : thi[dd];
        }
      }
    }
  }
  // the bounds are stored as int32 (CF); reduce them as int32 in one
  // redux.sync each
#pragma unroll
  for (int dd = 0; dd < ND; ++dd) {
    lo[dd] = __reduce_min_sync(0xffffffffu, (int)(lo[dd] < INT32_MAX ? lo[dd] : INT32_MAX));
    hi[dd] = __reduce_max_sync(0xffffffffu, (int)(hi[dd] > INT32_MIN ? hi[dd] : INT32_MIN));
    tlo[dd] = __reduce_min_sync(0xffffffffu, (int)(tlo[dd] < INT32_MAX ? tlo[dd] : INT32_MAX));
    thi[dd] = __reduce_max_sync(0xffffffffu, (int)(thi[dd] > INT32_MIN ? thi[dd] : INT32_MIN));
  }
  const CF<ND>& K = k.cf[cg0.kernel];
  if (d.kind == GS_FUSE_BLOCK) {
    int64_t nt = 1, sp = 1;
#pragma unroll
    for (int dd = 0; dd < ND; ++dd) {
      int s = (d.flags & 1) && dd < fn.ndim ? d.serial[dd] : 1;
      int64_t t = hi[dd] - lo[dd] + 1 + s - 1 >= 0 ? udiv(hi[dd] - lo[dd] + 1 + s - 1, s) : (hi[dd] - lo[dd] + s) / s;
      if (t < 1) t = 1;
      c.rlo[dd] = (int32_t)lo[dd];
      c.rhi[dd] = (int32_t)(lo[dd] + t * s - 1);
      c.tlo[dd] = (int32_t)tlo[dd];
      int64_t th = tlo[dd] + t * s - 1;
      c.thi[dd] = (int32_t)(thi[dd] > th ? thi[dd] : th);
      c.ctx[dd] = (int32_t)t; c.base[dd] = c.rlo[dd]; c.coeff[dd] = s; c.ext[dd] = s;
      nt *= t; sp *= s;
    }
    c.kind = K_BLOCK; c.tier = T_SHARED; c.kernel = cg0.kernel; c.realizations = K.n_blocks;
    c.n_threads = (int32_t)nt; c.unrolled = sp < 16; c.has_serial = 1; c.serial_prod = (int32_t)sp;
    __syncwarp();
    if (lane == 0) cf_store(k, f, c);
  } else {
    int64_t pe = 1;
#pragma unroll
    for (int dd = 0; dd < ND; ++dd) {
      c.rlo[dd] = (int32_t)lo[dd]; c.rhi[dd] = (int32_t)hi[dd];
      c.tlo[dd] = (int32_t)tlo[dd]; c.thi[dd] = (int32_t)thi[dd];
      c.ctx[dd] = cg0.ctx[dd]; c.base[dd] = c.rlo[dd];
      c.coeff[dd] = (int32_t)(cg0.coeff[dd] * ts0[dd]);
      c.ext[dd] = (int32_t)(hi[dd] - lo[dd] + 1);
      pe *= c.ext[dd];
    }
    c.kind = K_THREAD; c.tier = T_REGISTER; c.kernel = cg0.kernel;
    c.realizations = K.n_blocks * (int64_t)cg0.n_threads; c.n_threads = cg0.n_threads;
    c.unrolled = pe < 16; c.has_serial = 0; c.serial_prod = 1;
    __syncwarp();
    if (lane == 0) cf_store(k, f, c);
  }
  __syncwarp();
  return true;
}

// externals and unscheduled producers (resolve.py:396-425); one lane
template <int ND>
__device__ void external_one(K1<ND>& k, int f) {
  const GsFunc& fn = k.F[f];
  int64_t lo[ND], hi[ND];
#pragma unroll
  for (int dd = 0; dd < ND; ++dd) { lo[dd] = INT64_MAX; hi[dd] = INT64_MIN; }
  const int sb = k.srcb[f], se = k.srcb[f + 1];
  for (int q = sb; q < se; ++q) {
    const RRead& r = k.rd[k.srcl[q]];
    const CF<ND>& cg = k.cf[r.root];
#pragma unroll
    for (int dd = 0; dd < ND; ++dd) {
      int64_t a = cg.tlo[dd], b = cg.thi[dd];
      chain_iv(k.A, k.path + r.pbeg, r.plen, dd, a, b);
      lo[dd] = a < lo[dd] ? a : lo[dd]; hi[dd] = b > hi[dd] ? b : hi[dd];
    }
  }
  CF<ND> c;
  zero_cf(c);
  c.kind = K_EXTERNAL; c.tier = T_GLOBAL; c.kernel = -1; c.consumer = -1; c.n_threads = 1; c.serial_prod = 1;
#pragma unroll
  for (int dd = 0; dd < ND; ++dd) {
    int e = dd < fn.ndim ? fn.extent[dd] : 1;
    c.rlo[dd] = se > sb ? (int32_t)lo[dd] : 0; c.rhi[dd] = se > sb ? (int32_t)hi[dd] : e - 1;
    c.tlo[dd] = c.rlo[dd]; c.thi[dd] = c.rhi[dd];
    c.ctx[dd] = 1; c.ext[dd] = 1;
  }
  cf_store(k, f, c);
}

// kernel aggregates of a root (resolve.py:325-333): one lane
template <int ND>
__device__ void kernel_aggregates(K1<ND>& k, int kf) {
  CF<ND>& o = k.cf[kf];
  int32_t kt = o.n_threads;
  int64_t sh = 0;
  for (int q = k.kmb[kf]; q < k.kmb[kf + 1]; ++q) {
    const int f = k.kml[q];
    const CF<ND>& c = k.cf[f];
    if (c.n_threads > kt) kt = c.n_threads;
    if (c.kind == K_BLOCK) sh += alloc_of(c) * k.F[f].elem_bytes;
  }
  if (k.track && (o.k_threads != kt || o.k_shared != sh)) k.dirty[kf] |= 1 | 4;
  o.k_threads = kt;
  o.k_shared = sh;
}

// inline call totals / primary consumer (resolve.py:337-349); one lane.
// icall entries of f are visited in icall order, so the first maximum wins
// exactly as in the sequential pass over all entries.
template <int ND>
__device__ void inline_one(K1<ND>& k, int f) {
  CF<ND> ic;
  zero_cf(ic);
  ic.kind = K_INLINE; ic.consumer = -1;
  for (int q = k.icb[f]; q < k.icb[f + 1]; ++q) {
    const ICall& x = k.icall[k.icl[q]];
    const CF<ND>& c = k.cf[x.root];
    const int64_t calls = x.vol * prod_ext(c) * c.n_threads * k.cf[c.kernel].n_blocks;
    ic.calls += calls;
    if (calls > ic.best) { ic.best = calls; ic.consumer = x.root; }
  }
  const int prim = ic.consumer;
  ic.tier = T_NONE; ic.serial_prod = 1;
  if (prim >= 0) {
    const CF<ND>& h = k.cf[prim];
    ic.kernel = h.kernel; ic.n_threads = h.n_threads; ic.unrolled = h.unrolled;
    for (int dd = 0; dd < ND; ++dd) ic.ctx[dd] = h.ctx[dd];
  } else {
    ic.kernel = -1; ic.n_threads = 1; ic.unrolled = 1;
    for (int dd = 0; dd < ND; ++dd) ic.ctx[dd] = 1;
  }
  for (int dd = 0; dd < ND; ++dd) { ic.rhi[dd] = -1; ic.thi[dd] = -1; ic.ext[dd] = 1; }
  cf_store(k, f, ic);
}

// warp 0: decision validation + structure (if changed) + geometry.
//
// Siblings (same decision structure as the previous candidate of this CTA)
// re-resolve only the funcs whose dependency mask dm[f] meets the set of
// decision records that changed; every other func's record is the previous
// candidate's, which is what a full resolve would recompute bit for bit
// (geometry is a pure function of those records).  k.dirty[f] ends up 1 iff
// f's record may differ from the previous candidate's (rows use it).
// Per-phase cycle accounting of the scorer warps (diagnostics; build with
// -DGS_PHASES): 0 record load + diff, 1 resolve, 2 prune, 3 row flags,
// 4 sibling block copy, 5 row features, 6 key/source writes.
__device__ unsigned long long g_phase[16];
#ifdef GS_PHASES
#define GS_SUB(i) do { if (lane_id() == 0) { long long t_ = clock64(); atomicAdd(&g_phase[i], (unsigned long long)(t_ - tsub)); tsub = t_; } } while (0)
#define GS_MARK(i) do { if (lane == 0) { long long t_ = clock64(); ph[i] += t_ - tph; tph = t_; } } while (0)
#else
#define GS_SUB(i) do { } while (0)
#define GS_MARK(i) do { } while (0)
#endif

template <int ND>
__device__ void resolve(K1<ND>& k) {
  const int lane = lane_id();
#ifdef GS_PHASES
  long long tsub = clock64();
#endif
  Misc& m = *k.misc;
  const int nf = k.P->nf;
  const bool diff = m.same_struct;            // k.cf holds the previous candidate's geometry
  const bool incr = diff && k.mw > 0;
  if (!diff) {
    for (int f = lane; f < nf; f += 32) k.didx[f] = -1;
    __syncwarp();
    if (lane == 0) {
      int bad = 0;
      for (int i = 0; i < m.ndec; ++i) {
        const GsDecision& d = k.dec[i];
        if (d.func >= nf || d.kind > GS_INLINE || k.F[d.func].is_external || k.didx[d.func] >= 0 ||
            ((d.kind == GS_FUSE_BLOCK || d.kind == GS_FUSE_THREAD) && d.consumer >= nf))
          bad = 1;
        else
          k.didx[d.func] = (int16_t)i;
      }
      if (bad) m.err |= E_SCHEDULE;
      if (!m.err) resolve_structure(k);
    }
    __syncwarp();
    if (m.err) return;
  }
  if (incr) {
    for (int f = lane; f < nf; f += 32) {
      bool t = false;
      for (int w = 0; w < k.mw; ++w) t |= (k.dm[f * k.mw + w] & k.cmask[w]) != 0u;
      k.gdirty[f] = t;
      k.kdirty[f] = 0;
    }
    __syncwarp();
    for (int f = lane; f < nf; f += 32)
      if (k.gdirty[f] && k.kern[f] >= 0) k.kdirty[k.kern[f]] = 1;
  } else {
    for (int f = lane; f < nf; f += 32) { k.gdirty[f] = 1; k.kdirty[f] = 1; }
  }
  for (int f = lane; f < nf; f += 32) k.dirty[f] = diff ? 0 : 7;
  k.track = diff;
  __syncwarp();
  // decisions to re-resolve, in decision order
  int cnt = 0;
  for (int i0 = 0; i0 < m.ndec; i0 += 32) {
    const int i = i0 + lane;
    const bool t = i < m.ndec && k.dec[i].kind != GS_INLINE && k.gdirty[k.dec[i].func];
    const unsigned b = __ballot_sync(0xffffffffu, t);
    if (t) k.dlist[cnt + __popc(b & ((1u << lane) - 1))] = (int16_t)i;
    cnt += __popc(b);
  }
  __syncwarp();
  if (lane == 0) k.misc->ngeo = cnt;
  if (diff) GS_SUB(7); else GS_SUB(14);
  for (int q = 0; q < cnt; ++q)
    if (!geometry_one(k, k.dlist[q])) return;
  if (diff) GS_SUB(15); else GS_SUB(14);
  for (int f = lane; f < nf; f += 32)
    if ((k.F[f].is_external || k.didx[f] < 0) && k.gdirty[f]) external_one(k, f);
  __syncwarp();
  for (int f = lane; f < nf; f += 32)
    if (k.kdirty[f] && k.didx[f] >= 0 && k.dec[k.didx[f]].kind == GS_ROOT) kernel_aggregates(k, f);
  __syncwarp();
  for (int f = lane; f < nf; f += 32)
    if (k.gdirty[f] && k.didx[f] >= 0 && k.dec[k.didx[f]].kind == GS_INLINE) inline_one(k, f);
  __syncwarp();
  __syncwarp();
}

// prune verdict (options.py:200-255, machine.py:91-105), warp-wide: the
// rules are checked in the reference order (recompute, idle SMs, then per
// func in decision order warp utilization / serial / thread allocation,
// then hardware limits); sums are exact integers, so lane order is free.
template <int ND>
__device__ int prune_verdict(const K1<ND>& k) {
  const int lane = lane_id();
  const Misc& m = *k.misc;
  const GsMachine& M = k.P->m;
  const GsThresholds& th = k.P->th;
  const double minb = th.min_blocks_per_sm_factor * (double)M.num_sms;
  int64_t ci = 0;
  bool r2 = false, r6 = false;
  int first = 0;
  for (int i0 = 0; i0 < m.ndec; i0 += 32) {
    const int i = i0 + lane;
    int code = 0;
    if (i < m.ndec) {
      const GsDecision& d = k.dec[i];
      const CF<ND>& c = k.cf[d.func];
      if (d.kind == GS_INLINE) ci += c.calls;
      else {
        ci += prod_ext(c) * c.n_threads * k.cf[c.kernel].n_blocks;
        const int w = (c.n_threads + M.warp_size - 1) / M.warp_size;
        const double util = (double)c.n_threads / (double)(w * M.warp_size);
        if (util < th.warp_utilization_floor) code = GS_PRUNE_WARP_UTIL;
        else if (c.has_serial && (int64_t)c.serial_prod > th.unroll_budget) code = GS_PRUNE_SERIAL;
        else if (c.kind == K_THREAD && alloc_of(c) * k.F[d.func].elem_bytes > th.thread_alloc_bytes)
          code = GS_PRUNE_THREAD_ALLOC;
      }
      if (d.kind == GS_ROOT) {
        if ((double)c.n_blocks < minb) r2 = true;
        if (c.k_threads > M.max_threads_per_block || c.k_shared > M.shared_mem_per_block_limit) r6 = true;
      }
    }
    const unsigned b = __ballot_sync(0xffffffffu, code != 0);
    if (b && !first) first = __shfl_sync(0xffffffffu, code, __ffs(b) - 1);
  }
  for (int o = 16; o; o >>= 1) ci += __shfl_xor_sync(0xffffffffu, ci, o);
  r2 = __any_sync(0xffffffffu, r2);
  r6 = __any_sync(0xffffffffu, r6);
  if (m.ni && (double)ci > th.recompute_factor * (double)m.ni) return GS_PRUNE_RECOMPUTE;
  if (r2) return GS_PRUNE_IDLE_SMS;
  if (first) return first;
  if (r6) return GS_PRUNE_HW_LIMIT;
  return GS_VALID;
}

// ---------------------------------------------------------------------------
// exact unions of grid products (boxes.py:92-138), one lane per task
// ---------------------------------------------------------------------------
struct Iv { int64_t lo, hi; };

// footprint of [a,b] through links of dim d (resolve.py:36-44); appends to buf
__device__ int footprint(const GsAccess* A, const int16_t* p, int plen, int d, int64_t a, int64_t b,
                         Iv* buf, int cap, int& err) {
  if (cap < 1) { err |= E_LANEIV; return 0; }
  buf[0] = Iv{a, b};
  int n = 1;
  #pragma unroll 1
  for (int k = 0; k < plen; ++k) {
    const GsAccess& x = A[p[k]];
    const int64_t s = x.s[d], wl = x.lo[d], wh = x.hi[d];
    if (s <= wh - wl + 1) {       // every interval maps to one interval; merge in place
      int w = 0;
      #pragma unroll 1
      for (int i = 0; i < n; ++i) {
        Iv v{buf[i].lo * s + wl, buf[i].hi * s + wh};
        if (w && v.lo <= buf[w - 1].hi + 1) { if (v.hi > buf[w - 1].hi) buf[w - 1].hi = v.hi; }
        else buf[w++] = v;
      }
      n = w;
    } else {                      // one interval per point, already disjoint & sorted
      int64_t tot = 0;
      #pragma unroll 1
      for (int i = 0; i < n; ++i) tot += buf[i].hi - buf[i].lo + 1;
      if (tot > cap) { err |= E_LANEIV; return 0; }
      // expand from the back so the source is not overwritten
      int w = (int)tot;
      #pragma unroll 1
      for (int i = n - 1; i >= 0; --i)
        for (int64_t xx = buf[i].hi; xx >= buf[i].lo; --xx) buf[--w] = Iv{xx * s + wl, xx * s + wh};
      n = (int)tot;
    }
  }
  return n;
}

// Closed-form footprint of [a,b] through the links of dim d as an
// arithmetic progression of disjoint, non-adjacent intervals
// {start + i*step + [0, len-1] : i < cnt} (cnt == 1: one interval): a
// link x -> [x*s + lo, x*s + hi] maps an interval to an interval when s is
// at most the window width, else to a progression; a progression of
// intervals maps to a progression (merging into one interval when the
// images touch) unless both levels spread (returns false: expand).
// points = cnt*len, dim-0 runs = cnt (boxes.py:92-138 for one product).
__device__ bool footprint_ap(const GsAccess* A, const int16_t* p, int plen, int d, int64_t a, int64_t b,
                             int64_t& pts, int64_t& runs) {
  int64_t st = a, step = 1, len = b - a + 1, cnt = 1;
  if (len <= 0) { pts = runs = 0; return true; }
  #pragma unroll 1
  for (int k = 0; k < plen; ++k) {
    const GsAccess& x = A[p[k]];
    const int64_t s = x.s[d], wl = x.lo[d], w = (int64_t)x.hi[d] - x.lo[d] + 1;
    if (cnt == 1) {
      if (s <= w) { st = st * s + wl; len = (len - 1) * s + w; }
      else { cnt = len; st = st * s + wl; step = s; len = w; }
    } else if (s <= w) {
      const int64_t nl = (len - 1) * s + w, ns = step * s, n0 = st * s + wl;
      if (ns <= nl) { st = n0; len = (cnt - 1) * ns + nl; cnt = 1; step = 1; }
      else { st = n0; step = ns; len = nl; }
    } else if (len == 1) {
      const int64_t ns = step * s, n0 = st * s + wl;
      if (ns <= w) { st = n0; len = (cnt - 1) * ns + w; cnt = 1; step = 1; }
      else { st = n0; step = ns; len = w; }
    } else {
      return false;
    }
  }
  pts = cnt * len;
  runs = cnt;
  return true;
}

// A group of one read: closed form per dim, no interval lists (inlined:
// the common case); false = use the general union below.
template <int ND>
__device__ __forceinline__ bool union_count_one(const GsAccess* A, const RRead* rd, const int16_t* paths,
                                                const int16_t* rl, const int8_t* grp, int nr, int g,
                                                const int32_t* blo, const int32_t* bhi, int64_t& vol,
                                                int64_t& lines) {
  int K1 = 0, only = -1;
  for (int q = 0; q < nr; ++q) if (grp[q] == g) { ++K1; only = q; }
  if (K1 != 1) return false;
  const RRead& r = rd[rl[only]];
  int64_t pv[ND], rv[ND];
  bool ok = true;
#pragma unroll
  for (int d = 0; d < ND; ++d) ok = ok && footprint_ap(A, paths + r.pbeg, r.plen, d, blo[d], bhi[d], pv[d], rv[d]);
  if (!ok) return false;
  int64_t outer = 1;
#pragma unroll
  for (int d = 1; d < ND; ++d) outer *= pv[d];
  vol = pv[0] * outer;
  lines = rv[0] * outer;
  return true;
}

template <int ND>
__device__ __noinline__ void union_count(const GsAccess* A, const RRead* rd, const int16_t* paths,
                            const int16_t* rl, const int8_t* grp, int nr, int g,
                            const int32_t* blo, const int32_t* bhi,
                            int64_t& vol, int64_t& lines, int& err) {
  Iv buf[kLaneIv];
  int16_t off[kGroupReads][ND], cnt[kGroupReads][ND];
  int K = 0, used = 0;
  for (int q = 0; q < nr; ++q) {
    if (grp[q] != g) continue;
    if (K >= kGroupReads) { err |= E_GROUP; vol = lines = 0; return; }
    const RRead& r = rd[rl[q]];
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      int n = footprint(A, paths + r.pbeg, r.plen, d, blo[d], bhi[d], buf + used, kLaneIv - used, err);
      off[K][d] = (int16_t)used; cnt[K][d] = (int16_t)n; used += n;
    }
    ++K;
  }
  vol = lines = 0;
  if (err || K == 0) return;
  if (K == 1) {
    int64_t outer = 1;
    for (int d = 1; d < ND; ++d) {
      int64_t t = 0;
      #pragma unroll 1
      for (int i = 0; i < cnt[0][d]; ++i) t += buf[off[0][d] + i].hi - buf[off[0][d] + i].lo + 1;
      outer *= t;
    }
    int64_t t0 = 0;
    #pragma unroll 1
    for (int i = 0; i < cnt[0][0]; ++i) t0 += buf[off[0][0] + i].hi - buf[off[0][0] + i].lo + 1;
    vol = t0 * outer;
    lines = (int64_t)cnt[0][0] * outer;
    return;
  }
  // outer-dim cut points (coordinate compression)
  constexpr int kCuts = 64;
  int64_t cuts[ND > 1 ? ND - 1 : 1][kCuts];
  int ncut[ND > 1 ? ND - 1 : 1];
  for (int d = 1; d < ND; ++d) {
    int n = 0;
    #pragma unroll 1
    for (int q = 0; q < K; ++q)
      #pragma unroll 1
      for (int i = 0; i < cnt[q][d]; ++i) {
        int64_t v2[2] = {buf[off[q][d] + i].lo, buf[off[q][d] + i].hi + 1};
        for (int e = 0; e < 2; ++e) {
          int64_t v = v2[e];
          int pos = n;
          bool dup = false;
          #pragma unroll 1
          for (int t = 0; t < n; ++t) { if (cuts[d - 1][t] == v) { dup = true; break; } }
          if (dup) continue;
          if (n >= kCuts) { err |= E_LANEIV; return; }
          while (pos > 0 && cuts[d - 1][pos - 1] > v) { cuts[d - 1][pos] = cuts[d - 1][pos - 1]; --pos; }
          cuts[d - 1][pos] = v;
          ++n;
        }
      }
    ncut[d - 1] = n;
  }
  int idx[ND > 1 ? ND - 1 : 1];
  for (int d = 0; d < ND - 1; ++d) idx[d] = 0;
  while (true) {
    bool valid = true;
    for (int d = 0; d < ND - 1; ++d) if (ncut[d] < 2) valid = false;
    if (!valid && ND > 1) break;
    // cell = pieces idx[d]
    int64_t cellv = 1;
    unsigned act = 0;
    #pragma unroll 1
    for (int q = 0; q < K; ++q) {
      bool in = true;
      for (int d = 1; d < ND && in; ++d) {
        int64_t p0 = cuts[d - 1][idx[d - 1]];
        bool hit = false;
        #pragma unroll 1
        for (int i = 0; i < cnt[q][d]; ++i) {
          const Iv& v = buf[off[q][d] + i];
          if (v.lo <= p0 && p0 <= v.hi) { hit = true; break; }
        }
        in = hit;
      }
      if (in) act |= 1u << q;
    }
    for (int d = 1; d < ND; ++d) cellv *= cuts[d - 1][idx[d - 1] + 1] - cuts[d - 1][idx[d - 1]];
    if (act) {
      // k-way merge of the active dim-0 lists
      int head[kGroupReads];
      #pragma unroll 1
      for (int q = 0; q < K; ++q) head[q] = 0;
      int64_t runs = 0, len = 0, cl = 0, ch = 0;
      bool open = false;
      while (true) {
        int best = -1;
        int64_t bl = 0;
        #pragma unroll 1
        for (int q = 0; q < K; ++q) {
          if (!((act >> q) & 1) || head[q] >= cnt[q][0]) continue;
          int64_t l = buf[off[q][0] + head[q]].lo;
          if (best < 0 || l < bl) { best = q; bl = l; }
        }
        if (best < 0) break;
        const Iv& v = buf[off[best][0] + head[best]];
        ++head[best];
        if (open && v.lo <= ch + 1) { if (v.hi > ch) ch = v.hi; }
        else {
          if (open) { ++runs; len += ch - cl + 1; }
          cl = v.lo; ch = v.hi; open = true;
        }
      }
      if (open) { ++runs; len += ch - cl + 1; }
      vol += len * cellv;
      lines += runs * cellv;
    }
    // advance mixed radix
    if (ND == 1) break;
    int d = 0;
    while (d < ND - 1) {
      if (++idx[d] < ncut[d] - 1) break;
      idx[d] = 0;
      ++d;
    }
    if (d == ND - 1) break;
  }
}

// ---------------------------------------------------------------------------
// warp-instruction transaction counts (featurize.py:173-196, 508-571)
// ---------------------------------------------------------------------------
// Residue arithmetic modulo the transaction / bank period M: shifts and
// masks when M is a power of two (every real machine), divisions otherwise.

// out-of-line slow paths (non-power-of-two periods): keep 64-bit division
// code out of the hot loops' instruction footprint
__device__ __noinline__ int64_t floordiv_slow(int64_t a, int64_t b) { return floordiv(a, b); }
__device__ __noinline__ int64_t posmod_slow(int64_t a, int64_t m) { return posmod(a, m); }

template <int MC>
struct ModM {
  int M, lg;
  __device__ explicit ModM(int m) : M(MC ? MC : m), lg(-1) {
    if (MC) { lg = 0; while ((1 << lg) < MC) ++lg; }   // constant-folded
    else if (m > 0 && (m & (m - 1)) == 0) { lg = 0; while ((1 << lg) < m) ++lg; }
  }
  __device__ __forceinline__ int64_t fdiv(int64_t a) const {
    if (MC) return a >> lg;
    return lg >= 0 ? (a >> lg) : floordiv_slow(a, M);
  }
  __device__ __forceinline__ int pmod(int64_t a) const {
    if (MC) return (int)(a & (int64_t)(MC - 1));
    return lg >= 0 ? (int)(a & (int64_t)(M - 1)) : (int)posmod_slow(a, M);
  }
  // #{x in [a,b] : x = r (mod M)}
  __device__ __forceinline__ unsigned long long count_in(int64_t a, int64_t b, int r) const {
    if (b < a) return 0;
    return (unsigned long long)(fdiv(b - r) - fdiv(a - 1 - r));
  }
};

// Lane origins (byte address of instruction constant 0) of the emulated
// warps of block 0, warp after warp: thread t's coordinates are the
// mixed-radix digits of t over the thread extents (dim 0 fastest); moving
// to the next warp adds the digits of 32 with carries — no division in the
// loop.
template <int ND>
struct WarpWalk {
  int cd[ND], inc[ND], ext[ND];
  int64_t mul[ND], im[ND], em[ND], o;
  int t, n;
  __device__ WarpWalk(const CF<ND>& h, const int64_t* ts, const int64_t* bs, int64_t cst, int lane) {
    int a = lane, b = 32;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      ext[d] = h.ctx[d];
      cd[d] = a % ext[d]; a /= ext[d];
      inc[d] = b % ext[d]; b /= ext[d];
      mul[d] = (int64_t)h.coeff[d] * ts[d] * bs[d];
    }
    cd[ND - 1] += a * ext[ND - 1];   // top digit is unbounded
    inc[ND - 1] += b * ext[ND - 1];
    o = cst;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      o += (int64_t)cd[d] * mul[d];
      im[d] = (int64_t)inc[d] * mul[d];
      em[d] = (int64_t)ext[d] * mul[d];
    }
    t = lane;
    n = h.n_threads;
  }
  // the origin is carried along with the digits: adds only in the loop
  __device__ __forceinline__ int64_t origin(bool& active) const {
    active = t < n;
    return o;
  }
  __device__ __forceinline__ void next() {
    int carry = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      cd[d] += inc[d] + carry;
      o += im[d];
      if (carry) o += mul[d];
      carry = 0;
      if (d < ND - 1 && cd[d] >= ext[d]) { cd[d] -= ext[d]; o -= em[d]; carry = 1; }
    }
    t += 32;
  }
};

// Regular thread tiles — dim-0 rows of a multiple of 32 threads, or whole
// rows whose length divides 32 stacked without wrapping, and only full
// warps — give every emulated warp warp 0's lane pattern, shifted by the
// origin of its first thread.  A warp's transaction count depends on that
// shift only modulo the counter's period (32 B segments; 128 B of banks).
template <int ND>
__device__ __forceinline__ bool regular_tile(const CF<ND>& h) {
  if ((h.n_threads & 31) != 0) return false;
  const int cx = h.ctx[0];
  return (cx % 32 == 0) || (ND >= 2 && 32 % cx == 0 && h.ctx[ND >= 2 ? 1 : 0] % (32 / cx) == 0);
}

// Histogram of the emulated warps' shifts modulo 32 * NR: register j of
// lane b counts the warps whose shift = 32 j + b.  A uniform (scalar)
// mixed-radix walk over the warps' first threads: adds only.
template <int ND, int NR>
__device__ __forceinline__ void shift_hist(const WarpWalk<ND>& walk, int nwarps, int lane, unsigned (&cnt)[NR]) {
  int dg[ND];
#pragma unroll
  for (int d = 0; d < ND; ++d) dg[d] = 0;
#pragma unroll
  for (int j = 0; j < NR; ++j) cnt[j] = 0;
  int64_t dlt = 0;
#pragma unroll 1
  for (int w = 0; w < nwarps; ++w) {
    const int key = (int)(dlt & (int64_t)(32 * NR - 1));
    const bool me = lane == (key & 31);
#pragma unroll
    for (int j = 0; j < NR; ++j) cnt[j] += (unsigned)(me && (key >> 5) == j);
    int carry = 0;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      dg[d] += walk.inc[d] + carry;
      dlt += walk.im[d];
      if (carry) dlt += walk.mul[d];
      carry = 0;
      if (d < ND - 1 && dg[d] >= walk.ext[d]) { dg[d] -= walk.ext[d]; dlt -= walk.em[d]; carry = 1; }
    }
  }
}

// the regular-tile path pays off from this many emulated warps on
constexpr int kRegularMinWarps = 4;   // 2 and 8 measure the same

// transactions of one emulated warp for ONE instruction constant r
// (featurize.py:173-196): global = distinct segments; shared = max over
// banks of distinct words; warp-collective, lanes agree on the result
template <int MC>
__device__ __forceinline__ unsigned warp_count(unsigned long long a, bool active, int tier, const ModM<MC>& mg, int bw_lg,
                                               int bw, int banks) {
  const int lane = lane_id();
  if (tier == T_GLOBAL) {
    unsigned long long seg = mg.lg >= 0 ? (a >> mg.lg) : a / (unsigned long long)mg.M;
    if (!active) seg = ~0ull - lane;
    const unsigned lm = __match_any_sync(0xffffffffu, seg);
    const bool lead = active && (__ffs(lm) - 1 == lane);
    return __popc(__ballot_sync(0xffffffffu, lead));
  }
  unsigned long long word = bw_lg >= 0 ? (a >> bw_lg) : a / (unsigned long long)bw;
  unsigned bank = (unsigned)(word % (unsigned long long)banks);
  if (!active) { word = ~0ull - lane; bank = 0x80000000u + lane; }
  const unsigned lm = __match_any_sync(0xffffffffu, word);
  const bool lead = active && (__ffs(lm) - 1 == lane);
  const unsigned leaders = __ballot_sync(0xffffffffu, lead);
  const unsigned bm = __match_any_sync(0xffffffffu, bank);
  const unsigned per_bank = active ? __popc(bm & leaders) : 0u;
  return __reduce_max_sync(0xffffffffu, per_bank);
}

// Warp transactions of all load (or store) instructions of one read in
// block 0 (featurize.py:508-571).  All lanes; returns the total.
//
// 1. T[k], k < M: how many emitted instructions have address constant = k
//    (mod M), by cyclic convolution of per-dim histograms (the count of a
//    warp instruction depends on its constant only mod M: shifting every
//    lane by M shifts every segment / keeps every bank).
// 2. Emulated warps whose lane-origin pattern equals another's up to a
//    constant shift d are one "class": their counts are the class
//    representative's at residue k + d, so the representative is evaluated
//    once per residue against the shifted histograms of all its members.
//    For shared memory the count depends on the residue only mod the bank
//    width (adding whole words rotates the banks), so at most bank-width
//    evaluations are needed per class.
// Histogram of the emitted instructions' address constants modulo Q (a
// power of two <= 32), lane = residue, all in registers: per-dim coordinate
// counts, window taps and the byte-stride map are shuffles (odd multipliers
// permute Z/Q; a factor 2^a folds the top a bits), and the convolution into
// the running histogram runs over its nonzero residues.  Q = 32: global
// 32-byte segments.  Q = bank width: shared banks, whose count depends on
// the constant only modulo the bank width.  Lanes >= Q return 0.
template <int ND, int Q>
__device__ unsigned long long residue_hist(const GsAccess* A, const int16_t* path, int plen, bool identity,
                                           const CF<ND>& h, const int64_t* bs, WarpScr& W, int& err) {
  constexpr int QL = Q == 32 ? 5 : Q == 16 ? 4 : Q == 8 ? 3 : Q == 4 ? 2 : Q == 2 ? 1 : 0;
  const int lane = lane_id();
  const bool mine = lane < Q;
  const ModM<Q> mq(Q);
  unsigned long long T = lane == 0;
#pragma unroll 1
  for (int d = 0; d < ND; ++d) {
    const int e = h.ext[d];
    unsigned long long H = 0;
    if (identity || !h.unrolled) {
      if (mine) H = mq.count_in(0, e - 1, lane);
      if (!identity) {
#pragma unroll 1
        for (int q = 0; q < plen; ++q) {
          const GsAccess& x = A[path[q]];
          const int64_t s = x.s[d], wl = x.lo[d], wh = x.hi[d];
          unsigned long long S = 0;
          if (wh - wl + 1 >= Q) {
            unsigned nz = __ballot_sync(0xffffffffu, mine && H != 0);
            while (nz) {
              const int r = __ffs(nz) - 1; nz &= nz - 1;
              const unsigned long long hv = __shfl_sync(0xffffffffu, H, r);
              S += hv * mq.count_in(wl, wh, (int)((lane - (int64_t)r * s) & (Q - 1)));
            }
          } else if (s & 1) {
            int inv = (int)s;
            inv *= 2 - (int)s * inv;
            inv *= 2 - (int)s * inv;
#pragma unroll 1
            for (int64_t w = wl; w <= wh; ++w)
              S += __shfl_sync(0xffffffffu, H, (int)(((lane - w) * inv) & (Q - 1)));
          } else {   // even stride: scatter through shared memory
            if (mine) { W.H[lane] = H; W.S[lane] = 0; }
            __syncwarp();
            if (mine && H) {
              const int64_t base = (int64_t)lane * s;
#pragma unroll 1
              for (int64_t w = wl; w <= wh; ++w) atomicAdd(&W.S[(int)((base + w) & (Q - 1))], H);
            }
            __syncwarp();
            if (mine) S = W.S[lane];
            __syncwarp();
          }
          H = mine ? S : 0;
        }
      }
    } else {
      Iv buf[kLaneIv];
      const int n = footprint(A, path, plen, d, 0, e - 1, buf, kLaneIv, err);
#pragma unroll 1
      for (int i = 0; i < n; ++i) if (mine) H += mq.count_in(buf[i].lo, buf[i].hi, lane);
    }
    // scale by the byte stride of dim d: S2[(r * bm) mod Q] += H[r]
    const int bm = (int)(bs[d] & (Q - 1));
    unsigned long long S2;
    if (bm == 0) {
      unsigned long long u = H;
      for (int o = 16; o; o >>= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
      S2 = lane == 0 ? u : 0;
    } else {
      const int a = __ffs(bm) - 1, odd = bm >> a, lo = QL - a;
      int inv = odd;
      inv *= 2 - odd * inv;
      inv *= 2 - odd * inv;
      unsigned long long u = H;
      for (int o = 1 << lo; o < Q; o <<= 1) u += __shfl_xor_sync(0xffffffffu, u, o);
      const int src = ((lane >> a) * inv) & ((1 << lo) - 1);
      const unsigned long long g = __shfl_sync(0xffffffffu, u, src);
      S2 = mine && (lane & ((1 << a) - 1)) == 0 ? g : 0;
    }
    // T <- T (*) S2 (cyclic), summing over the sparser operand (S2 is
    // usually a single residue for outer dims: row pitches of 32 B multiples)
    unsigned long long Tn = 0;
    unsigned nzt = __ballot_sync(0xffffffffu, mine && T != 0);
    unsigned nzs = __ballot_sync(0xffffffffu, mine && S2 != 0);
    const bool over_s = __popc(nzs) < __popc(nzt);
    unsigned nz = over_s ? nzs : nzt;
    const unsigned long long X = over_s ? S2 : T, Y = over_s ? T : S2;
    while (nz) {
      const int r = __ffs(nz) - 1; nz &= nz - 1;
      const unsigned long long xr = __shfl_sync(0xffffffffu, X, r);
      Tn += xr * __shfl_sync(0xffffffffu, Y, (lane - r) & (Q - 1));
    }
    T = mine ? Tn : 0;
  }
  return T;
}

// Default machine (32-byte segments, 32 banks x 4 bytes): compact counters
// with only the code that machine runs, to keep the hot instruction
// footprint small.  bs: byte stride per dim of the producer's allocation;
// ts: chain stride product per dim; cst: address of the constant-0 access
// of thread 0 (+ bias).
template <int ND>
__device__ __forceinline__ void tx_strides(const GsAccess* A, const int16_t* path, int plen, bool identity,
                                           const CF<ND>& prod, int eb, int64_t* bs, int64_t* ts) {
  int64_t acc = eb;
#pragma unroll
  for (int d = 0; d < ND; ++d) {
    bs[d] = acc;
    acc *= (int64_t)prod.rhi[d] - prod.rlo[d] + 1;
    ts[d] = 1;
    if (!identity)
#pragma unroll 1
      for (int q = 0; q < plen; ++q) ts[d] *= A[path[q]].s[d];
  }
}

// global: register histogram mod 32 + interval sums over its prefix scan
template <int ND>
__device__ __forceinline__ unsigned long long tx_global32(const GsAccess* A, const int16_t* path, int plen,
                                                       bool identity, const CF<ND>& h, const CF<ND>& prod, int eb,
                                                       WarpScr& W, int& err) {
  const int lane = lane_id();
  int64_t bs[ND], ts[ND];
  tx_strides<ND>(A, path, plen, identity, prod, eb, bs, ts);
  const unsigned long long tv = residue_hist<ND, 32>(A, path, plen, identity, h, bs, W, err);
  int64_t cst = kAddrBias;
#pragma unroll
  for (int d = 0; d < ND; ++d) cst += ((int64_t)h.base[d] * ts[d] - prod.rlo[d]) * bs[d];
  unsigned long long incl = tv;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += u;
  }
  const unsigned long long pex = incl - tv;
  const unsigned long long tsum = __shfl_sync(0xffffffffu, incl, 31);
  const ModM<32> mm(32);
  unsigned long long total = 0, part = 0;   // part: per-lane shares, summed once after the walk
  const int nwarps = (h.n_threads + 31) / 32;
  WarpWalk<ND> walk(h, ts, bs, cst, lane);
  // lane share of one emulated warp whose lane addresses are non-decreasing
  auto mono_share = [&](int64_t org, int64_t up) {
    unsigned long long c = 0;
    int lo = 0, hi = 0;
    if (lane > 0) {
      const int64_t d = org - up;
      if (d >= 32) c = tsum;
      else { lo = (int)((32 - d - (up & 31)) & 31); hi = lo + (int)d; }
    } else {
      c = tsum;
    }
    const unsigned long long plo = __shfl_sync(0xffffffffu, pex, lo);
    const unsigned long long phi = __shfl_sync(0xffffffffu, pex, hi & 31);
    if (hi > lo) c = hi <= 32 ? (hi == 32 ? tsum : phi) - plo : (tsum - plo) + phi;
    return c;
  };
  if (nwarps >= kRegularMinWarps && regular_tile<ND>(h)) {
    bool active;
    const int64_t org = walk.origin(active);   // warp 0, all lanes active
    const int64_t up = __shfl_up_sync(0xffffffffu, org, 1);
    if (__all_sync(0xffffffffu, lane == 0 || org >= up)) {
      unsigned cnt[1];
      shift_hist<ND, 1>(walk, nwarps, lane, cnt);
      unsigned nz = __ballot_sync(0xffffffffu, cnt[0] != 0);
      while (nz) {
        const int r = __ffs(nz) - 1; nz &= nz - 1;
        const unsigned cr = __shfl_sync(0xffffffffu, cnt[0], r);
        part += (unsigned long long)cr * mono_share(org + r, up + r);
      }
      for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      return part;
    }
  }
  for (int w = 0; w < nwarps; ++w, walk.next()) {
    bool active;
    const int64_t org = walk.origin(active);
    const int64_t up = __shfl_up_sync(0xffffffffu, org, 1);
    if (__all_sync(0xffffffffu, lane == 0 || !active || org >= up)) {
      const unsigned long long c = mono_share(org, up);
      if (active) part += c;
    } else {
#pragma unroll 1
      for (int r = 0; r < 32; ++r) {
        const unsigned long long wr = __shfl_sync(0xffffffffu, tv, r);
        if (wr) total += wr * warp_count((unsigned long long)(org + r), active, T_GLOBAL, mm, 2, 4, 32);
      }
    }
  }
  for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  return total + part;
}

// shared: register histogram mod the 4-byte bank width, one evaluation
// per emulated warp per residue mod 4 that occurs
template <int ND>
__device__ __forceinline__ unsigned long long tx_shared4(const GsAccess* A, const int16_t* path, int plen,
                                                      bool identity, const CF<ND>& h, const CF<ND>& prod, int eb,
                                                      WarpScr& W, int& err) {
  const int lane = lane_id();
  int64_t bs[ND], ts[ND];
  tx_strides<ND>(A, path, plen, identity, prod, eb, bs, ts);
  const unsigned long long tb = residue_hist<ND, 4>(A, path, plen, identity, h, bs, W, err);
  int64_t cst = kAddrBias;
#pragma unroll
  for (int d = 0; d < ND; ++d) cst += ((int64_t)h.base[d] * ts[d] - prod.rlo[d]) * bs[d];
  const ModM<128> mm(128);
  const unsigned ew = __ballot_sync(0xffffffffu, lane < 4 && tb != 0) & 0xFu;
  unsigned long long tb_all = lane < 4 ? tb : 0;
  tb_all += __shfl_xor_sync(0xffffffffu, tb_all, 1);
  tb_all += __shfl_xor_sync(0xffffffffu, tb_all, 2);
  tb_all = __shfl_sync(0xffffffffu, tb_all, 0);
  unsigned long long total = 0;
  const int nwarps = (h.n_threads + 31) / 32;
  WarpWalk<ND> walk(h, ts, bs, cst, lane);
  // one emulated warp, every constant residue mod 4 that occurs
  auto warp_total = [&](int64_t org, int64_t up, bool active, bool mono) {
    unsigned long long t = 0;
    unsigned m4 = ew;
    while (m4) {
      const int e = __ffs(m4) - 1; m4 &= m4 - 1;
      const unsigned long long we = __shfl_sync(0xffffffffu, tb, e);
      if (mono) {
        const int64_t word = (org + e) >> 2, wup = (up + e) >> 2;
        const bool lead = active && (lane == 0 || word != wup);
        const unsigned bank = lead ? (unsigned)(word & 31) : 0x80000000u + lane;
        const unsigned bmask = __match_any_sync(0xffffffffu, bank);
        const unsigned per_bank = lead ? __popc(bmask) : 0u;
        t += we * __reduce_max_sync(0xffffffffu, per_bank);
      } else {
        t += we * warp_count((unsigned long long)(org + e), active, T_SHARED, mm, 2, 4, 32);
      }
    }
    return t;
  };
  if (nwarps >= kRegularMinWarps && regular_tile<ND>(h)) {
    // every warp has warp 0's lane pattern: the one-transaction test holds
    // for all warps or for none, and otherwise the count depends on the
    // shift mod 128 (32 banks x 4 B)
    bool active;
    const int64_t org = walk.origin(active);   // warp 0, all lanes active
    const int64_t up = __shfl_up_sync(0xffffffffu, org, 1);
    const bool mono = __all_sync(0xffffffffu, lane == 0 || org >= up);
    const int64_t span = __shfl_sync(0xffffffffu, org, 31) - __shfl_sync(0xffffffffu, org, 0);
    if (mono && span <= 124) return (unsigned long long)nwarps * tb_all;
    unsigned cnt[4];
    shift_hist<ND, 4>(walk, nwarps, lane, cnt);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      unsigned nz = __ballot_sync(0xffffffffu, cnt[j] != 0);
      while (nz) {
        const int b = __ffs(nz) - 1; nz &= nz - 1;
        const unsigned cr = __shfl_sync(0xffffffffu, cnt[j], b);
        total += (unsigned long long)cr * warp_total(org + 32 * j + b, up + 32 * j + b, true, mono);
      }
    }
    return total;
  }
  for (int w = 0; w < nwarps; ++w, walk.next()) {
    bool active;
    const int64_t org = walk.origin(active);
    // non-decreasing lane addresses (row-major tiles): equal words are
    // neighbours, so word leaders come from one shuffle, and only the bank
    // needs a match
    const int64_t up = __shfl_up_sync(0xffffffffu, org, 1);
    const unsigned act = __ballot_sync(0xffffffffu, active);
    const bool mono = __all_sync(0xffffffffu, lane == 0 || !active || org >= up);
    // the active lanes are a prefix starting at lane 0; when their bytes
    // span at most 124 (+3 for the residue), every distinct word falls in
    // a distinct bank: one transaction per instruction
    const int64_t span = __shfl_sync(0xffffffffu, org, 31 - __clz(act)) - __shfl_sync(0xffffffffu, org, 0);
    if (mono && span <= 124) { total += tb_all; continue; }
    total += warp_total(org, up, active, mono);
  }
  return total;
}

// MC / BW / NB: compile-time period, bank width and bank count for the
// common machines (0 = read them from Mc at run time).
template <int ND, int MC, int BW, int NB>
__device__ __noinline__ unsigned long long warp_tx(const GsAccess* A, const int16_t* path, int plen, bool identity,
                                      const CF<ND>& h, const CF<ND>& prod, int eb, int tier,
                                      const GsMachine& Mc, WarpScr& W, int& err) {
  if constexpr (MC == 32) {
    return tx_global32<ND>(A, path, plen, identity, h, prod, eb, W, err);
  } else if constexpr (MC == 128 && BW == 4) {
    return tx_shared4<ND>(A, path, plen, identity, h, prod, eb, W, err);
  }
  const int lane = lane_id();
#ifdef GS_PHASES
  long long tsub = clock64();
#endif
  const int M = MC ? MC : tier == T_GLOBAL ? Mc.global_transaction_bytes : Mc.shared_banks * Mc.bank_width_bytes;
  const ModM<MC> mm(M);
  const int per = (M + 31) / 32;
  int64_t bs[ND], ts[ND];
  {
    int64_t acc = eb;
#pragma unroll
    for (int d = 0; d < ND; ++d) {
      bs[d] = acc;
      acc *= (int64_t)prod.rhi[d] - prod.rlo[d] + 1;
      ts[d] = 1;
      if (!identity)
        #pragma unroll 1
        for (int q = 0; q < plen; ++q) ts[d] *= A[path[q]].s[d];
    }
  }
  // shared banks on the default machine: only the constants mod the 4-byte
  // bank width matter (see the class counting below)
  constexpr bool kFold4 = MC == 128 && BW == 4;
  unsigned long long tb4 = 0;
  if (MC == 32) {
    W.T[lane] = residue_hist<ND, 32>(A, path, plen, identity, h, bs, W, err);
    __syncwarp();
  } else if (kFold4 && tier != T_GLOBAL) {
    tb4 = residue_hist<ND, 4>(A, path, plen, identity, h, bs, W, err);
  } else {
    for (int j = 0; j < per; ++j) { int r = lane + 32 * j; if (r < M) W.T[r] = (r == 0); }
    __syncwarp();
    for (int d = 0; d < ND; ++d) {
      const int e = h.ext[d];
      // per-dim histogram of relative coordinates (mod M) into H
      if (identity || !h.unrolled) {
        for (int j = 0; j < per; ++j) { int r = lane + 32 * j; if (r < M) W.GH[r] = mm.count_in(0, e - 1, r); }
        __syncwarp();
        if (!identity) {
          for (int q = 0; q < plen; ++q) {
            const GsAccess& x = A[path[q]];
            const int64_t s = x.s[d], wl = x.lo[d], wh = x.hi[d];
            // S[k] = sum_r H[r] * #{w in [wl,wh] : r*s + w = k (mod M)}
            for (int j = 0; j < per; ++j) { int r = lane + 32 * j; if (r < M) W.GS[r] = 0; }
            __syncwarp();
            if (wh - wl + 1 < M) {       // short window: scatter each residue's taps
              for (int j = 0; j < per; ++j) {
                const int r = lane + 32 * j;
                if (r >= M) continue;
                const unsigned long long hv = W.GH[r];
                if (!hv) continue;
                const int64_t base = (int64_t)r * s;
                #pragma unroll 1
                for (int64_t w = wl; w <= wh; ++w) atomicAdd(&W.GS[mm.pmod(base + w)], hv);
              }
            } else {
              for (int c = 0; c < per; ++c) {
                unsigned nz = __ballot_sync(0xffffffffu, (c * 32 + lane) < M && W.GH[c * 32 + lane] != 0);
                while (nz) {
                  const int b = __ffs(nz) - 1; nz &= nz - 1;
                  const int r = c * 32 + b;
                  const unsigned long long hv = W.GH[r];
                  const int64_t sh = mm.pmod((int64_t)r * s);
                  for (int j = 0; j < per; ++j) {
                    const int k = lane + 32 * j;
                    if (k < M) W.GS[k] += hv * mm.count_in(wl, wh, mm.pmod(k - sh));
                  }
                }
              }
            }
            __syncwarp();
            for (int j = 0; j < per; ++j) { int r = lane + 32 * j; if (r < M) W.GH[r] = W.GS[r]; }
            __syncwarp();
          }
        }
      } else {
        // unrolled: unique points of the chain footprint of [0, e-1]
        Iv buf[kLaneIv];
        int n = footprint(A, path, plen, d, 0, e - 1, buf, kLaneIv, err);
        for (int j = 0; j < per; ++j) {
          int r = lane + 32 * j;
          if (r >= M) continue;
          unsigned long long c = 0;
          #pragma unroll 1
          for (int i = 0; i < n; ++i) c += mm.count_in(buf[i].lo, buf[i].hi, r);
          W.GH[r] = c;
        }
        __syncwarp();
      }
      // scale by the byte stride of dim d, then convolve into T
      const int64_t bm = mm.pmod(bs[d]);
      for (int j = 0; j < per; ++j) { int r = lane + 32 * j; if (r < M) W.GS[r] = 0; }
      __syncwarp();
      for (int j = 0; j < per; ++j) {
        int r = lane + 32 * j;
        if (r < M && W.GH[r]) atomicAdd(&W.GS[mm.pmod((int64_t)r * bm)], W.GH[r]);
      }
      // nonzero residues of T, then H[k] = sum_r T[r] S[k - r] (lane per k)
      int nnz = 0;
      for (int c = 0; c < per; ++c) {
        const int r = c * 32 + lane;
        const bool t = r < M && W.T[r] != 0;
        const unsigned b = __ballot_sync(0xffffffffu, t);
        if (t) W.nz[nnz + __popc(b & ((1u << lane) - 1))] = (int16_t)r;
        nnz += __popc(b);
      }
      __syncwarp();
      for (int j = 0; j < per; ++j) {
        const int k = lane + 32 * j;
        if (k >= M) continue;
        unsigned long long acc = 0;
        #pragma unroll 1
        for (int i = 0; i < nnz; ++i) {
          const int r = W.nz[i];
          acc += W.T[r] * W.GS[mm.pmod(k - r)];
        }
        W.GH[k] = acc;
      }
      __syncwarp();
      for (int j = 0; j < per; ++j) { int r = lane + 32 * j; if (r < M) W.T[r] = W.GH[r]; }
      __syncwarp();
    }
  }
  GS_SUB(7);
  // ---- count: warp-pattern classes ---------------------------------------
  const int nwarps = (h.n_threads + 31) / 32;
  int64_t cst = kAddrBias;
#pragma unroll
  for (int d = 0; d < ND; ++d) cst += ((int64_t)h.base[d] * ts[d] - prod.rlo[d]) * bs[d];
  const int bw = BW ? BW : Mc.bank_width_bytes, banks = NB ? NB : Mc.shared_banks;
  const int bw_lg = BW ? (BW == 4 ? 2 : BW == 8 ? 3 : __ffs(BW) - 1) : (bw & (bw - 1)) == 0 ? __ffs(bw) - 1 : -1;
  // residues that matter per class: all M (global), M mod bank width (shared)
  const bool fold = tier != T_GLOBAL && bw_lg >= 0 && bw <= 32 && (M % bw) == 0;
  const int P = fold ? bw : M;                 // class weight vector length
  const int pp = (P + 31) / 32;
  // TB[e] = sum of T[r] over r = e (mod P): lane e (fold) holds it
  unsigned long long tb = 0;
  if (kFold4 && fold) {
    tb = tb4;                      // lane e < 4 holds TB[e]
  } else if (fold) {
    for (int j = 0; j < per; ++j) {
      const int r = lane + 32 * j;
      const unsigned long long v = r < M ? W.T[r] : 0ull;
      // lanes with the same residue mod bw add up (bw divides 32)
      unsigned long long sum = v;
      for (int o = bw; o < 32; o <<= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      tb += sum;
    }
  }
  if (MC == 32 && tier == T_GLOBAL) {
    // 32-byte segments, lanes = residues.  For a warp whose active lane
    // addresses are non-decreasing, lane i > 0 opens a new segment for the
    // residues r with ((a[i-1] + r) mod 32) >= 32 - d (d = a[i] - a[i-1]),
    // a cyclic interval of d residues (all of them when d >= 32), so the
    // T-weighted count of the warp is a sum of interval sums of T: one
    // prefix scan of T per read, then O(1) per lane per emulated warp.
    const unsigned long long tv = W.T[lane];
    unsigned long long incl = tv;
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long u = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += u;
    }
    const unsigned long long pex = incl - tv;                       // sum of T[0..lane)
    const unsigned long long tsum = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long total = 0;
    WarpWalk<ND> walk(h, ts, bs, cst, lane);
    for (int w = 0; w < nwarps; ++w, walk.next()) {
      bool active;
      const int64_t org = walk.origin(active);
      const int64_t up = __shfl_up_sync(0xffffffffu, org, 1);
      if (__all_sync(0xffffffffu, lane == 0 || !active || org >= up)) {
        unsigned long long c = 0;
        int lo = 0, hi = 0;
        if (active && lane > 0) {
          const int64_t d = org - up;
          if (d >= 32) c = tsum;
          else { lo = (int)((32 - d - (up & 31)) & 31); hi = lo + (int)d; }
        } else if (active) {
          c = tsum;                                                 // lane 0: the first segment
        }
        const unsigned long long plo = __shfl_sync(0xffffffffu, pex, lo);
        const unsigned long long phi = __shfl_sync(0xffffffffu, pex, hi & 31);
        if (hi > lo) c = hi <= 32 ? (hi == 32 ? tsum : phi) - plo : (tsum - plo) + phi;
        for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
        total += c;
      } else {
        for (int r = 0; r < 32; ++r) {
          const unsigned long long wr = __shfl_sync(0xffffffffu, tv, r);
          if (wr) total += wr * warp_count((unsigned long long)(org + r), active, tier, mm, bw_lg, bw, banks);
        }
      }
    }
    __syncwarp();
    GS_SUB(14);
    return total;
  }
  if (kFold4 && fold) {
    // shared banks, 4-byte words: each emulated warp is evaluated once per
    // constant residue mod 4 that occurs (one, for 4-byte elements)
    const unsigned ew = __ballot_sync(0xffffffffu, lane < 4 && tb != 0) & 0xFu;
    unsigned long long total = 0;
    WarpWalk<ND> walk(h, ts, bs, cst, lane);
    for (int w = 0; w < nwarps; ++w, walk.next()) {
      bool active;
      const int64_t org = walk.origin(active);
      unsigned m4 = ew;
      while (m4) {
        const int e = __ffs(m4) - 1; m4 &= m4 - 1;
        const unsigned long long we = __shfl_sync(0xffffffffu, tb, e);
        total += we * warp_count((unsigned long long)(org + e), active, tier, mm, bw_lg, bw, banks);
      }
    }
    __syncwarp();
    GS_SUB(14);
    return total;
  }
  // two classes: weights in H (class 0) and S (class 1); registers are
  // named, not indexed, so they stay out of local memory
  for (int j = 0; j < pp; ++j) { int r = lane + 32 * j; if (r < P) { W.GH[r] = 0; W.GS[r] = 0; } }
  __syncwarp();
  int ncls = 0;
  int64_t rel0 = 0, rel1 = 0, o00 = 0, o01 = 0;
  unsigned am0 = 0u, am1 = 0u;
  unsigned long long total = 0;
  WarpWalk<ND> walk(h, ts, bs, cst, lane);
  // Regular thread tiles — dim-0 rows of a multiple of 32 threads, or whole
  // rows whose length divides 32 stacked without wrapping — give every warp
  // warp 0's lane pattern: one class whose member shifts are the origins of
  // the warps' first threads (a scalar mixed-radix walk), folded into a
  // histogram of shifts mod P and one cyclic convolution with T.
  bool regular = false;
  if ((MC == 32 || MC == 128) && P <= 32 && (h.n_threads & 31) == 0) {
    const int cx = h.ctx[0];
    regular = (cx % 32 == 0) || (ND >= 2 && 32 % cx == 0 && h.ctx[ND >= 2 ? 1 : 0] % (32 / cx) == 0);
  }
  if (regular) {
    bool active;
    const int64_t org = walk.origin(active);
    o00 = __shfl_sync(0xffffffffu, org, 0);
    rel0 = org - o00;
    am0 = __ballot_sync(0xffffffffu, active);
    ncls = 1;
    int dg[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) dg[d] = 0;
    unsigned long long cnt = 0;   // lane d: members whose shift = d (mod P)
    for (int w = 0; w < nwarps; ++w) {
      int64_t dlt = 0;
#pragma unroll
      for (int d = 0; d < ND; ++d) dlt += (int64_t)dg[d] * walk.mul[d];
      cnt += (unsigned long long)(lane == (int)(dlt & (int64_t)(P - 1)));
      int carry = 0;
#pragma unroll
      for (int d = 0; d < ND; ++d) {
        dg[d] += walk.inc[d] + carry;
        carry = 0;
        if (d < ND - 1 && dg[d] >= walk.ext[d]) { dg[d] -= walk.ext[d]; carry = 1; }
      }
    }
    unsigned long long acc = 0;
    unsigned nzd = __ballot_sync(0xffffffffu, lane < P && cnt != 0);
    while (nzd) {
      const int d = __ffs(nzd) - 1; nzd &= nzd - 1;
      const unsigned long long cd = __shfl_sync(0xffffffffu, cnt, d);
      if (fold) acc += cd * __shfl_sync(0xffffffffu, tb, (lane - d) & (P - 1));
      else acc += cd * W.T[(lane - d) & (P - 1)];
    }
    if (lane < P) W.GH[lane] = acc;
    __syncwarp();
  }
  for (int w = 0; w < nwarps && !regular; ++w, walk.next()) {
    bool active;
    const int64_t org = walk.origin(active);
    const unsigned amask = __ballot_sync(0xffffffffu, active);
    const int64_t ow = __shfl_sync(0xffffffffu, org, 0);
    const int64_t rw = org - ow;
    int cls = -1;
    if (ncls > 0 && amask == am0 && __all_sync(0xffffffffu, !active || rw == rel0)) cls = 0;
    else if (ncls > 1 && amask == am1 && __all_sync(0xffffffffu, !active || rw == rel1)) cls = 1;
    else if (ncls == 0) { cls = 0; ncls = 1; rel0 = rw; am0 = amask; o00 = ow; }
    else if (ncls == 1) { cls = 1; ncls = 2; rel1 = rw; am1 = amask; o01 = ow; }
    if (cls >= 0) {
      const int64_t dlt = ow - (cls ? o01 : o00);
      unsigned long long* wv = cls ? W.GS : W.GH;
      if (fold) {
        const int src = (int)((lane - dlt) & (int64_t)(bw - 1));
        const unsigned long long add = __shfl_sync(0xffffffffu, tb, src);
        if (lane < bw) wv[lane] += add;
      } else {
        for (int j = 0; j < per; ++j) {
          const int k = lane + 32 * j;
          if (k < M) wv[k] += W.T[mm.pmod(k - dlt)];
        }
      }
      __syncwarp();
      continue;
    }
    // a third lane pattern: evaluate this warp directly
    if (fold) {                      // shared: the count depends on r mod bw only
      for (int e = 0; e < bw; ++e) {
        const unsigned long long we = __shfl_sync(0xffffffffu, tb, e);
        if (we) total += we * warp_count((unsigned long long)(org + e), active, tier, mm, bw_lg, bw, banks);
      }
      continue;
    }
    if (MC == 32 && tier == T_GLOBAL) {   // lanes = residues (see the class evaluation below)
      const int64_t up = __shfl_up_sync(0xffffffffu, org, 1);
      if (__all_sync(0xffffffffu, lane == 0 || !active || org >= up)) {
        const int na = __popc(amask);
        int64_t prev = ow + lane;
        unsigned cnt = na > 0 ? 1u : 0u;
#pragma unroll 4
        for (int i = 1; i < na; ++i) {
          const int64_t cur = __shfl_sync(0xffffffffu, org, i) + lane;
          cnt += (unsigned)((cur >> 5) != (prev >> 5));
          prev = cur;
        }
        unsigned long long part = W.T[lane] * cnt;
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        total += part;
        continue;
      }
    }
    for (int c = 0; c < per; ++c) {
      unsigned nz = __ballot_sync(0xffffffffu, (c * 32 + lane) < M && W.T[c * 32 + lane] != 0);
      while (nz) {
        const int b = __ffs(nz) - 1; nz &= nz - 1;
        const int r = c * 32 + b;
        total += W.T[r] * warp_count((unsigned long long)(org + r), active, tier, mm, bw_lg, bw, banks);
      }
    }
  }
  __syncwarp();
  GS_SUB(14);
  for (int j = 0; j < ncls; ++j) {
    const bool active = ((j ? am1 : am0) >> lane) & 1u;
    const int64_t org = j ? o01 + rel1 : o00 + rel0;
    const unsigned long long* wv = j ? W.GS : W.GH;
    if (MC == 32 && tier == T_GLOBAL) {
      // lanes = residues.  When the representative's lane addresses are
      // non-decreasing (row-major thread tiles), the segments of one
      // instruction are too, so its count is 1 + the segment changes
      // between consecutive active lanes: every residue at once, no match.
      const int64_t up = __shfl_up_sync(0xffffffffu, org, 1);
      if (__all_sync(0xffffffffu, lane == 0 || !active || org >= up)) {
        const int na = __popc(j ? am1 : am0);   // active lanes are a prefix
        int64_t prev = __shfl_sync(0xffffffffu, org, 0) + lane;
        unsigned cnt = na > 0 ? 1u : 0u;
#pragma unroll 4
        for (int i = 1; i < na; ++i) {
          const int64_t cur = __shfl_sync(0xffffffffu, org, i) + lane;
          cnt += (unsigned)((cur >> 5) != (prev >> 5));
          prev = cur;
        }
        unsigned long long part = wv[lane] * cnt;
        for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        total += part;
        continue;
      }
    }
    for (int c = 0; c < pp; ++c) {
      unsigned nz = __ballot_sync(0xffffffffu, (c * 32 + lane) < P && wv[c * 32 + lane] != 0);
      while (nz) {
        const int b = __ffs(nz) - 1; nz &= nz - 1;
        const int r = c * 32 + b;
        total += wv[r] * warp_count((unsigned long long)(org + r), active, tier, mm, bw_lg, bw, banks);
      }
    }
  }
  __syncwarp();
  GS_SUB(15);
  return total;
}

// ---------------------------------------------------------------------------
// one feature row (warp)
// ---------------------------------------------------------------------------
enum FeatIdx {
  F_NUM_SCALARS = 0, F_PTS_PER_THREAD = 1, F_UG_REAL = 2, F_UG_THREAD = 8, F_ALLOC_G = 14,
  F_G_AT_TASK = 17, F_GI_AT_TASK = 20, F_NUM_BLOCKS = 23, F_WARPS_PB = 24, F_ACTIVE_WARPS = 25,
  F_THREADS_PB = 26, F_EXPR = 27, F_BLOCK_OCC = 28, F_WARP_UTIL = 29, F_IDLE = 30,
  F_SH_LOADS = 31, F_GL_LOADS = 32, F_SH_STORES = 33, F_GL_STORES = 34, F_SH_ST_EFF = 35,
  F_SH_LD_EFF = 36, F_GL_ST_EFF = 37, F_GL_LD_EFF = 38, F_WS_THREAD = 39, F_SH_OCC = 40,
  F_SH_LIMIT = 41, F_MAX_WARP_OCC = 42, F_MAX_BLOCK_OCC = 43, F_NUM_REAL = 44, F_NUM_PROD = 45,
  F_NUM_TASKS = 46, F_INNER_PAR = 47, F_TASKS_PER_CORE = 48, F_NUM_CORES = 49, F_INLINED = 50,
  F_UB_POINT = 51, F_UL_POINT = 52, F_UB_TASK = 53, F_UL_TASK = 54, F_WORKING_SET = 55
};

template <int ND>
__device__ __forceinline__ void parallel_feats(double* v, const GsMachine& M, int n, const CF<ND>& kern) {
  // featurize.py:317-363, warp-wide: every lane derives the integer
  // occupancy terms (thread / warp / block counts are < 2^31: 32-bit
  // division), then lane i forms feature i as ONE quotient, so the eight
  // IEEE divisions run side by side and exist once in the instruction
  // stream.  Quotients by 1 are the integer values themselves.
  const int lane = lane_id();
  const int kt = kern.k_threads, ws = M.warp_size;
  const bool w32 = ws == 32;   // the common warp: shifts instead of divisions
  const int aw = w32 ? (n + 31) >> 5 : (n + ws - 1) / ws;
  const int kw = w32 ? (kt + 31) >> 5 : (kt + ws - 1) / ws;
  int wpb = kw;
  if (wpb < 1) wpb = 1;
  int by_shared;
  if (kern.k_shared > 0) {
    // shared_mem_per_sm fits 32 bits; a kernel needing more than that
    // fits zero blocks
    by_shared = kern.k_shared > (int64_t)M.shared_mem_per_sm ? 0 : M.shared_mem_per_sm / (int)kern.k_shared;
    if (by_shared < 1) by_shared = 1;
  } else {
    by_shared = M.max_active_blocks_per_sm;
  }
  const int mb = M.max_active_blocks_per_sm;
  int act = mb;
  if (by_shared < act) act = by_shared;
  if (M.max_active_warps_per_sm / wpb < act) act = M.max_active_warps_per_sm / wpb;
  if (act < 1) act = 1;
  int64_t awsm = (int64_t)act * wpb;
  if (awsm > M.max_active_warps_per_sm) awsm = M.max_active_warps_per_sm;
  // operands selected per lane without branching (a switch on the lane
  // would serialise fifteen divergent paths)
  const bool shp = kern.k_shared > 0;
  const double nb = (double)kern.n_blocks, nn = (double)n, mt = (double)M.max_threads_per_block;
  double num = 0.0, den = 1.0;
  num = lane == 0 || lane == 11 || lane == 14 ? nb : num;
  num = lane == 1 ? (double)kw : num;
  num = lane == 2 ? (double)aw : num;
  num = lane == 3 || lane == 4 || lane == 12 ? nn : num;
  num = lane == 5 ? (double)(ws * aw - n) : num;
  num = lane == 6 ? (double)kt : num;
  num = lane == 7 && shp ? (double)kern.k_shared : num;
  num = lane == 8 ? (double)(by_shared < mb ? by_shared : mb) : num;
  num = lane == 9 ? (double)awsm : num;
  num = lane == 10 ? (double)act : num;
  num = lane == 13 ? (double)M.num_sms : num;
  den = lane == 4 ? (double)(ws * aw) : den;
  den = lane == 5 || lane == 6 ? mt : den;
  den = lane == 7 && shp ? (double)M.shared_mem_per_block_limit : den;
  den = lane == 8 || lane == 10 ? (double)mb : den;
  den = lane == 9 ? (double)M.max_active_warps_per_sm : den;
  den = lane == 14 ? (double)M.num_sms : den;
  const bool clamp = lane == 7 && shp;
  // feature index of lane i: 6-bit fields of two constants (no local array)
  constexpr unsigned long long kIdxLo =
      (unsigned long long)F_NUM_BLOCKS | (unsigned long long)F_WARPS_PB << 6 |
      (unsigned long long)F_ACTIVE_WARPS << 12 | (unsigned long long)F_THREADS_PB << 18 |
      (unsigned long long)F_WARP_UTIL << 24 | (unsigned long long)F_IDLE << 30 |
      (unsigned long long)F_BLOCK_OCC << 36 | (unsigned long long)F_SH_OCC << 42 |
      (unsigned long long)F_SH_LIMIT << 48 | (unsigned long long)F_MAX_WARP_OCC << 54;
  constexpr unsigned long long kIdxHi =
      (unsigned long long)F_MAX_BLOCK_OCC | (unsigned long long)F_NUM_TASKS << 6 |
      (unsigned long long)F_INNER_PAR << 12 | (unsigned long long)F_NUM_CORES << 18 |
      (unsigned long long)F_TASKS_PER_CORE << 24;
  const int idx = lane < 10 ? (int)((kIdxLo >> (6 * lane)) & 63) : lane < 15 ? (int)((kIdxHi >> (6 * (lane - 10))) & 63) : -1;
  double q = num / den;
  if (clamp && !(q < 1.0)) q = 1.0;
  if (idx >= 0) v[idx] = q;
}


template <int ND>
__device__ __forceinline__ void row_features(K1<ND>& k, WarpScr& W, int func, int si, bool inl, double* out) {
  const int lane = lane_id();
#ifdef GS_PHASES
  long long tsub = clock64();
#endif
  const GsMachine& M = k.P->m;
  Misc& m = *k.misc;
  const CF<ND>& g = k.cf[func];
  const GsFunc& fn = k.F[func];
  const int gstage = fn.stage_begin + si;
  int err = 0;
  // defaults (featurize.py:78-147), one lane per feature
  {
    constexpr unsigned long long kOnes =
        (1ull << F_BLOCK_OCC) | (1ull << F_WARP_UTIL) | (1ull << F_SH_ST_EFF) | (1ull << F_SH_LD_EFF) |
        (1ull << F_GL_ST_EFF) | (1ull << F_GL_LD_EFF) | (1ull << F_SH_LIMIT) | (1ull << F_MAX_WARP_OCC) |
        (1ull << F_MAX_BLOCK_OCC) | (1ull << F_INNER_PAR) | (1ull << F_NUM_CORES);
    const double br = (double)k.ST[gstage].branching;
    for (int i = lane; i < GS_NUM_FEATURES; i += 32)
      W.feat[i] = i == F_EXPR ? br : ((kOnes >> i) & 1ull) ? 1.0 : 0.0;
    if (lane < 24) (&W.acc[0][0][0])[lane] = 0ull;
  }
  __syncwarp();
  const CF<ND>* hp = inl ? (g.consumer >= 0 ? &k.cf[g.consumer] : nullptr) : &g;
  if (inl && hp == nullptr) {
    if (lane == 0) {
      W.feat[F_INLINED] = (double)(g.calls > 1 ? g.calls : 1);
      W.feat[F_NUM_SCALARS] = (double)g.calls;
    }
    __syncwarp();
    for (int i = lane; i < GS_NUM_FEATURES; i += 32) out[i] = W.feat[i];
    return;
  }
  const CF<ND>& h = *hp;
  const CF<ND>& kern = k.cf[h.kernel];
  // ---- reads attributed to this row, in order
  int lo_r = inl ? 0 : k.rdb[2 * gstage], hi_r = inl ? m.nreads : k.rdb[2 * gstage + 1];
  int nr = 0;
  for (int j0 = lo_r; j0 < hi_r; j0 += 32) {
    int j = j0 + lane;
    bool hit = j < hi_r && k.rd[j].owner == func;
    unsigned bal = __ballot_sync(0xffffffffu, hit);
    int pos = nr + __popc(bal & ((1u << lane) - 1));
    if (hit && pos < kRowReads) W.rl[pos] = (int16_t)j;
    nr += __popc(bal);
  }
  if (nr > kRowReads) { if (lane == 0) atomicOr(k.gerr, E_ROWREADS); nr = kRowReads; }
  __syncwarp();
  // (tier, producer) groups in first-appearance order: one lane per read
  if (nr <= 32) {
    bool has = lane < nr;
    const RRead* r = has ? &k.rd[W.rl[lane]] : nullptr;
    const unsigned key = has ? ((unsigned)(uint8_t)r->tier << 16) | (uint16_t)r->producer : 0xFFFFFFFFu - lane;
    const unsigned same = __match_any_sync(0xffffffffu, key);
    const int leader = __ffs(same) - 1;
    const unsigned leaders = __ballot_sync(0xffffffffu, has && leader == lane);
    const int gi = __popc(leaders & ((1u << leader) - 1));
    if (has) {
      W.grp[lane] = (int8_t)gi;
      if (leader == lane) { W.gtier[gi] = r->tier; W.gprod[gi] = r->producer; }
    }
    if (lane == 0) { W.ngroups = __popc(leaders); W.nr = nr; }
  } else if (lane == 0) {
    int ng = 0;
    for (int q = 0; q < nr; ++q) {
      const RRead& r = k.rd[W.rl[q]];
      int gi = -1;
      for (int t = 0; t < ng; ++t) if (W.gtier[t] == r.tier && W.gprod[t] == r.producer) { gi = t; break; }
      if (gi < 0) { gi = ng++; W.gtier[gi] = r.tier; W.gprod[gi] = r.producer; }
      W.grp[q] = (int8_t)gi;
    }
    W.ngroups = ng;
    W.nr = nr;
  }
  __syncwarp();
  parallel_feats(W.feat, M, h.n_threads, kern);
  __syncwarp();
  const int ng = W.ngroups;
  GS_SUB(8);
  // ---- unions: tasks (box, group); boxes 0 region, 1 lane, 2 point, 3 block
  const int nbox_tasks = 4 * ng;
  for (int t = lane; t < nbox_tasks; t += 32) {
    const int box = t / ng, gi = t % ng;
    if (box == 0 && inl) continue;
    int32_t blo[ND], bhi[ND];
    if (box == 0) { for (int d = 0; d < ND; ++d) { blo[d] = g.rlo[d]; bhi[d] = g.rhi[d]; } }
    else if (box == 1) { for (int d = 0; d < ND; ++d) { blo[d] = h.base[d]; bhi[d] = h.base[d] + h.ext[d] - 1; } }
    else if (box == 2) { for (int d = 0; d < ND; ++d) { blo[d] = bhi[d] = h.base[d]; } }
    else block_box(h, blo, bhi);
    int64_t vol, lines;
    if (!union_count_one<ND>(k.A, k.rd, k.path, W.rl, W.grp, nr, gi, blo, bhi, vol, lines))
      union_count<ND>(k.A, k.rd, k.path, W.rl, W.grp, nr, gi, blo, bhi, vol, lines, err);
    const int eb = k.F[W.gprod[gi]].elem_bytes;
    atomicAdd(&W.acc[box][W.gtier[gi]][0], (unsigned long long)(vol * eb));
    atomicAdd(&W.acc[box][W.gtier[gi]][1], (unsigned long long)lines);
  }
  __syncwarp();
  GS_SUB(9);
  // ---- loads (block 0 of the host's kernel)
  // the default machine (32 B transactions, 32 banks x 4 B) gets the
  // compile-time-specialised counter
  const bool vdef = M.global_transaction_bytes == 32 && M.shared_banks == 32 && M.bank_width_bytes == 4;
  auto tx = [&](const int16_t* path, int plen, bool identity, const CF<ND>& host, const CF<ND>& prod, int eb,
                int tier) -> unsigned long long {
    if (vdef) {
      if (tier == T_GLOBAL) return tx_global32<ND>(k.A, path, plen, identity, host, prod, eb, W, err);
      return tx_shared4<ND>(k.A, path, plen, identity, host, prod, eb, W, err);
    }
    return warp_tx<ND, 0, 0, 0>(k.A, path, plen, identity, host, prod, eb, tier, M, W, err);
  };
  // one call site for loads and the store (q == nr) keeps a single copy of
  // the counters in the instruction stream
  unsigned long long ld[2] = {0, 0}, st = 0;
#pragma unroll 1
  for (int q = 0; q <= nr; ++q) {
    const bool store = q == nr;
    const RRead* r = store ? nullptr : &k.rd[W.rl[q]];
    const int tier = store ? (inl ? -1 : g.tier) : r->tier;
    if (tier != T_GLOBAL && tier != T_SHARED) continue;
    const int pr = store ? func : r->producer;
    const unsigned long long c = tx(store ? nullptr : k.path + r->pbeg, store ? 0 : r->plen, store, store ? g : h,
                                    k.cf[pr], k.F[pr].elem_bytes, tier);
    if (store) st = c; else ld[tier] += c;
  }
  GS_SUB(13);
  GS_SUB(10);
  // ---- working set at thread: fuse_at_thread children (featurize.py:482-492)
  int64_t wsc = 0;
  if (!inl) {
    for (int f2 = lane; f2 < k.P->nf; f2 += 32) {
      const CF<ND>& o = k.cf[f2];
      if (o.kind == K_THREAD && o.consumer == func) wsc += alloc_of(o) * k.F[f2].elem_bytes;
    }
    for (int o = 16; o; o >>= 1) wsc += __shfl_xor_sync(0xffffffffu, wsc, o);
  }
  GS_SUB(11);
  int lerr = err;
  for (int o = 16; o; o >>= 1) lerr |= __shfl_xor_sync(0xffffffffu, lerr, o);
  double* v = W.feat;
  const int gtx = M.global_transaction_bytes, stx = M.shared_banks * M.bank_width_bytes;
  // lane-parallel part of the assembly: the union counts (acc[box][tier]
  // [bytes, lines]) as features, the per-task / per-point sums over tiers
  // (the reference sums ints: integer sums), loads and load efficiencies
  if (lane < 12) {
    const int b = lane / 6, t = (lane % 6) >> 1, w = lane & 1;   // box 0 realization, 1 thread
    if (b == 1 || !inl) v[(b == 1 ? F_UG_THREAD : F_UG_REAL) + 3 * w + t] = (double)W.acc[b][t][w];
  } else if (lane < 16) {
    const int b = lane < 14 ? 3 : 2, w = lane & 1;                // box 3 task, 2 point
    const int idx = lane == 12 ? F_UB_TASK : lane == 13 ? F_UL_TASK : lane == 14 ? F_UB_POINT : F_UL_POINT;
    v[idx] = (double)(W.acc[b][0][w] + W.acc[b][1][w] + W.acc[b][2][w]);
  } else if (lane < 18) {
    const int t = lane - 16;                                       // 0 global, 1 shared
    const double loads = (double)ld[t];
    v[t == 0 ? F_GL_LOADS : F_SH_LOADS] = loads;
    if (loads > 0) {
      const double e = (double)W.acc[3][t][0] / (loads * (t == 0 ? gtx : stx));
      v[t == 0 ? F_GL_LD_EFF : F_SH_LD_EFF] = e < 1.0 ? e : 1.0;
    }
  }
  __syncwarp();
  if (lane == 0) {
    if (lerr) atomicOr(k.gerr, lerr);
    if (inl) {
      v[F_INLINED] = (double)g.calls;
      v[F_NUM_SCALARS] = (double)g.calls;
      const int64_t den = kern.n_blocks * (int64_t)h.n_threads;
      v[F_PTS_PER_THREAD] = den ? (double)g.calls / (double)den : 0.0;
    } else {
      const int64_t ppt = prod_ext(g), ppb = ppt * g.n_threads;
      v[F_NUM_SCALARS] = (double)(ppb * kern.n_blocks);
      v[F_PTS_PER_THREAD] = (double)ppt;
      v[F_NUM_REAL] = v[F_NUM_PROD] = (double)g.realizations;
      int64_t alloc[3] = {0, 0, 0};
      for (int gi = 0; gi < ng; ++gi)
        alloc[W.gtier[gi]] += alloc_of(k.cf[W.gprod[gi]]) * k.F[W.gprod[gi]].elem_bytes;
      for (int t = 0; t < 3; ++t) v[F_ALLOC_G + t] = (double)alloc[t];
      const int eb = fn.elem_bytes;
      const int64_t written = ppb * eb;
      int32_t blo[ND], bhi[ND];
      block_box(g, blo, bhi);
      v[F_G_AT_TASK + g.tier] = (double)written;
      v[F_GI_AT_TASK + g.tier] = (double)(((int64_t)bhi[0] - blo[0] + 1) * eb);
      if (g.tier == T_GLOBAL) v[F_GL_STORES] = (double)st;
      else if (g.tier == T_SHARED) v[F_SH_STORES] = (double)st;
      if (g.tier == T_GLOBAL && st > 0) {
        double e = (double)written / (double)(st * (unsigned long long)gtx); v[F_GL_ST_EFF] = e < 1.0 ? e : 1.0;
      } else if (g.tier == T_SHARED && st > 0) {
        double e = (double)written / (double)(st * (unsigned long long)stx); v[F_SH_ST_EFF] = e < 1.0 ? e : 1.0;
      }
      const int64_t al = alloc_of(g);
      int64_t wsi = (g.tier == T_REGISTER ? al * eb : 0) + wsc;
      double wsd = (double)wsi;
      if (g.unrolled) { wsd += v[F_UG_THREAD + 0]; wsd += v[F_UG_THREAD + 1]; }
      v[F_WS_THREAD] = wsd;
      v[F_WORKING_SET] = (double)(al * eb);
    }
  }
  __syncwarp();
  for (int i = lane; i < GS_NUM_FEATURES; i += 32) out[i] = W.feat[i];
  GS_SUB(12);
}

// ---------------------------------------------------------------------------
// kernel
// ---------------------------------------------------------------------------
// TMA bulk copy global -> shared completing on an mbarrier.  Thread 0
// initialises the barrier; the CTA barrier that follows makes the
// initialisation visible before anyone waits on it; thread 0 then posts the
// expected bytes and issues the copy.
__device__ __forceinline__ void bulk_init(uint64_t* bar) {
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
  asm volatile("fence.mbarrier_init.release.cluster;");
}
__device__ __forceinline__ void bulk_stage(void* dst_smem, const void* src, int bytes, uint64_t* bar) {
  unsigned dst = (unsigned)__cvta_generic_to_shared(dst_smem);
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
               ::"r"(dst), "l"(src), "r"(bytes), "r"(b) : "memory");
}
__device__ __forceinline__ void bulk_wait(uint64_t* bar) {
  unsigned b = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                 : "=r"(done) : "r"(b) : "memory");
  }
}

// Every warp is an independent scorer: it walks its own contiguous range of
// candidates (consecutive candidates of a beam step are siblings), keeping
// its decision structure, geometry and scratch in its own slice of shared
// memory; the candidate-independent pipeline descriptor is shared by the
// CTA.  The warps take their candidates in lockstep: a CTA barrier separates
// each candidate's resolve phase from its feature-row phase (see the main loop).

template <int ND>
__global__ void __launch_bounds__(kK1MaxWarps * 32, 1)
featurize_kernel(const PipeDev* __restrict__ P, const uint8_t* __restrict__ blob, const GsDecision* __restrict__ dec,
                 int64_t n, int S, double* __restrict__ feats, int32_t* __restrict__ row_key,
                 int32_t* __restrict__ n_rows, uint8_t* __restrict__ verdict, int32_t* __restrict__ row_src,
                 Layout L, int* gerr, int reuse, uint8_t* __restrict__ gscratch, const uint8_t* __restrict__ heads,
                 int mode, const int32_t* __restrict__ run_id, const int32_t* __restrict__ run_head,
                 const uint32_t* __restrict__ nruns_dev, int64_t max_runs,
                 uint8_t* __restrict__ slots, int64_t slot_bytes, int32_t* __restrict__ row_kernel) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ uint64_t bar;
  const int warp = threadIdx.x >> 5, lane = lane_id(), nw = blockDim.x >> 5;
  // Two-phase launches read the run count the preparation kernels left on
  // the device.  Too many runs for the slots, or runs shorter than 8 on
  // average: the run-head launch does the one-phase (run-aligned unit)
  // schedule instead and the sibling launch has nothing to do.
  int64_t nruns = 0;
  if (mode != 0) {
    nruns = (int64_t)*nruns_dev;
    if (nruns > max_runs || nruns * 8 > n) {
      if (mode == 2) return;
      mode = 0;
    }
  }
  if (threadIdx.x == 0) bulk_init(&bar);
  __syncthreads();
  if (threadIdx.x == 0) bulk_stage(sm + L.blob, blob, P->blob_bytes, &bar);
  uint8_t* ws = sm + L.warps + (size_t)warp * L.warp_bytes;   // this warp's slice
  // capacity-sized structure arrays live in the slice, or — for pipelines
  // whose worst-case inline expansion does not fit shared memory — in this
  // warp's slice of a global scratch (generic pointers: same code)
  uint8_t* wgs = gscratch + ((size_t)blockIdx.x * (blockDim.x >> 5) + warp) * L.gl_bytes;
  // warp w's scorer state
  auto bind = [&](K1<ND>& k, int w) {
    uint8_t* ws = sm + L.warps + (size_t)w * L.warp_bytes;
    uint8_t* wgs = gscratch + ((size_t)blockIdx.x * (blockDim.x >> 5) + w) * L.gl_bytes;
    // spill level 1: the resolve-side capacity arrays in global scratch;
    // level 2: also the expanded reads and chain paths the rows walk
    uint8_t* wg = L.spill >= 1 ? wgs : ws;
    uint8_t* wg2 = L.spill >= 2 ? wgs : ws;
    k.P = P;
    k.F = reinterpret_cast<const GsFunc*>(sm + L.blob);
    k.ST = reinterpret_cast<const GsStage*>(sm + L.blob + P->off_stages);
    k.A = reinterpret_cast<const GsAccess*>(sm + L.blob + P->off_access);
    k.dec = reinterpret_cast<GsDecision*>(ws + L.dec);
    k.didx = reinterpret_cast<int16_t*>(ws + L.didx);
    k.cf = reinterpret_cast<CF<ND>*>(ws + L.cf);
    k.rd = reinterpret_cast<RRead*>(wg2 + L.reads);
    k.path = reinterpret_cast<int16_t*>(wg2 + L.paths);
    k.rdb = reinterpret_cast<int32_t*>(ws + L.rdb);
    k.rows = reinterpret_cast<int32_t*>(ws + L.rows);
    k.stack = reinterpret_cast<Frame*>(wgs + L.stack);       // structure-build scratch: global
    k.volacc = reinterpret_cast<int64_t*>(wgs + L.volacc);
    k.touched = reinterpret_cast<int16_t*>(wgs + L.touched);
    k.icall = reinterpret_cast<ICall*>(wgs + L.icall);
    k.srcb = reinterpret_cast<int32_t*>(ws + L.srcb);
    k.srcl = reinterpret_cast<int16_t*>(wg + L.srcl);
    k.rdepb = reinterpret_cast<int32_t*>(ws + L.rdepb);
    k.rdep = reinterpret_cast<int16_t*>(wg2 + L.rdep);
    k.dirty = reinterpret_cast<uint8_t*>(ws + L.dirty);
    k.rowlist = reinterpret_cast<int16_t*>(ws + L.rowlist);
    k.kern = reinterpret_cast<int16_t*>(ws + L.kern);
    k.dm = reinterpret_cast<uint32_t*>(wgs + L.dm);          // dependency masks: global (L1)
    k.cmask = reinterpret_cast<uint32_t*>(ws + L.cmask);
    k.kmb = reinterpret_cast<int32_t*>(wg + L.kmb);
    k.kml = reinterpret_cast<int16_t*>(wg + L.kml);
    k.icb = reinterpret_cast<int32_t*>(wg + L.icb);
    k.icl = reinterpret_cast<int16_t*>(wgs + L.icl);
    k.dlist = reinterpret_cast<int16_t*>(wg + L.dlist);
    k.gdirty = reinterpret_cast<uint8_t*>(ws + L.gdirty);
    k.kdirty = reinterpret_cast<uint8_t*>(ws + L.kdirty);
    k.misc = reinterpret_cast<Misc*>(ws + L.misc);
    k.rcap = L.rcap; k.pcap = L.pcap; k.gerr = gerr; k.mw = L.mw; k.track = false;
  };
  K1<ND> k;
  bind(k, warp);
  WarpScr& W = *reinterpret_cast<WarpScr*>(ws + L.scr);
  int* s_nd = reinterpret_cast<int*>(sm + L.cta);                  // [nw] dirty rows of each warp's candidate
  int* s_next = s_nd + kK1MaxWarps;                               // next pooled row
  int64_t* s_cand = reinterpret_cast<int64_t*>(sm + L.cta + 64);   // [nw] each warp's candidate
  uint8_t* rflag = ws + L.rflag;
  int32_t* rsrc = reinterpret_cast<int32_t*>(ws + L.rsrc);
  // Work units: kUnit-candidate slices of the batch, each extended to start
  // and end at a decision-structure run head, handed out dynamically; a unit
  // therefore never splits a run of siblings (whose first member needs the
  // full resolve anyway), and warps that drew cheap runs take more of them.
  Misc& m = *k.misc;
  unsigned long long st_cand = 0, st_inc = 0, st_rows = 0, st_emit = 0, st_geo = 0;   // (lane 0)
#ifdef GS_PHASES
  long long ph[8] = {0, 0, 0, 0, 0, 0, 0, 0}, tph = 0;
#endif
  unsigned* work = reinterpret_cast<unsigned*>(gerr + 14);
  // Small batches (a search phase of a few hundred candidates) take smaller
  // units so every scorer warp gets work; below 16 candidates per unit runs
  // are split (latency over sibling reuse).
  const int64_t twarps = (int64_t)gridDim.x * nw;
  const int64_t unit = n >= (int64_t)kUnit * twarps ? kUnit : (n + twarps - 1) / twarps;
  const int64_t nunits = (n + unit - 1) / unit;
  const bool snapping = unit >= 16;
  auto snap = [&](int64_t x) -> int64_t {
    if (x >= n) return n;
    if (!heads || !snapping) return x;
    for (int64_t i = x; i < n; i += 32) {
      const bool h = i + lane < n && heads[i + lane];
      const unsigned b = __ballot_sync(0xffffffffu, h);
      if (b) return i + __ffs(b) - 1;
    }
    return n;
  };
  // Modes (see launch_featurize): 0 run-aligned units; 1 run heads only,
  // each head's warp state saved to its run's slot; 2 siblings in kChunk2
  // slices, a slice resuming from its run head's saved state (no re-resolve,
  // no row recompute), so runs split freely across warps.
  // The last ~2 slices per warp are cut 4x finer (8 candidates), so the
  // launch does not end waiting on a few warps' full 32-candidate slices;
  // a slice costs one 26 KB state restore, small against 8 candidates.
  const int64_t nbig_all = (n + kChunk2 - 1) / kChunk2;
  const int64_t tail_big = 3 * (int64_t)gridDim.x * nw < nbig_all ? 3 * (int64_t)gridDim.x * nw : nbig_all;
  const int64_t nbig = nbig_all - tail_big;
  constexpr int kFine = kChunk2 / 4 > 0 ? kChunk2 / 4 : 1;
  const int64_t nchunks = nbig + (n - nbig * kChunk2 + kFine - 1) / kFine;
  // warp state <-> run slot: the shared-memory slice and the global scratch
  // copy n int4 from src to dst with eight loads in flight per lane before
  // their stores (a load-store-load loop waited one HBM round trip per
  // 512 bytes: ~36 of them to restore a slot)
  auto copy16 = [&](int4* __restrict__ dst, const int4* __restrict__ src, int n) {
    constexpr int U = 8;
    int i = lane;
    for (; i + 32 * (U - 1) < n; i += 32 * U) {
      int4 t[U];
#pragma unroll
      for (int u = 0; u < U; ++u) t[u] = src[i + 32 * u];
#pragma unroll
      for (int u = 0; u < U; ++u) dst[i + 32 * u] = t[u];
    }
    for (; i < n; i += 32) dst[i] = src[i];
  };
  auto slot_copy = [&](int64_t r, bool save) {
    uint8_t* sl = slots + r * slot_bytes;
    int4* a = reinterpret_cast<int4*>(sl);
    int4* b = reinterpret_cast<int4*>(ws);
    const int nw1 = L.keep / 16;
    int4* a2 = reinterpret_cast<int4*>(sl + L.keep);
    int4* b2 = reinterpret_cast<int4*>(wgs);
    const int nw2 = L.gkeep / 16;
    if (save) { copy16(a, b, nw1); copy16(a2, b2, nw2); }
    else { copy16(b, a, nw1); copy16(b2, a2, nw2); }
    __syncwarp();
  };
  bulk_wait(&bar);
  __syncthreads();   // descriptor staged
  // Per-candidate work, in two phases: A (records, diff, resolve, prune,
  // row flags) and B (rows and outputs).
  int nr = 0, nd = 0;
  bool diffable = false;
  auto phaseA = [&](int64_t c, int64_t pc) {
    if (lane == 0) st_cand++;
#ifdef GS_PHASES
    tph = clock64();
#endif
    {
      const uint4* src = reinterpret_cast<const uint4*>(dec + c * S);
      uint4* dst = reinterpret_cast<uint4*>(k.dec);
      for (int i = lane; i < S; i += 32) dst[i] = __ldg(src + i);   // 128-bit loads
      if (lane < k.mw) k.cmask[lane] = 0u;
      __syncwarp();
      unsigned cnt = 0, diff = 0;
      // the previous candidate's records: still in L2 (this warp just read them)
      const uint4* prv = reinterpret_cast<const uint4*>(dec + pc * S);
      for (int i0 = 0; i0 < S; i0 += 32) {
        const int i = i0 + lane;
        const bool live = i < S && k.dec[i].func != 0xFFFF;
        cnt += __popc(__ballot_sync(0xffffffffu, live));
        bool d = false;
        if (i < S) {
          const uint4 x = reinterpret_cast<const uint4*>(k.dec)[i];
          const uint4 y = __ldg(prv + i);
          // func | consumer << 16 in .x, kind in the low byte of .y
          d = x.x != y.x || ((x.y ^ y.y) & 0xFFu) != 0u;
          if (live && k.mw > 0 && !d && (x.y != y.y || x.z != y.z || x.w != y.w))
            atomicOr(&k.cmask[k.dec[i].func >> 5], 1u << (k.dec[i].func & 31));
        }
        diff |= __ballot_sync(0xffffffffu, d);
      }
      __syncwarp();
#ifdef GS_DEBUG_DIFF
      if (lane == 0 && n < 64) printf("c=%lld pc=%lld diff=%x prev_valid=%d cnt=%u ndec=%d mode=%d\n", (long long)c, (long long)pc, diff, m.prev_valid, cnt, m.ndec, mode);
#endif
      if (lane == 0) {
        m.same_struct = reuse && m.prev_valid && diff == 0 && (int)cnt == m.ndec;
        m.ndec = (int)cnt; m.err = 0; m.ngeo = 0;
        if (!m.same_struct) m.nrows = 0;
      }
      __syncwarp();
      GS_MARK(0);
    }
  };
  auto phaseResolve = [&]() { resolve<ND>(k); };
  auto phaseA2 = [&](int64_t c, int64_t pc) {
    {
      GS_MARK(1);
      const int v = m.err ? 255 : prune_verdict<ND>(k);
      GS_MARK(2);
      if (lane == 0) {
        if (m.err) { atomicOr(gerr, m.err); m.nrows = 0; }
        verdict[c] = (uint8_t)v;
        n_rows[c] = m.nrows;
      }
      __syncwarp();
    }
    nr = feats ? m.nrows : 0;   // feats == NULL: prune verdict only
    diffable = m.same_struct && !m.err;
    // rows to recompute: own func, host, host kernel, read producers and
    // fuse_at_thread children unchanged => features are bit-identical
    nd = 0;
    for (int r0 = 0; r0 < nr; r0 += 32) {
      const int r = r0 + lane;
      bool d = false;
      if (r < nr) {
        d = true;
        if (diffable) {
          const int f = k.rows[r] >> 8;
          const CF<ND>& g = k.cf[f];
          const int host = g.kind == K_INLINE ? g.consumer : f;
          d = k.dirty[f] & 1;
          // own and host records: any field; the host's kernel: its aggregates
          if (host >= 0) { d |= k.dirty[host] & 1; if (k.cf[host].kernel >= 0) d |= (k.dirty[k.cf[host].kernel] >> 2) & 1; }
          // read producers / thread children: only their layout matters
          for (int q = k.rdepb[r]; q < k.rdepb[r + 1] && !d; ++q) d |= (k.dirty[k.rdep[q]] >> 1) & 1;
        }
        rflag[r] = d;
        if (d) rsrc[r] = (int32_t)c;
      }
      const unsigned b = __ballot_sync(0xffffffffu, d);
      if (d) k.rowlist[nd + __popc(b & ((1u << lane) - 1))] = (int16_t)r;
      nd += __popc(b);
    }
    __syncwarp();
    if (lane == 0) { st_inc += m.same_struct; st_rows += nd; st_emit += nr; st_geo += m.ngeo; }
  };
  auto phaseB = [&](int64_t c, int64_t pc) {
    // a sibling starts from the previous candidate's feature block (this
    // warp wrote it: visible after __syncwarp), copied as one contiguous run
    // of 16-byte vectors with four loads in flight per lane; the dirty rows
    // are then recomputed over it
    GS_MARK(3);
    if (diffable && nd < nr && reuse != 2) {
      const int4* src = reinterpret_cast<const int4*>(feats + (int64_t)pc * L.R * GS_NUM_FEATURES);
      int4* dst = reinterpret_cast<int4*>(feats + (int64_t)c * L.R * GS_NUM_FEATURES);
      const int nv = nr * (GS_NUM_FEATURES * 8 / 16);
      int i = lane;
      for (; i + 96 < nv; i += 128) {
        const int4 a0 = src[i], a1 = src[i + 32], a2 = src[i + 64], a3 = src[i + 96];
        dst[i] = a0; dst[i + 32] = a1; dst[i + 64] = a2; dst[i + 96] = a3;
      }
      for (; i < nv; i += 32) dst[i] = src[i];
      __syncwarp();
    }
    GS_MARK(4);
  };
  // row q of candidate c, scorer state `ko`
  auto phaseRow = [&](K1<ND>& ko, int64_t c, int q) {
    const int r = ko.rowlist[q];
    const int key = ko.rows[r];
    const int f = key >> 8, si = key & 255;
    row_features<ND>(ko, W, f, si, ko.cf[f].kind == K_INLINE, feats + ((int64_t)c * L.R + r) * GS_NUM_FEATURES);
  };
  auto phaseB3 = [&](int64_t c) {
    GS_MARK(5);
    for (int r = lane; r < nr; r += 32) {
      row_key[c * L.R + r] = k.rows[r];
      if (row_src) row_src[c * L.R + r] = rsrc[r];
      if (row_kernel) {
        // the row's kernel (resolve.py:251-355: an inline func runs in its
        // primary consumer's kernel), bit 30 = that kernel breaks a hardware
        // limit (machine.py:91-105 validate_limits)
        const CF<ND>& g = k.cf[k.rows[r] >> 8];
        const int kk = g.kind == K_INLINE ? (g.consumer >= 0 ? k.cf[g.consumer].kernel : -1) : g.kernel;
        int32_t v = kk;
        if (kk >= 0 && (k.cf[kk].k_threads > k.P->m.max_threads_per_block ||
                        k.cf[kk].k_shared > (int64_t)k.P->m.shared_mem_per_block_limit))
          v |= 0x40000000;
        row_kernel[c * L.R + r] = v;
      }
    }
    __syncwarp();
    GS_MARK(6);
    if (lane == 0) m.prev_valid = m.err == 0;   // geometry reuse holds with or without feature rows
    __syncwarp();
  };
  // The CTA's warps take their candidates in lockstep: every warp runs
  // phase A (records, diff, resolve, prune, row flags) for its next
  // candidate, a CTA barrier, then phase B (feature rows and outputs), and a
  // barrier again.  K1 is bound by instruction delivery (DESIGN.md §(d)):
  // with all warps in the same phase the SM streams one phase's code at a
  // time.  240K C5 candidates: 27.6 ms free-running, 25.1 ms in lockstep;
  // a barrier around every feature row as well (load imbalance) measured
  // 27.5 ms, and a separate resolve phase 25.1-25.3 ms.  Lockstep needs
  // even work per candidate: sibling slices (modes 1, 2) or pipelines with
  // many rows per candidate.  Random schedules of a small pipeline (C4:
  // eight rows, some of them 256-channel windows) run free (the same loop
  // without barriers): lockstep took C4's K1 from 88 to 122 ms.
  const bool lockstep = mode != 0 || L.R >= 16;   // 1M C5 K1 without: 101 ms
  // Reuse mode 2 (rows written only where computed): the run-head launch
  // resolves and prunes the heads but leaves their feature rows to the
  // sibling launch, where a head is the first candidate of its run with
  // every row dirty and its rows join the CTA's pool — the head launch's
  // tail (~2.4 heads per warp) shrinks to the resolve.  With reuse mode 1
  // a sibling copies its predecessor's feature block, so heads keep their
  // rows.
  const bool heads_later = reuse == 2 && feats != nullptr && mode != 0;
  {
    int64_t c = 0, c1 = 0, pc = 0, cur_run = -1, jcur = -1;
    bool done = false;
    // sibling slices: the CTA's warps take nw consecutive slices together
    // (mostly one run: the same decision structure and dirty rows, so the
    // warps run the same instruction stream), the next block once all are
    // done.  240K C5 candidates: 24.9 ms claiming per warp, 23.0 ms per CTA.
    __shared__ int64_t s_base;
    const bool cta_blocks = mode == 2 && lockstep;
    for (;;) {
      bool have = false;
      if (cta_blocks) {
        while (c < c1 && heads[c] && !heads_later) { cur_run = -1; ++c; }
        if (__syncthreads_and(c >= c1)) {
          if (threadIdx.x == 0) s_base = (int64_t)atomicAdd(work, (unsigned)nw);
          __syncthreads();
          const int64_t base = s_base;
          __syncthreads();
          if (base >= nchunks) break;
          const int64_t j = base + warp;
          c = c1 = 0;
          if (j < nchunks) {
            int64_t c0;
            if (j < nbig) { c0 = j * kChunk2; c1 = c0 + kChunk2; }
            else { c0 = nbig * kChunk2 + (j - nbig) * kFine; c1 = c0 + kFine < n ? c0 + kFine : n; }
            c = c0; pc = c0; cur_run = -1;
            if (lane == 0) { m.prev_valid = 0; m.same_struct = 0; m.ndec = 0; }
            __syncwarp();
            while (c < c1 && heads[c] && !heads_later) { cur_run = -1; ++c; }
          }
        }
        have = c < c1;
      }
      while (!done && !cta_blocks) {
        if (c >= c1) {
          if (mode == 1 && jcur >= 0) { slot_copy(jcur, true); jcur = -1; }
          unsigned uj = 0;
          if (lane == 0) uj = atomicAdd(work, 1u);
          const int64_t j = __shfl_sync(0xffffffffu, uj, 0);
          int64_t c0;
          if (mode == 0) {
            if (j >= nunits) { done = true; break; }
            c0 = snap(j * unit); c1 = snap((j + 1) * unit);
          } else if (mode == 1) {
            if (j >= nruns) { done = true; break; }
            c0 = run_head[j]; c1 = c0 + 1;
          } else {
            if (j >= nchunks) { done = true; break; }
            if (j < nbig) { c0 = j * kChunk2; c1 = c0 + kChunk2; }
            else { c0 = nbig * kChunk2 + (j - nbig) * kFine; c1 = c0 + kFine < n ? c0 + kFine : n; }
          }
          if (c0 >= c1) continue;
          c = c0; pc = c0; cur_run = -1; jcur = j;
          if (lane == 0) { m.prev_valid = 0; m.same_struct = 0; m.ndec = 0; }
          __syncwarp();
        }
        if (mode == 2 && heads[c] && !heads_later) { cur_run = -1; ++c; continue; }
        have = true;
        break;
      }
      if (cta_blocks) {
        if (!__syncthreads_or(have)) continue;   // a block of head-only slices: claim the next
      } else if (lockstep) {
        if (!__syncthreads_or(have)) break;
      } else if (!have) {
        break;
      }
      bool head_rows = false;   // mode 2: a run head whose state the slot holds
      if (have) {
        if (mode == 2) {
          const int64_t r = run_id[c];
          if (r != cur_run) { slot_copy(r, false); pc = run_head[r]; cur_run = r; }
          head_rows = heads_later && c == pc && heads[c];
        }
        if (!head_rows) phaseA(c, pc);
      }
      if (have && !head_rows) { phaseResolve(); phaseA2(c, pc); }
      if (head_rows) {
        // verdict and n_rows came from the head launch; every row is computed
        nr = m.nrows;
        nd = nr;
        diffable = false;
        for (int r = lane; r < nr; r += 32) { k.rowlist[r] = (int16_t)r; rsrc[r] = (int32_t)c; }
        __syncwarp();
        if (lane == 0) st_rows += nd;
      }
      if (have && mode == 1 && heads_later) {   // the head's rows: in the sibling launch
        if (lane == 0) st_rows -= nd;
        nd = 0;
      }
      // sibling slices pool their rows (1M C5 K1 58.3 -> 54.4 ms, C2 7.0 ->
      // 5.2 ms); run heads and whole candidates (modes 1 / 0: ~100 rows
      // each, even work) measured 1-10 % slower pooled
      const bool pool = lockstep && mode == 2;
      if (pool) {
        if (lane == 0) { s_nd[warp] = have ? nd : 0; s_cand[warp] = c; }
        if (threadIdx.x == 0) *s_next = 0;
      }
      if (lockstep) __syncthreads();
      if (have) phaseB(c, pc);
      if (pool && reuse == 1 && feats) __syncthreads();   // copied blocks land before pooled rows
      // the rows read the scorer state through a view rebuilt per row: its
      // pointers are rematerialised from the slice base instead of staying
      // live across the row code (60.1 vs 61.0 ms per 1M C5 K1).  Pooled:
      // the CTA's rows in row-major order (row q of every warp's candidate,
      // then row q + 1: siblings' row q run the same code), each taken by
      // the next free warp.
      if (pool) {
        const int myn = lane < nw ? s_nd[lane] : 0;
        for (;;) {
          int p = 0;
          if (lane == 0) p = atomicAdd(s_next, 1);
          p = __shfl_sync(0xffffffffu, p, 0);
          int q = 0, o = -1;
          for (;; ++q) {
            const unsigned has = __ballot_sync(0xffffffffu, myn > q);
            if (!has) break;
            const int cnt = __popc(has);
            if (p < cnt) { o = __fns(has, 0, p + 1); break; }
            p -= cnt;
          }
          if (o < 0) break;
          K1<ND> kr;
          bind(kr, o);
          phaseRow(kr, s_cand[o], q);
        }
      } else if (have) {
        for (int q = 0; q < nd; ++q) {
          K1<ND> kr;
          bind(kr, warp);
          phaseRow(kr, c, q);
        }
      }
      if (have) {
        if (mode == 1 && heads_later) {   // row keys / sources are written with the rows
          if (lane == 0) m.prev_valid = m.err == 0;
          __syncwarp();
        } else {
          phaseB3(c);
        }
        pc = c; ++c;
      }
      if (lockstep) __syncthreads();
    }
  }
#ifdef GS_PHASES
  if (lane == 0)
    for (int i = 0; i < 7; ++i) atomicAdd(&g_phase[i], (unsigned long long)ph[i]);
#endif
  if (lane == 0 && st_cand) {
    unsigned long long* ctr = reinterpret_cast<unsigned long long*>(gerr + 2);
    atomicAdd(ctr + 0, st_cand);
    atomicAdd(ctr + 1, st_inc); atomicAdd(ctr + 2, st_rows); atomicAdd(ctr + 3, st_emit); atomicAdd(ctr + 4, st_geo);
  }
}

// Decision-structure run heads for the K1 work units: candidate c starts a
// run when any record's (func, consumer, kind) differs from candidate c-1's
// (the K1 sibling test); one warp per candidate, coalesced record loads.
// `hflag` (optional) receives the same flag as a u32 for the run scan.
__global__ void k1_heads_kernel(const GsDecision* __restrict__ dec, int64_t n, int S, uint8_t* __restrict__ head,
                                uint32_t* __restrict__ hflag) {
  const int lane = threadIdx.x & 31;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= n) return;
  bool diff = c == 0;
  if (c > 0) {
    const uint2* a = reinterpret_cast<const uint2*>(dec + c * S);
    const uint2* b = reinterpret_cast<const uint2*>(dec + (c - 1) * S);
    for (int i = lane; i < S; i += 32) {
      const uint2 x = __ldg(a + 2 * i), y = __ldg(b + 2 * i);
      diff |= x.x != y.x || ((x.y ^ y.y) & 0xFFu) != 0u;
    }
    diff = __any_sync(0xffffffffu, diff);
  }
  if (lane == 0) {
    head[c] = diff;
    if (hflag) hflag[c] = diff ? 1u : 0u;
  }
}

// run_id = inclusive scan of the head flags - 1; run_head[r] = first
// candidate of run r
__global__ void k1_run_heads_kernel(const uint8_t* __restrict__ head, int32_t* __restrict__ run_id, int64_t n,
                                    int32_t* __restrict__ run_head) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  const int32_t r = run_id[c] - 1;
  run_id[c] = r;
  if (head[c]) run_head[r] = (int32_t)c;
}

}  // namespace gs

// ---------------------------------------------------------------------------
// host launch helpers (used by api.cu)
// ---------------------------------------------------------------------------
namespace gs {

template <int ND>
static int cf_size() { return (int)sizeof(CF<ND>); }

// Shared memory: [pipeline descriptor | warp 0 slice | warp 1 slice | ...];
// offsets inside a slice are relative to the slice.  Arrays placed with
// gplace live in the warp's global scratch instead (offsets relative to it).
Layout make_layout(int nd, int nf, int ns, int blob_bytes, int S, int R, int rcap, int pcap, int nwarps,
                   int spill, bool generic) {
  auto al = [](int x) { return (x + 15) & ~15; };
  Layout L{};
  L.blob = 0;
  L.cta = al(blob_bytes);            // CTA header: pooled-row bookkeeping
  L.warps = L.cta + kCtaHeaderBytes;
  int o = 0;
  int g = 0;   // global scratch bytes per warp (spill)
  // capacity-sized arrays: in the smem slice, or in global scratch
  auto place_at = [&](int level, int bytes) {
    int r;
    if (spill >= level) { r = g; g += al(bytes); } else { r = o; o += al(bytes); }
    return r;
  };
  auto place = [&](int bytes) { return place_at(1, bytes); };
  auto gplace = [&](int bytes) { int r = g; g += al(bytes); return r; };   // always global
  L.didx = o; o += al(nf * 2);
  int cfs = nd == 1 ? cf_size<1>() : nd == 2 ? cf_size<2>() : nd == 3 ? cf_size<3>() : cf_size<4>();
  L.cf = o; o += al(nf * cfs);
  L.pcf = 0;
  L.reads = place_at(2, rcap * (int)sizeof(RRead));
  L.paths = place_at(2, pcap * 2);
  L.rdb = o; o += al(2 * ns * 4);
  L.rows = o; o += al(R * 4);
  L.icall = gplace(pcap * (int)sizeof(ICall));
  L.srcb = o; o += al((nf + 1) * 4);
  L.srcl = place(rcap * 2);
  L.rdepb = o; o += al((R + 1) * 4);
  L.rdep = place_at(2, (rcap + nf) * 2);
  L.dirty = o; o += al(nf);
  L.rflag = o; o += al(R);
  L.rowlist = o; o += al(R * 2);
  L.rsrc = o; o += al(R * 4);
  L.mw = nf <= 32 * kMaxMaskWords ? (nf + 31) / 32 : 0;
  L.kern = o; o += al(nf * 2);
  L.dm = gplace(nf * L.mw * 4);
  L.cmask = o; o += al(kMaxMaskWords * 4);
  L.kmb = place((nf + 1) * 4);
  L.kml = place(nf * 2);
  L.icb = place((nf + 1) * 4);
  L.icl = gplace(pcap * 2);
  L.dlist = place(nf * 2);
  L.gdirty = o; o += al(nf);
  L.kdirty = o; o += al(nf);
  L.misc = o; o += al((int)sizeof(Misc));
  // row scratch; the structure-build scratch (DFS stack, volume
  // accumulators, touched list: used once per decision structure) lives in
  // the warp's global scratch, as do the dependency masks, so that the
  // default machine's slice fits ten scorer warps per SM
  // Everything from here on is per-candidate scratch (the candidate's own
  // records, row scratch, structure-build scratch): a run slot keeps only
  // the prefixes [0, keep) and [0, gkeep) of the slice and global scratch.
  L.keep = o;
  L.gkeep = g;
  L.dec = o; o += al(S * 16);
  L.scr = o;
  L.stack = gplace((nf + 2) * (int)sizeof(Frame));
  L.volacc = gplace(nf * 8);
  L.touched = gplace(2 * nf * 2 + 4);
  const int scr_bytes = generic ? (int)sizeof(WarpScr) : kScrDefaultBytes;
  o += al(scr_bytes);
  L.warp_bytes = al(o);
  L.gl_bytes = g;
  L.spill = spill;
  L.total = L.warps + nwarps * L.warp_bytes;
  L.rcap = rcap; L.pcap = pcap; L.S = S; L.R = R;
  return L;
}

// warps per CTA that fit the shared memory budget (one CTA per SM)
int read_phases(long long* out) {
  unsigned long long h[16];
  if (cudaMemcpyFromSymbol(h, g_phase, sizeof(h)) != cudaSuccess) return -1;
  for (int i = 0; i < 16; ++i) out[i] = (long long)h[i];
  unsigned long long z[16] = {};
  cudaMemcpyToSymbol(g_phase, z, sizeof(z));
  return 0;
}

int featurize_warps(const Layout& L1, int max_smem) {
  int w = (max_smem - L1.warps) / L1.warp_bytes;
  return w < 1 ? 0 : (w > kK1MaxWarps ? kK1MaxWarps : w);
}

// Run heads of a batch (K1 sibling structure) and, for the two-phase
// schedule, each candidate's run index, each run's head and the run count
// (`nruns`, left on the device: no host synchronization).
void k1_prepare_runs(const GsDecision* dec, int64_t n, int S, uint8_t* heads, int32_t* run_id, int32_t* run_head,
                     uint32_t* sums, uint32_t* nruns, cudaStream_t st) {
  uint32_t* flag = reinterpret_cast<uint32_t*>(run_id);
  k1_heads_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(dec, n, S, heads, flag);
  scan_u32(flag, flag, n, nullptr, true, sums, nruns, st);
  k1_run_heads_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(heads, run_id, n, run_head);
  g_launch_count += 2;
}

size_t k1_runs_sums_bytes(int64_t n) { return align256(4 * (scan_tiles_of(n) + 1)); }

int launch_featurize(int nd, const PipeDev* P, const uint8_t* blob, const GsDecision* dec, int64_t n, int S,
                     double* feats, int32_t* row_key, int32_t* n_rows, uint8_t* verdict, int32_t* row_src,
                     const Layout& L, int nwarps, int grid, int* gerr, int reuse, uint8_t* gscratch,
                     uint8_t* heads, int mode, const int32_t* run_id, const int32_t* run_head,
                     const uint32_t* nruns, int64_t max_runs, uint8_t* slots, int64_t slot_bytes,
                     int32_t* row_kernel, cudaStream_t st) {
  dim3 b(nwarps * 32);
  if (heads && reuse && mode == 0) {
    k1_heads_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(dec, n, S, heads, nullptr);
    g_launch_count++;
  }
  cudaMemsetAsync(gerr + 14, 0, sizeof(unsigned), st);   // work-unit counter
  switch (nd) {
#define GS_CASE(D)                                                                                  \
  case D:                                                                                           \
    cudaFuncSetAttribute(featurize_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, L.total); \
    featurize_kernel<D><<<grid, b, L.total, st>>>(P, blob, dec, n, S, feats, row_key, n_rows, verdict, row_src, L, gerr, reuse, gscratch, reuse ? heads : nullptr, mode, run_id, run_head, nruns, max_runs, slots, slot_bytes, row_kernel); \
    g_launch_count++;                                                                               \
    break;
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4)
#undef GS_CASE
    default: return -1;
  }
  return 0;
}


}  // namespace gs
