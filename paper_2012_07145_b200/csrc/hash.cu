// K3 — structural hash = blake2b-64 over the bytes of Python repr() of the
// canonical decision tuple (reference loopnest.py:131-165).  One thread per
// candidate streams the repr bytes straight into the blake2b compressor:
// func names come from a pre-rendered repr table (host), walked in Python
// str order (name_rank), so no string sorting happens on the device.
#include "gs_internal.cuh"

namespace gs {

constexpr int kHashMaxFuncs = 1024;

__constant__ uint64_t kIV[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                                0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                                0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};

__device__ __forceinline__ uint64_t rotr(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

// blake2b-64, unkeyed.  The current 128-byte block is staged in this
// thread's shared-memory slot (byte appends are plain st.shared.u8); the
// 12 rounds are fully unrolled with compile-time message schedules, so the
// message words and the state stay in registers.
template <int R>
__device__ __forceinline__ void blake_round(uint64_t* v, const uint64_t* m) {
  constexpr uint8_t S[12][16] = {
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
      {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
      {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
      {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
      {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
      {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};
#define G(a, b, c, d, x, y)                     \
  v[a] = v[a] + v[b] + m[S[R][x]];              \
  v[d] = rotr(v[d] ^ v[a], 32);                 \
  v[c] = v[c] + v[d];                           \
  v[b] = rotr(v[b] ^ v[c], 24);                 \
  v[a] = v[a] + v[b] + m[S[R][y]];              \
  v[d] = rotr(v[d] ^ v[a], 16);                 \
  v[c] = v[c] + v[d];                           \
  v[b] = rotr(v[b] ^ v[c], 63);
  G(0, 4, 8, 12, 0, 1) G(1, 5, 9, 13, 2, 3) G(2, 6, 10, 14, 4, 5) G(3, 7, 11, 15, 6, 7)
  G(0, 5, 10, 15, 8, 9) G(1, 6, 11, 12, 10, 11) G(2, 7, 8, 13, 12, 13) G(3, 4, 9, 14, 14, 15)
#undef G
}

struct Blake {
  uint64_t h[8];
  uint8_t* blk;     // this thread's 128-byte block in shared memory
  uint64_t t;       // bytes compressed so far
  int fill;         // bytes in the current block

  __device__ void init(uint8_t* block) {
    blk = block;
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] = kIV[i];
    h[0] ^= 0x01010000ULL ^ 8ULL;   // digest 8 bytes, no key
    t = 0; fill = 0;
  }
  __device__ void compress(bool last) {
    uint64_t m[16], v[16];
    for (int i = fill; i < 128; ++i) blk[i] = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      uint64_t w = 0;
#pragma unroll
      for (int b = 0; b < 8; ++b) w |= (uint64_t)blk[8 * i + b] << (8 * b);
      m[i] = w;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) { v[i] = h[i]; v[i + 8] = kIV[i]; }
    v[12] ^= t;
    if (last) v[14] = ~v[14];
    blake_round<0>(v, m); blake_round<1>(v, m); blake_round<2>(v, m); blake_round<3>(v, m);
    blake_round<4>(v, m); blake_round<5>(v, m); blake_round<6>(v, m); blake_round<7>(v, m);
    blake_round<8>(v, m); blake_round<9>(v, m); blake_round<10>(v, m); blake_round<11>(v, m);
#pragma unroll
    for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
  }
  __device__ __forceinline__ void byte(uint8_t b) {
    if (fill == 128) {
      t += 128;
      compress(false);
      fill = 0;
    }
    blk[fill++] = b;
  }
  __device__ void str(const char* s) { while (*s) byte((uint8_t)*s++); }
  __device__ void bytes(const uint8_t* p, int n) { for (int i = 0; i < n; ++i) byte(p[i]); }
  __device__ uint64_t final() {
    t += fill;
    compress(true);
    return h[0];
  }
};

__device__ const char* kind_repr(int k) {
  switch (k) {
    case GS_ROOT: return "'compute_root'";
    case GS_FUSE_BLOCK: return "'fuse_at_block'";
    case GS_FUSE_THREAD: return "'fuse_at_thread'";
    default: return "'inline'";
  }
}

// Does candidate c hash like candidate c-1?  The canonical tuple reads only
// (func, kind, consumer, serial is not None, thread is not None) of every
// decision (loopnest.py:151-165), so equal fields => equal bytes => equal
// hash at every depth.  Beam-step siblings differ only in tilings.
// run heads, one warp per candidate: coalesced 8-byte loads of the two
// logs, one ballot per 32 records
__global__ void hash_head_kernel(const GsDecision* __restrict__ dec, int64_t n, int S,
                                 uint8_t* __restrict__ head) {
  const int lane = threadIdx.x & 31;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= n) return;
  if (c == 0) { if (lane == 0) head[0] = 1; return; }
  const uint2* a = reinterpret_cast<const uint2*>(dec + c * S);
  const uint2* b = reinterpret_cast<const uint2*>(dec + (c - 1) * S);
  bool diff = false;
  for (int i = lane; i < S; i += 32) {
    const uint2 x = __ldg(a + 2 * i), y = __ldg(b + 2 * i);   // first 8 bytes of record i
    diff |= x.x != y.x || ((x.y ^ y.y) & 0x0003FFu) != 0u;
  }
  diff = __any_sync(0xffffffffu, diff);
  if (lane == 0) head[c] = diff;
}

__global__ void hash_kernel(const GsDecision* __restrict__ dec, int64_t n, int S, int nf, int depth,
                            const int32_t* __restrict__ sorted_funcs, const uint8_t* __restrict__ names,
                            const int32_t* __restrict__ name_off, uint64_t* __restrict__ out,
                            const uint8_t* __restrict__ head) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n) return;
  if (head && !head[c]) return;
  __shared__ uint8_t blocks[128 * 128];
  const GsDecision* d = dec + c * S;
  int16_t didx[kHashMaxFuncs];
  for (int f = 0; f < nf; ++f) didx[f] = -1;
  int nd = 0;
  for (int i = 0; i < S && d[i].func != 0xFFFF; ++i) { didx[d[i].func] = (int16_t)i; ++nd; }
  Blake b;
  b.init(blocks + 128 * threadIdx.x);
  auto name = [&](int f) { b.bytes(names + name_off[f], name_off[f + 1] - name_off[f]); };
  if (depth == 0) {
    b.str("('kernels', (");
    int cnt = 0;
    for (int q = 0; q < nf; ++q) {
      int f = sorted_funcs[q];
      int i = didx[f];
      if (i < 0 || d[i].kind != GS_ROOT) continue;
      if (cnt) b.str(", ");
      name(f);
      ++cnt;
    }
    if (cnt == 1) b.byte(',');
    b.str("))");
  } else {
    b.byte('(');
    b.byte((uint8_t)('0' + depth));
    b.str(", (");
    int cnt = 0;
    for (int q = 0; q < nf; ++q) {
      int f = sorted_funcs[q];
      int i = didx[f];
      if (i < 0) continue;
      if (cnt) b.str(", ");
      b.byte('(');
      name(f);
      b.str(", ");
      b.str(kind_repr(d[i].kind));
      b.str(", ");
      // kernel_of (loopnest.py:87-94)
      int kf = f, ki = i, guard = 0;
      while (ki >= 0 && (d[ki].kind == GS_FUSE_BLOCK || d[ki].kind == GS_FUSE_THREAD) && guard++ < nf) {
        kf = d[ki].consumer;
        ki = kf < nf ? didx[kf] : -1;
      }
      if (ki < 0 || d[ki].kind == GS_INLINE) b.str("None");
      else name(kf);
      if (depth >= 2) {
        b.str(", ");
        if (d[i].consumer == 0xFFFF) b.str("None");
        else name(d[i].consumer);
      }
      if (depth >= 3) {
        b.str((d[i].flags & 1) ? ", True" : ", False");
        b.str((d[i].flags & 2) ? ", True" : ", False");
      }
      b.byte(')');
      ++cnt;
    }
    if (cnt == 1) b.byte(',');
    b.str("))");
  }
  out[c] = b.final();
}

// ---------------------------------------------------------------------------
// Warp-per-candidate variant: the 32 lanes render the canonical repr in
// parallel (one decision entry per lane, offsets by a warp scan of entry
// lengths) into this warp's shared-memory buffer, then the warp runs the
// blake2b compressions over it (four lanes per state, blake_buf4).  Used whenever the longest possible repr
// fits the buffer (kHashBuf); the thread-per-candidate kernel above covers
// the rest.
constexpr int kHashBuf = 8192;
constexpr int kHashWarps = 4;   // warps per block

__device__ __forceinline__ int cstr_len(const char* s) { int n = 0; while (s[n]) ++n; return n; }
__device__ __forceinline__ int put(uint8_t* buf, int o, const char* s) { while (*s) buf[o++] = (uint8_t)*s++; return o; }

// blake2b-64 of buf[0, len) by the whole warp: lane group of four (lane &
// 3 = q) holds state column q (v[q], v[4+q], v[8+q], v[12+q]); a round is
// G on the four columns, a rotation of the b / c / d rows across the group
// (shuffles), G on the four diagonals, and the inverse rotation.  The
// serial chain is a quarter of the one-lane compressor's; the eight groups
// compute the same value.  sig: lane q's message indices, 4 bits each:
// round r's (2q, 2q+1, 8+2q, 9+2q) schedule entries at bits 16r..16r+15
// (three 64-bit words, four rounds each).
__device__ __forceinline__ void gmix(uint64_t& a, uint64_t& b, uint64_t& c, uint64_t& d, uint64_t x, uint64_t y) {
  a = a + b + x; d = rotr(d ^ a, 32); c = c + d; b = rotr(b ^ c, 24);
  a = a + b + y; d = rotr(d ^ a, 16); c = c + d; b = rotr(b ^ c, 63);
}

__device__ __forceinline__ uint64_t blake_buf4(const uint8_t* buf, int len, const uint64_t (&sig)[3]) {
  const int q = threadIdx.x & 3;
  uint64_t ha = kIV[q], hb = kIV[4 + q];
  if (q == 0) ha ^= 0x01010000ULL ^ 8ULL;
  const int nblk = len == 0 ? 1 : (len + 127) / 128;
  for (int b = 0; b < nblk; ++b) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(buf + 128 * b);
    const bool last = b == nblk - 1;
    uint64_t va = ha, vb = hb, vc = kIV[q], vd = kIV[4 + q];
    if (q == 0) vd ^= (uint64_t)(last ? len : 128 * (b + 1));
    if (q == 2 && last) vd = ~vd;
#pragma unroll
    for (int r = 0; r < 12; ++r) {
      const unsigned e = (unsigned)(sig[r >> 2] >> (16 * (r & 3))) & 0xFFFFu;
      gmix(va, vb, vc, vd, w[e & 15], w[(e >> 4) & 15]);
      vb = __shfl_sync(0xffffffffu, vb, (q + 1) & 3, 4);
      vc = __shfl_sync(0xffffffffu, vc, (q + 2) & 3, 4);
      vd = __shfl_sync(0xffffffffu, vd, (q + 3) & 3, 4);
      gmix(va, vb, vc, vd, w[(e >> 8) & 15], w[(e >> 12) & 15]);
      vb = __shfl_sync(0xffffffffu, vb, (q + 3) & 3, 4);
      vc = __shfl_sync(0xffffffffu, vc, (q + 2) & 3, 4);
      vd = __shfl_sync(0xffffffffu, vd, (q + 1) & 3, 4);
    }
    ha ^= va ^ vc;
    hb ^= vb ^ vd;
  }
  return __shfl_sync(0xffffffffu, ha, 0);
}

__constant__ uint8_t kSigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__device__ __forceinline__ void sigma_of_lane(uint64_t (&sig)[3]) {
  const int q = threadIdx.x & 3;
  sig[0] = sig[1] = sig[2] = 0;
  for (int r = 0; r < 12; ++r) {
    const uint64_t e = (uint64_t)kSigma[r][2 * q] | (uint64_t)kSigma[r][2 * q + 1] << 4 |
                       (uint64_t)kSigma[r][8 + 2 * q] << 8 | (uint64_t)kSigma[r][9 + 2 * q] << 12;
    sig[r >> 2] |= e << (16 * (r & 3));
  }
}

__global__ void __launch_bounds__(kHashWarps * 32) hash_warp_kernel(
    const GsDecision* __restrict__ dec, int64_t n, int S, int nf, HashDepths D, const int32_t* __restrict__ sorted_funcs,
    const uint8_t* __restrict__ names, const int32_t* __restrict__ name_off, uint64_t* __restrict__ out,
    const uint8_t* __restrict__ head) {
  extern __shared__ __align__(16) uint8_t smh[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint8_t* buf = smh + wib * (kHashBuf + 2 * kHashMaxFuncs);
  uint64_t sig[3];
  sigma_of_lane(sig);
  int16_t* didx = reinterpret_cast<int16_t*>(buf + kHashBuf);
  // contiguous candidate ranges per warp: run heads are periodic in a beam
  // step (one per parent), and a grid stride sharing a factor with that
  // period would hand all of them to a few warps
  const int64_t nwarps = (int64_t)gridDim.x * kHashWarps;
  const int64_t wid = (int64_t)blockIdx.x * kHashWarps + wib;
  const int64_t per = (n + nwarps - 1) / nwarps;
  const int64_t c_end = (wid + 1) * per < n ? (wid + 1) * per : n;
  for (int64_t c = wid * per; c < c_end; ++c) {
    if (head) {   // next run head at or after c, 32 flags per probe
      int64_t nxt = c_end;
      for (int64_t b = c; b < c_end; b += 32) {
        const unsigned m = __ballot_sync(0xffffffffu, b + lane < c_end && head[b + lane]);
        if (m) { nxt = b + __ffs(m) - 1; break; }
      }
      c = nxt;
      if (c >= c_end) break;
    }
    const GsDecision* d = dec + c * S;
    for (int f = lane; f < nf; f += 32) didx[f] = -1;
    __syncwarp();
    for (int i = lane; i < S; i += 32) {
      const int f = d[i].func;
      if (f != 0xFFFF && f < nf) didx[f] = (int16_t)i;
    }
    __syncwarp();
    // every requested depth from the same records (out: [D.n][n]); a run
    // at the deepest key is a run at every shallower one
#pragma unroll 1
    for (int dk = 0; dk < D.n; ++dk) {
    const int depth = D.d[dk];
    uint64_t* outk = out + (int64_t)dk * n;
    int pos;
    if (depth == 0) {
      if (lane == 0) put(buf, 0, "('kernels', (");
      pos = 13;
    } else {
      if (lane == 0) { buf[0] = '('; buf[1] = (uint8_t)('0' + depth); put(buf, 2, ", ("); }
      pos = 5;
    }
    int cnt = 0;
    for (int q0 = 0; q0 < nf; q0 += 32) {
      const int q = q0 + lane;
      const int f = q < nf ? sorted_funcs[q] : -1;
      const int i = f >= 0 ? didx[f] : -1;
      const bool incl = i >= 0 && (depth > 0 || d[i].kind == GS_ROOT);
      const unsigned bal = __ballot_sync(0xffffffffu, incl);
      const int before = cnt + __popc(bal & ((1u << lane) - 1));
      int len = 0, kf = -1;
      if (incl) {
        const int nl = name_off[f + 1] - name_off[f];
        len = (before ? 2 : 0) + nl;
        if (depth > 0) {
          // kernel_of (loopnest.py:87-94)
          int ki = i, guard = 0;
          kf = f;
          while (ki >= 0 && (d[ki].kind == GS_FUSE_BLOCK || d[ki].kind == GS_FUSE_THREAD) && guard++ < nf) {
            kf = d[ki].consumer;
            ki = kf < nf ? didx[kf] : -1;
          }
          if (ki < 0 || d[ki].kind == GS_INLINE) kf = -1;
          len += 1 + 2 + cstr_len(kind_repr(d[i].kind)) + 2 +
                 (kf >= 0 ? name_off[kf + 1] - name_off[kf] : 4) + 1;
          if (depth >= 2) {
            const int cf = d[i].consumer;
            len += 2 + (cf == 0xFFFF ? 4 : name_off[cf + 1] - name_off[cf]);
          }
          if (depth >= 3) len += ((d[i].flags & 1) ? 6 : 7) + ((d[i].flags & 2) ? 6 : 7);
        }
      }
      int ex = len;   // exclusive scan of entry lengths
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(0xffffffffu, ex, o);
        if (lane >= o) ex += u;
      }
      const int tot = __shfl_sync(0xffffffffu, ex, 31);
      ex -= len;
      if (incl && pos + ex + len <= kHashBuf) {
        int o = pos + ex;
        if (before) { buf[o++] = ','; buf[o++] = ' '; }
        if (depth > 0) buf[o++] = '(';
        for (int k = name_off[f]; k < name_off[f + 1]; ++k) buf[o++] = names[k];
        if (depth > 0) {
          o = put(buf, o, ", ");
          o = put(buf, o, kind_repr(d[i].kind));
          o = put(buf, o, ", ");
          if (kf >= 0) { for (int k = name_off[kf]; k < name_off[kf + 1]; ++k) buf[o++] = names[k]; }
          else o = put(buf, o, "None");
          if (depth >= 2) {
            o = put(buf, o, ", ");
            const int cf = d[i].consumer;
            if (cf == 0xFFFF) o = put(buf, o, "None");
            else for (int k = name_off[cf]; k < name_off[cf + 1]; ++k) buf[o++] = names[k];
          }
          if (depth >= 3) {
            o = put(buf, o, (d[i].flags & 1) ? ", True" : ", False");
            o = put(buf, o, (d[i].flags & 2) ? ", True" : ", False");
          }
          buf[o++] = ')';
        }
      }
      pos += tot;
      cnt += __popc(bal);
    }
    // trailer, zero padding of the last block, compression
    int len = pos + (cnt == 1 ? 1 : 0) + 2;
    if (lane == 0 && len <= kHashBuf) {
      int o = pos;
      if (cnt == 1) buf[o++] = ',';
      buf[o++] = ')';
      buf[o++] = ')';
    }
    const int padded = ((len + 127) / 128) * 128;
    for (int k = len + lane; k < padded && k < kHashBuf; k += 32) buf[k] = 0;
    __syncwarp();
    const unsigned long long hv = len <= kHashBuf ? blake_buf4(buf, len, sig) : 0ull;
    if (lane == 0) outk[c] = hv;
    if (head) {   // the run's followers (up to the next head, past this warp's range) copy it
      for (int64_t b = c + 1; b < n; b += 32) {
        const bool follower = b + lane < n && !head[b + lane];
        const unsigned m = __ballot_sync(0xffffffffu, !follower);   // first head / end of batch
        const int stop = m ? __ffs(m) - 1 : 32;
        if (lane < stop) outk[b + lane] = hv;
        if (m) break;
      }
    }
    __syncwarp();
    }
  }
}

// non-head candidates copy the hash of the head of their run (after the
// per-thread hash_kernel; hash_warp_kernel fills followers itself)
__global__ void hash_fill_kernel(const uint8_t* __restrict__ head, int64_t n, uint64_t* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= n || head[c]) return;
  int64_t j = c - 1;
  while (!head[j]) --j;
  out[c] = out[j];
}

int launch_hash(const GsDecision* dec, int64_t n, int S, int nf, HashDepths D, const int32_t* sorted_funcs,
                const uint8_t* names, const int32_t* name_off, uint64_t* out, uint8_t* head, int repr_bound,
                int num_sms, cudaStream_t st) {
  if (n == 0) return 0;
  if (nf > kHashMaxFuncs) return -1;
  if (D.n < 1 || D.n > 4) return -1;
  for (int k = 0; k < D.n; ++k) D.d[k] = D.d[k] > 3 ? 3 : D.d[k];
  int64_t blocks = (n + 127) / 128;
  if (head) {
    hash_head_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, st>>>(dec, n, S, head);
    g_launch_count++;
  }
  if (repr_bound <= kHashBuf) {
    const int smem = kHashWarps * (kHashBuf + 2 * kHashMaxFuncs);
    cudaFuncSetAttribute(hash_warp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int64_t want = (n + kHashWarps - 1) / kHashWarps;
    const int grid = (int)(want < (int64_t)num_sms * 8 ? want : (int64_t)num_sms * 8);
    hash_warp_kernel<<<grid, kHashWarps * 32, smem, st>>>(dec, n, S, nf, D, sorted_funcs, names, name_off, out,
                                                           head);
    g_launch_count++;
    return 0;
  }
  for (int k = 0; k < D.n; ++k) {   // per-thread kernel (representations beyond the warp buffer)
    uint64_t* outk = out + (int64_t)k * n;
    hash_kernel<<<(unsigned)blocks, 128, 0, st>>>(dec, n, S, nf, D.d[k], sorted_funcs, names, name_off, outk, head);
    g_launch_count++;
    if (head) {
      hash_fill_kernel<<<(unsigned)blocks, 128, 0, st>>>(head, n, outk);
      g_launch_count++;
    }
  }
  return 0;
}

}  // namespace gs
