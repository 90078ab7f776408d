// Internal device-side definitions shared by the gs_sched kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <atomic>
#include "../../include/gs_sched.h"

namespace gs {

// Count of this library's own kernel launches (host side), for the bench.
inline std::atomic<long long> g_launch_count{0};

constexpr int kWarp = 32;
constexpr int kMaxM = 128;          // largest residue modulus (transaction / bank period)
constexpr int kRowReads = 64;       // reads attributed to one row
constexpr int kGroupReads = 16;     // reads in one (tier, producer) group
constexpr int kLaneIv = 96;         // per-lane interval capacity for unions
constexpr int kK1MaxWarps = 12;      // K1 warps per CTA (one CTA per SM)
constexpr int kCtaHeaderBytes = 256;  // K1 CTA header in dynamic shared memory (pooled-row bookkeeping)
constexpr int kUnit = 64;           // K1 work-unit size (candidates, before run-head snapping)
#ifndef GS_CHUNK2
#define GS_CHUNK2 5
#endif
constexpr int kChunk2 = GS_CHUNK2;  // K1 two-phase schedule: sibling slice size (1M C5 K1, one 12-warp CTA per SM: 3 -> 63.4 ms, 4 -> 61.9, 5 -> 58.5, 6 -> 64.8, 8 -> 66.4)
constexpr int64_t kAddrBias = int64_t(1) << 40;  // featurize.py:256

enum Tier : int8_t { T_GLOBAL = 0, T_SHARED = 1, T_REGISTER = 2, T_NONE = 3 };
enum Kind : int8_t { K_ROOT = 0, K_BLOCK = 1, K_THREAD = 2, K_INLINE = 3, K_EXTERNAL = 4,
                     K_ABSENT = -1 };

// Error word bits (device -> host).
enum : int { E_READS = 1, E_PATHS = 2, E_ROWREADS = 4, E_GROUP = 8, E_LANEIV = 16,
             E_SCHEDULE = 32, E_STACK = 64 };

struct PipeDev {              // device copy of the pipeline (global memory)
  int nf, ns, na;
  int blob_bytes;             // funcs | stages | access, 16-byte aligned sections
  int off_stages, off_access; // byte offsets inside the blob
  int max_rows;
  int nd;                     // max ndim over funcs
  GsMachine m;
  GsThresholds th;
};

// Per-func resolved geometry (reference resolve.py:82-129 ConcreteFunc,
// 132-142 KernelInfo folded into the kernel owner's record).
template <int ND>
struct alignas(16) CF {
  int8_t kind, tier, unrolled, has_serial;
  int16_t kernel;     // kernel owner func id, -1 = none
  int16_t consumer;   // fused: d.consumer; inline: primary consumer
  int32_t n_threads;
  int32_t rlo[ND], rhi[ND];       // padded realization region
  int32_t tlo[ND], thi[ND];       // union of realizations over the run
  int32_t ctx[ND], base[ND], coeff[ND], ext[ND];
  int32_t serial_prod;
  int32_t k_threads;              // kernel owner only: max threads per block
  int32_t spare[(ND & 1) ? 2 : 1];  // explicit: no padding bytes (records are memcmp'd)
  int64_t realizations;
  union { int64_t n_blocks; int64_t calls; };   // kernel owner: blocks; inline: total calls
  union { int64_t k_shared; int64_t best; };    // kernel owner: shared bytes; inline: best per-consumer calls
};

struct RRead {                // one expanded read (resolve.py:56-79 ResolvedRead)
  int16_t owner, producer;
  int16_t root;               // non-inline func whose stage expansion produced it
  int8_t tier;
  uint8_t plen;               // links in the chain
  uint16_t pbeg;              // first access id in the path pool
  uint16_t pad;
};

struct Layout {                 // byte offsets inside dynamic shared memory (K1)
  int blob, dec, didx, cf, pcf, reads, paths, rdb, rows, stack, volacc, touched, icall, srcb,
      srcl, rdepb, rdep, dirty, rflag, rowlist, rsrc, kern, dm, cmask, kmb, kml, icb, icl, dlist, gdirty,
      kdirty, misc, warps, scr, cta;
  int mw;                       // dependency-mask words per func (0 = incremental resolve off)
  int gl_bytes;                 // per-warp global scratch bytes (inline-call lists, spilled arrays)
  int spill;                    // capacity-sized structure arrays in global scratch: 0 none, 1 resolve-side, 2 all
  int warp_bytes, total;
  int keep, gkeep;              // slice / global-scratch prefixes a run slot saves (the rest is per-candidate)
  int rcap, pcap, S, R;
};

// Phase-1 menus (options.py:103-141): static per-func facts, packed by the
// host from the pipeline (gs_set_placement_info) — the same definitions the
// reference evaluates per call.
enum : uint8_t { P1_OUTPUT = 1, P1_SINGLE_STAGE = 2, P1_POINTWISE_CALLED = 4, P1_INLINE_OK = 8, P1_CHEAP = 16 };
struct P1Static {
  const uint8_t* flags;      // [nf]
  const int32_t* cons_off;   // [nf + 1] consumers_of CSR (self-reads excluded)
  const int16_t* cons;
  const int32_t* sorted;     // funcs in Python str (name) order
};

struct HashDepths {             // K3: the depths one pass hashes (out: [n][...] per depth, depth-major)
  int n;
  int d[4];
};

struct NetDev {                 // device copies of the coefficient network (K2)
  int E, H;                     // embed / hidden dims
  const double *algo_w, *algo_b, *sched_w, *sched_b, *head_w, *head_b, *out_w, *out_b;
  double* hoisted;              // [n_stages][H] = relu(xa Wa + ba) Wh[:E] + bh
};

__host__ __device__ inline int64_t floordiv(int64_t a, int64_t b) {
  int64_t q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
__host__ __device__ inline int64_t posmod(int64_t a, int64_t m) {
  int64_t r = a % m;
  return r < 0 ? r + m : r;
}

}  // namespace gs
