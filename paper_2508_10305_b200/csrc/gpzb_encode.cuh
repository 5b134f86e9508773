// K1 (range) and K1.5 (geometry) of the GPZ B200 compressor, plus the
// shared helpers of the encoders.
//
// Compress pipeline (all stream-ordered; the host reads the 128-byte result
// record once, after K3a, to size the exact container):
//   K1   k_range_w       per-block bounds, joint range (REL), finiteness
//   K1.5 k_geometry      per-block geometry record; routes each block to an
//                        encoder (K2s / K2p / K2 / K2w lists, counts on the device)
//   K2*  encoders        each block's payload into its staging slot, its
//                        length into sizes[blk]
//   K3a  k_scan_sizes    decoupled look-back scan of the lengths (gpzb_compact.cuh)
//   K3b  k_copy_payloads table, global header, payloads to their final offsets
#pragma once

#include <type_traits>

#include "gpzb_common.cuh"

namespace gpzb {

struct BlkRec;

struct EncParams {
  const void* axes[3];
  uint64_t count;          // particles in this call (shard)
  uint64_t nblocks;        // blocks in this call
  uint32_t bs;
  uint32_t target;
  double eb;               // configured bound
  int rel;                 // eb_mode == RANGE_RELATIVE
  int vec;                 // all axis pointers 16B aligned
  DevResult* res;
  const void* bounds;      // K1 per-block [min,max] x dims in input precision
  unsigned long long* status;  // payload length per block (K2) -> exclusive offset (K3)
  unsigned long long* tstat;   // K3 scan tile look-back words
  uint8_t* payload;        // where block 0's payload starts
  uint8_t* table;          // where block 0's inclusive table entry goes (entry 1)
  uint8_t* table0;         // entry 0 (written by block 0) or null
  uint8_t* header;         // global header (written by block 0) or null
  uint64_t table_base;     // added to every table entry
  uint64_t header_count, header_blocks;
  int eb_mode_code;
  int preserve;
  BlkRec* rec;             // per-block geometry records (K1.5)
  uint32_t* wide_list;     // blocks routed to the general encoder
  uint32_t* cta_list;      // narrow blocks for the general CTA encoder K2 (K1.5, then K2s hand-backs)
  uint32_t* small_list;    // K2s blocks: with offsets from the front, offset-free from the back
  uint32_t* warp_list;     // K2p blocks (K1.5; length res->warp_count)
  uint8_t* big;            // K2b: per-CTA workspace slices (block_size > 1024)
  int small0;              // route offset-free full f32 blocks to K2s (1) or to the warp encoder K2p (0)
  int use_small;           // route blocks to K2s at all (diagnostics switch)
  uint8_t* side;           // staging for the general encoder's payloads
  uint64_t side_cap;       // its capacity in bytes (K2w reports a shortfall instead of writing past it)
  uint8_t* staging;        // narrow payloads: one kSlotBytes slot per block (K3 concatenates)
};

// ----------------------------------------------------------------- loads
template <int D, typename T>
__device__ __forceinline__ void load_particles(const EncParams& P, uint64_t first, int n, int p0,
                                               T (&x)[D][kItems]) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const T* base = reinterpret_cast<const T*>(P.axes[a]) + first + p0;
    if (P.vec && p0 + kItems <= n) {
      if constexpr (sizeof(T) == 4) {
        float4 v = __ldcs(reinterpret_cast<const float4*>(base));
        x[a][0] = v.x; x[a][1] = v.y; x[a][2] = v.z; x[a][3] = v.w;
      } else {
        double2 v0 = __ldcs(reinterpret_cast<const double2*>(base));
        double2 v1 = __ldcs(reinterpret_cast<const double2*>(base) + 1);
        x[a][0] = v0.x; x[a][1] = v0.y; x[a][2] = v1.x; x[a][3] = v1.y;
      }
    } else {
#pragma unroll
      for (int k = 0; k < kItems; ++k) x[a][k] = (p0 + k < n) ? __ldcs(base + k) : T(0);
    }
  }
}

// ------------------------------------------------------------------- K1
// K1, warp per block: each warp streams whole blocks (16-byte loads, eight
// per lane and axis in flight, no CTA barriers) and reduces them with warp
// primitives; one atomic per CTA for the joint range.
template <int D, typename T>
__global__ void __launch_bounds__(kThreads) k_range_w(const EncParams P) {
  __shared__ double cta_lo[kWarps], cta_hi[kWarps];
  __shared__ uint32_t cta_nf[kWarps];
  constexpr int VE = 16 / sizeof(T);  // elements per 16-byte load
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const uint64_t gw = (uint64_t)blockIdx.x * kWarps + wid, nw = (uint64_t)gridDim.x * kWarps;
  double run_lo = __longlong_as_double(0x7ff0000000000000ll), run_hi = -run_lo;
  uint32_t nf_all = 0;
  for (uint64_t blk = gw; blk < P.nblocks; blk += nw) {
    const uint64_t first = blk * (uint64_t)P.bs;
    const uint32_t n = (uint32_t)min((uint64_t)P.bs, P.count - first);
    const bool vec = P.vec && (n % VE) == 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const T* base = reinterpret_cast<const T*>(P.axes[a]) + first;
      double lo, hi;
      uint32_t nf = 0;
      if constexpr (sizeof(T) == 4) {
        // float: 32-bit order-preserving keys (fkey), warp REDUX
        int mn = 0x7fffffff, mx = (int)0x80000000;
        uint32_t ex = 0;  // OR of exponent fields == 0xff marks inf / nan
        if (vec) {
          const uint32_t nv = n / VE;
          constexpr int U = 8;
          for (uint32_t c0 = 0; c0 < nv; c0 += 32 * U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t c = c0 + u * 32 + lane;
              v[u] = c < nv ? __ldcs(reinterpret_cast<const uint4*>(base) + c) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (c0 + u * 32 + lane < nv) {
                const uint32_t w4[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                  const int k = fkey(__uint_as_float(w4[j]));
                  mn = min(mn, k);
                  mx = max(mx, k);
                  ex |= ((w4[j] & 0x7f800000u) == 0x7f800000u);
                }
              }
            }
          }
        } else {
          for (uint32_t p = lane; p < n; p += 32) {
            const float f = __ldcs(base + p);
            const int k = fkey(f);
            mn = min(mn, k);
            mx = max(mx, k);
            ex |= !isfinite(f);
          }
        }
        mn = __reduce_min_sync(kFull, mn);
        mx = __reduce_max_sync(kFull, mx);
        nf = __reduce_or_sync(kFull, ex);
        lo = (double)fkey_inv(mn);
        hi = (double)fkey_inv(mx);
      } else {
        unsigned long long mn = ~0ull, mx = 0ull;  // order-preserving keys
        if (vec) {
          const uint32_t nv = n / VE;
          constexpr int U = 8;
          for (uint32_t c0 = 0; c0 < nv; c0 += 32 * U) {
            uint4 v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
              const uint32_t c = c0 + u * 32 + lane;
              v[u] = c < nv ? __ldcs(reinterpret_cast<const uint4*>(base) + c) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
              if (c0 + u * 32 + lane < nv) {
                const double* e = reinterpret_cast<const double*>(&v[u]);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                  if (!isfinite(e[j])) nf = 1;
                  const unsigned long long k = ukey(e[j]);
                  mn = min(mn, k);
                  mx = max(mx, k);
                }
              }
            }
          }
        } else {
          for (uint32_t p = lane; p < n; p += 32) {
            const double f = __ldcs(base + p);
            if (!isfinite(f)) nf = 1;
            const unsigned long long k = ukey(f);
            mn = min(mn, k);
            mx = max(mx, k);
          }
        }
#pragma unroll
        for (int o = 16; o; o >>= 1) {
          mn = min(mn, __shfl_xor_sync(kFull, mn, o));
          mx = max(mx, __shfl_xor_sync(kFull, mx, o));
        }
        nf = __reduce_or_sync(kFull, nf);
        lo = ukey_inv(mn);
        hi = ukey_inv(mx);
      }
      if (lane == 0) {
        T* out = reinterpret_cast<T*>(const_cast<void*>(P.bounds)) + blk * 2 * D;
        out[2 * a] = (T)lo;
        out[2 * a + 1] = (T)hi;
      }
      nf_all |= nf << a;
      run_lo = fmin(run_lo, lo);
      run_hi = fmax(run_hi, hi);
    }
  }
  if (lane == 0) { cta_lo[wid] = run_lo; cta_hi[wid] = run_hi; cta_nf[wid] = nf_all; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double lo = cta_lo[0], hi = cta_hi[0];
    uint32_t nf = cta_nf[0];
    for (int w = 1; w < kWarps; ++w) { lo = fmin(lo, cta_lo[w]); hi = fmax(hi, cta_hi[w]); nf |= cta_nf[w]; }
    if (lo <= hi) {
      atomicMax(&P.res->range_w[0], ukey(-lo));
      atomicMax(&P.res->range_w[1], ukey(hi));
    }
    if (nf) atomicOr(&P.res->nonfinite_mask, nf);
  }
}

// ------------------------------------------------------------------ K1.5
// Per-block geometry record: everything the 32-bit encoder needs, so K2
// never runs the float64 geometry (one thread per block here instead of a
// serial phase inside every K2 CTA).
struct __align__(16) BlkRec {
  double lo[3];       // block minimum per axis (exact)
  double rinv[3];     // RN(1/w), certified-reciprocal quantizer
  double w[3];        // bin width 2*eb_int (exact-division fallback)
  uint32_t N[3];      // segments per axis
  uint32_t PN;        // Π N (narrow blocks: <= 65536)
  uint64_t side_off;  // wide blocks: byte offset of the staged payload
  uint32_t side_len;  // wide blocks: payload length (written by K2w)
  uint8_t b[3];       // log2(m) per axis
  uint8_t sumb;       // Σ log2(m)
  uint8_t kind;       // KIND_* below
  uint8_t path;       // K2 / K2p / K2w: the offset-order path taken (diagnostics, gpzb_encode_path_counts)
  uint8_t pad[22];
};
static_assert(sizeof(BlkRec) == 128, "BlkRec layout");

enum : uint8_t { KIND_NARROW = 0, KIND_WIDE = 1, KIND_ERROR = 2, KIND_WARP = 3, KIND_SMALL = 4 };

// Full float32 blocks with Σ log2 m <= kSmallMaxSumb (16 nibble counters in
// one u64 per segment rank) take the K2s encoder (gpzb_encode_small.cuh).
constexpr uint32_t kSmallMaxSumb = 4;
// Added to t * RN(1/w) by the K2s / K2p quantizers' FMA: 2^-60 (1 + 5 * 2^-52),
// whose low word (5) passes the certificate, so an exact zero (x == block
// minimum) needs no special case; for r >= 2^-8 it moves the product by
// < 2^-8 ulp, inside the certificate's two-ulp slack.
constexpr unsigned long long kCertNudgeBits = 0x3C30000000000005ull;
constexpr uint32_t kSmallMaxPN = 32768;  // ... and Π N <= 2^15

// Narrow blocks the warp encoder K2p takes: full, vector-loadable, no
// offset stream (every log2 m == 0) and Π N <= 16384.
constexpr uint32_t kWarpEncMaxPN = 16384;

// Largest payload a block can produce given its geometry (stream widths are
// bounded by bitlen(ΠN - 1), bitlen(n), Σb and bitlen(n - 1)).
__host__ __device__ inline uint64_t payload_bound(int D, int S, bool pres, uint32_t n, uint32_t wdel_max,
                                                  uint32_t sumb) {
  uint32_t wc = 0, wr = 0;
  for (uint32_t v = n; v; v >>= 1) ++wc;
  for (uint32_t v = n ? n - 1 : 0; v; v >>= 1) ++wr;
  const uint64_t H = 8 + D * (2 * S + 5) + (pres ? 4 : 3);
  return H + (((uint64_t)n * wdel_max + 7) >> 3) + (((uint64_t)n * wc + 7) >> 3) +
         (((uint64_t)n * sumb + 7) >> 3) + (pres ? (((uint64_t)n * wr + 7) >> 3) : 0);
}

template <int D, typename T>
__global__ void __launch_bounds__(256) k_geometry(const EncParams P) {
  const uint64_t blk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  DevResult* R = P.res;
  double eb_abs = P.eb;
  if (P.rel) {  // model.py:194-199, identical IEEE ops
    const double glo = -ukey_inv(R->range_w[0]);
    const double ghi = ukey_inv(R->range_w[1]);
    double span = __dsub_rn(ghi, glo);
    if (span <= 0.0) span = 1.0;
    eb_abs = __dmul_rn(P.eb, span);
  }
  if (blk == 0) R->eb_abs = eb_abs;
  if (blk >= P.nblocks) return;
  const T* bnd = reinterpret_cast<const T*>(P.bounds) + blk * 2 * D;
  BlkRec rec;
  memset(&rec, 0, sizeof(rec));
  int err = R_NONE, eax = 0;
  AxisGeo g[D];
  if (!(eb_abs > 0.0)) {
    err = R_EB_NOT_POSITIVE;
  } else {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (!err && axis_geometry((double)bnd[2 * a], (double)bnd[2 * a + 1], eb_abs, sizeof(T) == 8, P.target, g[a])) {
        err = R_AXIS_RANGE;
        eax = a;
      }
    }
  }
  unsigned __int128 PN = 1;
  uint32_t sumb = 0;
  bool narrow = !P.preserve && P.bs <= (uint32_t)kMaxBs;  // larger blocks: K2b, through the general list
  if (!err) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      PN *= g[a].N;
      if (PN > ((unsigned __int128)1 << 64)) { err = R_GEOMETRY; break; }
      sumb += g[a].b;
      narrow = narrow && g[a].mode == 0;
      rec.lo[a] = g[a].lo;
      rec.rinv[a] = g[a].rinv;
      rec.w[a] = g[a].w;
      rec.N[a] = (uint32_t)g[a].N;
      rec.b[a] = (uint8_t)g[a].b;
    }
    if (!err && sumb > 64) err = R_GEOMETRY;
  }
  if (err) {
    rec.kind = KIND_ERROR;
    atomicMax(&R->err_block, err_code(blk, eax, err));
    P.status[blk] = 0;  // error blocks contribute no bytes
  } else {
    narrow = narrow && PN <= 65536 && sumb <= 32;
    rec.PN = narrow ? (uint32_t)PN : 0u;
    rec.sumb = (uint8_t)sumb;
    if (narrow) {
      const uint64_t n = min((uint64_t)P.bs, P.count - blk * (uint64_t)P.bs);
      const bool full = n == (uint64_t)kMaxBs && P.vec;
      if (full && sizeof(T) == 4 && sumb <= kSmallMaxSumb && PN <= kSmallMaxPN && P.use_small &&
          (sumb > 0 || P.small0)) {
        // K2s (gpzb_encode_small.cuh): with offsets from the front of the list, offset-free from the back
        rec.kind = KIND_SMALL;
        if (sumb) P.small_list[atomicAdd(&R->small_count, 1u)] = (uint32_t)blk;
        else P.small_list[P.nblocks - 1 - atomicAdd(&R->small0_count, 1u)] = (uint32_t)blk;
      } else if (sumb == 0 && PN <= kWarpEncMaxPN && full) {
        rec.kind = KIND_WARP;
      } else {
        rec.kind = KIND_NARROW;
        P.cta_list[atomicAdd(&R->cta_count, 1u)] = (uint32_t)blk;
      }
    } else {
      rec.kind = KIND_WIDE;
      const uint32_t n = (uint32_t)min((uint64_t)P.bs, P.count - blk * (uint64_t)P.bs);
      const uint32_t wdel = (uint32_t)bitlen64((uint64_t)(PN - 1));
      const uint64_t lb = (payload_bound(D, sizeof(T), P.preserve, n, wdel, sumb) + 15) & ~15ull;
      rec.side_off = atomicAdd(&R->side_bytes, (unsigned long long)lb);
      const uint32_t slot = atomicAdd(&R->wide_count, 1u);
      P.wide_list[slot] = (uint32_t)blk;
    }
  }
  {  // K2p's list: one atomic per warp, entries in block order within it
    const bool isw = rec.kind == KIND_WARP;
    const unsigned am = __activemask(), m = __ballot_sync(am, isw);
    if (m) {
      const int lane = threadIdx.x & 31, leader = __ffs(m) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(&R->warp_count, (unsigned)__popc(m));
      base = __shfl_sync(am, base, leader);
      if (isw) P.warp_list[base + __popc(m & ((1u << lane) - 1u))] = (uint32_t)blk;
    }
  }
  reinterpret_cast<BlkRec*>(P.rec)[blk] = rec;
}

// --------------------------------------------------- shared K2 building blocks
// Bitmap rank machinery: zero / set / prefix.  Words [0, nw) of bm, prefix
// counts into wp.  bm_prefix returns the number of set bits.
// bm must be 16B aligned and sized to a multiple of 4 words >= nw.
__device__ __forceinline__ void bm_zero(uint32_t* bm, int nw) {
  for (int w = threadIdx.x; w < (nw + 3) >> 2; w += kThreads) reinterpret_cast<uint4*>(bm)[w] = make_uint4(0, 0, 0, 0);
}
// Each thread owns a run of whole uint4 groups of words.
__device__ __forceinline__ uint32_t bm_prefix(const uint32_t* bm, uint16_t* wp, int nw, uint32_t* scan_ws) {
  const int ng = (nw + 3) >> 2;
  const int gpt = (ng + kThreads - 1) / kThreads;
  const int g0 = threadIdx.x * gpt;
  const int g1 = min(g0 + gpt, ng);
  uint32_t local = 0;
  for (int g = g0; g < g1; ++g) {
    const uint4 q = reinterpret_cast<const uint4*>(bm)[g];
    local += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
  }
  uint32_t total;
  uint32_t run = block_excl_scan<uint32_t>(local, total, scan_ws);
  for (int g = g0; g < g1; ++g) {
    const uint4 q = reinterpret_cast<const uint4*>(bm)[g];
    const uint32_t a = run, b = a + __popc(q.x), c = b + __popc(q.y), d = c + __popc(q.z);
    reinterpret_cast<uint2*>(wp)[g] = make_uint2(a | (b << 16), c | (d << 16));
    run = d + __popc(q.w);
  }
  return total;
}
__device__ __forceinline__ uint32_t bm_rank(const uint32_t* bm, const uint16_t* wp, uint32_t c) {
  const uint32_t w = c >> 5;
  return (uint32_t)wp[w] + __popc(bm[w] & ((1u << (c & 31)) - 1u));
}

// One stable LSD pass over composite (digit << 10 | position): returns the
// new position of each of this thread's elements.
__device__ __forceinline__ void lsd_ranks(const uint32_t (&digit)[kItems], int dlen, int n, int p0,
                                          uint32_t* bm, uint16_t* wp, uint32_t* scan_ws,
                                          uint32_t (&newpos)[kItems]) {
  const int nw = 1 << (dlen + 10 - 5);
  bm_zero(bm, nw);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kItems; ++k)
    if (p0 + k < n) {
      uint32_t c = (digit[k] << 10) | (uint32_t)(p0 + k);
      red_or_shared(&bm[c >> 5], 1u << (c & 31));
    }
  __syncthreads();
  bm_prefix(bm, wp, nw, scan_ws);
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kItems; ++k)
    newpos[k] = (p0 + k < n) ? bm_rank(bm, wp, (digit[k] << 10) | (uint32_t)(p0 + k)) : 0u;
}

__device__ __forceinline__ void put_le(uint8_t* dst, uint64_t v, int nbytes) {
  for (int i = 0; i < nbytes; ++i) dst[i] = (uint8_t)(v >> (8 * i));
}

constexpr unsigned long long kFlagAgg = 1ull << 62, kFlagInc = 2ull << 62, kValMask = kFlagAgg - 1;

}  // namespace gpzb
