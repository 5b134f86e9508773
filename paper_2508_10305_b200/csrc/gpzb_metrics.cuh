// K5: error-bound verification and rate-distortion statistics on the GPU
// (the reference's gpz.metrics, metrics.py:49-152), for datasets far beyond
// what the CPU pairing can handle.
//
//   K5a k_pair_blocks  one CTA per block: both datasets quantized with the
//                      ORIGINAL block's geometry (block_bounds +
//                      derive_geometry + quantize_block with the exact
//                      clip + snap rule, quantizer.py:51-191), then each side
//                      sorted by (seg_id, offset, index) — np.lexsort of
//                      metrics._block_order (metrics.py:49-51) — with a
//                      bitonic network in shared memory; position j of the
//                      two orders is a pair (metrics.pair_blocks, :54-81).
//   K5b k_pair_stats   grid-stride over the pairs: per axis Σ (o - r)^2
//                      (nrmse, :84-104), the field range, max |o - r| and the
//                      pairs beyond eb_abs (verify_bound, :131-152); per-CTA
//                      partials reduced in a fixed order by K5c, so results
//                      are deterministic run to run.
#pragma once

#include "gpzb_common.cuh"

namespace gpzb {

struct PairParams {
  const void* orig[3];
  const void* rec[3];
  uint64_t count;
  uint64_t nblocks;
  uint32_t bs;
  uint32_t target;
  double eb_abs;
  int64_t* orig_idx;  // out (K5a) / in (K5b; null = identity)
  int64_t* rec_idx;
  DevResult* res;
  // K5b
  double* partial;      // [grid][1 + 3 * dims]: max_err, then per axis sumsq, lo, hi
  double* out;          // [1 + 3 * dims] after K5c
  unsigned long long* viol_count;
  unsigned long long* viol;  // [cap][3]: axis << 56 | position, original index, |error| bits
  uint64_t viol_cap;
  uint8_t* big;         // K5a for blocks above 1024 particles: per-CTA key slices
  uint32_t big_grid;
};

template <typename T>
__device__ __forceinline__ bool finite_t(T v) { return isfinite((double)v); }

// Ordered integer keys: min/max of the keys == exact min/max of the values
// (-0.0 orders below +0.0, as in the range kernel K1).
__device__ __forceinline__ unsigned long long okey(double v) { return ukey(v); }

constexpr int kPairSortN = kMaxBs;

struct PairSmem {
  unsigned long long seg[kPairSortN];
  unsigned long long off[kPairSortN];
  uint16_t idx[kPairSortN];
  unsigned long long red[2 * 3 * kWarps];
  AxisGeo geo[3];
  int err;
};

__device__ __forceinline__ bool key_less(const PairSmem& sm, int i, int j) {
  if (sm.seg[i] != sm.seg[j]) return sm.seg[i] < sm.seg[j];
  if (sm.off[i] != sm.off[j]) return sm.off[i] < sm.off[j];
  return sm.idx[i] < sm.idx[j];
}

// Ascending bitonic sort of the 1024 (seg, off, idx) keys in shared memory.
__device__ void bitonic_sort(PairSmem& sm) {
  for (int k = 2; k <= kPairSortN; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int t = threadIdx.x; t < kPairSortN / 2; t += kThreads) {
        const int i = 2 * t - (t & (j - 1));  // lower index of the pair
        const int l = i + j;
        const bool up = (i & k) == 0;
        if (key_less(sm, l, i) == up) {
          const unsigned long long s = sm.seg[i], o = sm.off[i];
          const uint16_t x = sm.idx[i];
          sm.seg[i] = sm.seg[l]; sm.off[i] = sm.off[l]; sm.idx[i] = sm.idx[l];
          sm.seg[l] = s; sm.off[l] = o; sm.idx[l] = x;
        }
      }
      __syncthreads();
    }
  }
}

template <int D, typename T, typename R>
__global__ void __launch_bounds__(kThreads) k_pair_blocks(const PairParams P) {
  __shared__ PairSmem sm;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t blk = blockIdx.x;
  const uint64_t first = blk * (uint64_t)P.bs;
  const int n = (int)min((uint64_t)P.bs, P.count - first);
  constexpr bool F64 = sizeof(T) == 8;

  // ---- original values, their block bounds (quantizer.block_bounds, :51-57)
  double xo[D][kItems], xr[D][kItems];
  unsigned long long kmin[D], kmax[D];
  uint32_t nf = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    kmin[a] = ~0ull;
    kmax[a] = 0ull;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int p = tid * kItems + k;
      xo[a][k] = 0.0;
      xr[a][k] = 0.0;
      if (p < n) {
        const T v = reinterpret_cast<const T*>(P.orig[a])[first + p];
        // the reconstruction in the original's precision (metrics.py:74)
        const T w = (T)reinterpret_cast<const R*>(P.rec[a])[first + p];
        xo[a][k] = (double)v;
        xr[a][k] = (double)w;
        if (!finite_t(v)) nf |= 1u << a;
        if (!finite_t(w)) nf |= 1u << (4 + a);
        const unsigned long long kk = okey((double)v);
        kmin[a] = min(kmin[a], kk);
        kmax[a] = max(kmax[a], kk);
      }
    }
  }
  // exact 64-bit min/max over the CTA (two-step: warp shuffles, then shared)
#pragma unroll
  for (int a = 0; a < D; ++a) {
    unsigned long long mn = kmin[a], mx = kmax[a];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      mn = min(mn, __shfl_xor_sync(kFull, mn, o));
      mx = max(mx, __shfl_xor_sync(kFull, mx, o));
    }
    if (lane == 0) { sm.red[(2 * a) * kWarps + wid] = mn; sm.red[(2 * a + 1) * kWarps + wid] = mx; }
  }
  nf = __reduce_or_sync(kFull, nf);
  if (lane == 0 && nf) atomicOr(&P.res->nonfinite_mask, nf);
  __syncthreads();
  if (tid == 0) {
    int err = R_NONE, eax = 0;
    if (!(P.eb_abs > 0.0)) err = R_EB_NOT_POSITIVE;
    unsigned __int128 pn = 1;
    uint32_t sumb = 0;
    for (int a = 0; a < D && !err; ++a) {
      unsigned long long mn = ~0ull, mx = 0ull;
      for (int w = 0; w < kWarps; ++w) {
        mn = min(mn, sm.red[(2 * a) * kWarps + w]);
        mx = max(mx, sm.red[(2 * a + 1) * kWarps + w]);
      }
      if (axis_geometry(ukey_inv(mn), ukey_inv(mx), P.eb_abs, F64, P.target, sm.geo[a])) {
        err = R_AXIS_RANGE;
        eax = a;
      } else {
        pn *= sm.geo[a].N;
        if (pn > ((unsigned __int128)1 << 64)) pn = ((unsigned __int128)1 << 64) + 1;
        sumb += sm.geo[a].b;
      }
    }
    if (!err && (pn > ((unsigned __int128)1 << 64) || sumb > 64)) err = R_GEOMETRY;
    if (err) atomicMax(&P.res->err_block, err_code(blk, eax, err));
    sm.err = err | (int)nf;
  }
  __syncthreads();
  if (sm.err) return;

  // ---- both sides: quantize with the original's geometry, linearize, sort, emit
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int p = tid * kItems + k;
      unsigned long long seg = ~0ull, off = ~0ull;
      if (p < n) {
        seg = 0;
        off = 0;
        unsigned long long stride = 1;
        uint32_t shift = 0;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const AxisGeo& g = sm.geo[a];
          const double x = side ? xr[a][k] : xo[a][k];
          const uint64_t q = quantize_snap(x, g, P.eb_abs, F64);  // quantizer.py:142-173
          seg += shr64(q, g.b) * stride;                           // quantizer.py:176-191
          off |= shl64(q & (g.b >= 64 ? ~0ull : ((1ull << g.b) - 1)), shift);
          stride *= g.N;
          shift += g.b;
        }
      }
      sm.seg[p] = seg;
      sm.off[p] = off;
      sm.idx[p] = (uint16_t)p;
    }
    __syncthreads();
    bitonic_sort(sm);
    int64_t* dst = side ? P.rec_idx : P.orig_idx;
    for (int p = tid; p < n; p += kThreads) dst[first + p] = (int64_t)(first + sm.idx[p]);
    __syncthreads();
  }
}

// K5a for blocks of more than 1024 particles (gpzb_big.cuh's layout): one
// CTA per block, persistent; the (seg, off, index) keys of each side in a
// per-CTA slice of `scratch` (big_enc_slice bytes), padded with all-ones keys
// to a power of two and bitonic-sorted there; same results as k_pair_blocks.
template <int D, typename T, typename R>
__global__ void __launch_bounds__(kThreads) k_pair_blocks_big(const PairParams P, uint8_t* scratch, uint64_t npad,
                                                              uint64_t slice) {
  __shared__ unsigned long long red[2 * 3 * kWarps];
  __shared__ AxisGeo geo[3];
  __shared__ int serr;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  constexpr bool F64 = sizeof(T) == 8;
  unsigned long long* seg = reinterpret_cast<unsigned long long*>(scratch + blockIdx.x * slice);
  unsigned long long* off = seg + npad;
  uint32_t* idx = reinterpret_cast<uint32_t*>(off + npad);
  for (uint64_t blk = blockIdx.x; blk < P.nblocks; blk += gridDim.x) {
    __syncthreads();
    const uint64_t first = blk * (uint64_t)P.bs;
    const uint32_t n = (uint32_t)min((uint64_t)P.bs, P.count - first);
    // ---- the original block's bounds (quantizer.block_bounds) and finiteness of both sides
    unsigned long long kmin[D], kmax[D];
    uint32_t nf = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) { kmin[a] = ~0ull; kmax[a] = 0ull; }
    for (uint32_t p = tid; p < n; p += kThreads) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const T v = reinterpret_cast<const T*>(P.orig[a])[first + p];
        const T w = (T)reinterpret_cast<const R*>(P.rec[a])[first + p];  // metrics.py:74
        if (!finite_t(v)) nf |= 1u << a;
        if (!finite_t(w)) nf |= 1u << (4 + a);
        const unsigned long long kk = okey((double)v);
        kmin[a] = min(kmin[a], kk);
        kmax[a] = max(kmax[a], kk);
      }
    }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      unsigned long long mn = kmin[a], mx = kmax[a];
#pragma unroll
      for (int o = 16; o; o >>= 1) {
        mn = min(mn, __shfl_xor_sync(kFull, mn, o));
        mx = max(mx, __shfl_xor_sync(kFull, mx, o));
      }
      if (lane == 0) { red[(2 * a) * kWarps + wid] = mn; red[(2 * a + 1) * kWarps + wid] = mx; }
    }
    nf = __reduce_or_sync(kFull, nf);
    if (lane == 0 && nf) atomicOr(&P.res->nonfinite_mask, nf);
    __syncthreads();
    if (tid == 0) {
      int err = R_NONE, eax = 0;
      if (!(P.eb_abs > 0.0)) err = R_EB_NOT_POSITIVE;
      unsigned __int128 pn = 1;
      uint32_t sumb = 0;
      for (int a = 0; a < D && !err; ++a) {
        unsigned long long mn = ~0ull, mx = 0ull;
        for (int w = 0; w < kWarps; ++w) {
          mn = min(mn, red[(2 * a) * kWarps + w]);
          mx = max(mx, red[(2 * a + 1) * kWarps + w]);
        }
        if (axis_geometry(ukey_inv(mn), ukey_inv(mx), P.eb_abs, F64, P.target, geo[a])) {
          err = R_AXIS_RANGE;
          eax = a;
        } else {
          pn *= geo[a].N;
          if (pn > ((unsigned __int128)1 << 64)) pn = ((unsigned __int128)1 << 64) + 1;
          sumb += geo[a].b;
        }
      }
      if (!err && (pn > ((unsigned __int128)1 << 64) || sumb > 64)) err = R_GEOMETRY;
      if (err) atomicMax(&P.res->err_block, err_code(blk, eax, err));
      serr = err;  // non-finite values: reported as DomainError by the host (results discarded)
    }
    __syncthreads();
    if (serr) continue;
    // ---- each side: keys with the original's geometry, sorted; positional pairs
    for (int side = 0; side < 2; ++side) {
      for (uint64_t p = tid; p < npad; p += kThreads) {
        unsigned long long s = ~0ull, o = ~0ull;
        uint32_t ix = ~0u;
        if (p < n) {
          s = 0;
          o = 0;
          ix = (uint32_t)p;
          unsigned long long stride = 1;
          uint32_t shift = 0;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const AxisGeo& g = geo[a];
            const double x = side ? (double)(T)reinterpret_cast<const R*>(P.rec[a])[first + p]
                                  : (double)reinterpret_cast<const T*>(P.orig[a])[first + p];
            const uint64_t q = quantize_snap(x, g, P.eb_abs, F64);  // quantizer.py:142-173
            s += shr64(q, g.b) * stride;                           // quantizer.py:176-191
            o |= shl64(q & (g.b >= 64 ? ~0ull : ((1ull << g.b) - 1)), shift);
            stride *= g.N;
            shift += g.b;
          }
        }
        seg[p] = s;
        off[p] = o;
        idx[p] = ix;
      }
      __syncthreads();
      for (uint64_t k = 2; k <= npad; k <<= 1) {
        for (uint64_t j = k >> 1; j > 0; j >>= 1) {
          for (uint64_t i = tid; i < npad; i += kThreads) {
            const uint64_t l = i ^ j;
            if (l > i) {
              const unsigned long long s1 = seg[i], o1 = off[i], s2 = seg[l], o2 = off[l];
              const uint32_t i1 = idx[i], i2 = idx[l];
              const bool lt21 = s2 < s1 || (s2 == s1 && (o2 < o1 || (o2 == o1 && i2 < i1)));
              const bool lt12 = s1 < s2 || (s1 == s2 && (o1 < o2 || (o1 == o2 && i1 < i2)));
              if ((i & k) == 0 ? lt21 : lt12) {
                seg[i] = s2; off[i] = o2; idx[i] = i2;
                seg[l] = s1; off[l] = o1; idx[l] = i1;
              }
            }
          }
          __syncthreads();
        }
      }
      int64_t* dst = side ? P.rec_idx : P.orig_idx;
      for (uint32_t p = tid; p < n; p += kThreads) dst[first + p] = (int64_t)(first + idx[p]);
      __syncthreads();
    }
  }
}

template <int D, typename T, typename R>
__global__ void __launch_bounds__(kThreads) k_pair_stats(const PairParams P) {
  constexpr int NS = 1 + 3 * D;
  __shared__ double red[kWarps][NS];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  double mx_err = 0.0, sq[D], lo[D], hi[D];
#pragma unroll
  for (int a = 0; a < D; ++a) { sq[a] = 0.0; lo[a] = INFINITY; hi[a] = -INFINITY; }
  for (uint64_t i = blockIdx.x * (uint64_t)kThreads + tid; i < P.count; i += (uint64_t)gridDim.x * kThreads) {
    const uint64_t oi = P.orig_idx ? (uint64_t)P.orig_idx[i] : i;
    const uint64_t ri = P.rec_idx ? (uint64_t)P.rec_idx[i] : i;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double o = (double)reinterpret_cast<const T*>(P.orig[a])[oi];
      const double r = (double)reinterpret_cast<const R*>(P.rec[a])[ri];
      const double d = __dsub_rn(o, r);
      sq[a] = __dadd_rn(sq[a], __dmul_rn(d, d));
      lo[a] = fmin(lo[a], o);
      hi[a] = fmax(hi[a], o);
      const double e = fabs(d);
      mx_err = fmax(mx_err, e);
      if (e > P.eb_abs) {
        const unsigned long long slot = atomicAdd(P.viol_count, 1ull);
        if (slot < P.viol_cap) {
          P.viol[3 * slot] = ((unsigned long long)a << 56) | i;
          P.viol[3 * slot + 1] = oi;
          P.viol[3 * slot + 2] = (unsigned long long)__double_as_longlong(e);
        }
      }
    }
  }
  // fixed-order reduction: warp butterflies, then warps in index order
  double v[NS];
  v[0] = mx_err;
#pragma unroll
  for (int a = 0; a < D; ++a) { v[1 + 3 * a] = sq[a]; v[2 + 3 * a] = lo[a]; v[3 + 3 * a] = hi[a]; }
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    const int kind = s == 0 ? 0 : (s - 1) % 3;  // 0 max | 0 sum, 1 min, 2 max
    double x = v[s];
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      const double y = __shfl_xor_sync(kFull, x, o);
      x = s == 0 ? fmax(x, y) : kind == 0 ? __dadd_rn(x, y) : kind == 1 ? fmin(x, y) : fmax(x, y);
    }
    if (lane == 0) red[wid][s] = x;
  }
  __syncthreads();
  if (tid < NS) {
    const int s = tid, kind = s == 0 ? 0 : (s - 1) % 3;
    double x = red[0][s];
    for (int w = 1; w < kWarps; ++w) {
      const double y = red[w][s];
      x = s == 0 ? fmax(x, y) : kind == 0 ? __dadd_rn(x, y) : kind == 1 ? fmin(x, y) : fmax(x, y);
    }
    P.partial[blockIdx.x * (uint64_t)NS + s] = x;
  }
}

// K5c: the per-CTA partials, reduced in index order by one thread per statistic.
template <int D>
__global__ void k_pair_stats_final(const PairParams P, int nparts) {
  constexpr int NS = 1 + 3 * D;
  const int s = threadIdx.x;
  if (s >= NS) return;
  const int kind = s == 0 ? 0 : (s - 1) % 3;
  double x = s == 0 ? 0.0 : kind == 0 ? 0.0 : kind == 1 ? INFINITY : -INFINITY;
  for (int i = 0; i < nparts; ++i) {
    const double y = P.partial[(uint64_t)i * NS + s];
    x = s == 0 ? fmax(x, y) : kind == 0 ? __dadd_rn(x, y) : kind == 1 ? fmin(x, y) : fmax(x, y);
  }
  P.out[s] = x;
}

}  // namespace gpzb
