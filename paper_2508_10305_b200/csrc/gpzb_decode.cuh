// K4a + K4: the GPZ B200 decompressor.
//
// Together they restate pipeline._decode_block (pipeline.py:106-157) for
// every block, plus read_container's offset-table checks
// (container.py:282-290) and the per-block count check (pipeline.py:174-181):
//
//   K4a k_decode_plan  one thread per block: table entries, parse_block's
//                      header checks and exact stream lengths
//                      (container.py:128-193), the re-derived geometry
//                      (pipeline.py:128-145), the finiteness bound of the
//                      reconstruction; writes a 128-byte record per block
//   K4  k_decode       one CTA per block: payload window -> unpack_fixed
//                      (codec.py:132-151) -> delta / run-length decode with
//                      the decoder's checks (pipeline.py:116-125) ->
//                      _delinearize + dequantize_block (quantizer.py:194-272)
//                      -> rank scatter (pipeline.py:149-156) -> stores
//
// The first failing check of the lowest failing block is reported, in the
// reference's order: K4a reports header errors directly and hands the
// geometry errors to K4 as bits ranked behind the stream checks.
#pragma once

#include <type_traits>

#include "gpzb_common.cuh"

namespace gpzb {

struct __align__(16) DecRec {
  double lo[3];       // block minimum per axis (f64)
  double w[3];        // bin width 2*eb_int
  uint64_t e0;        // payload start within the payload region
  uint64_t PN;        // Π N, saturated at 2^64-1
  uint32_t N[3];      // segments per axis (u32 in the header)
  uint32_t mg_m[3];   // magic multiplier for / N
  uint32_t n, U;      // particles, unique ids
  uint16_t sd, sc, so, sr;  // stream byte offsets within the payload
  uint8_t b[3];       // log2(m)
  uint8_t mg_l[3];    // magic shift
  uint8_t wd, wc, wo, wr;
  uint8_t kind;       // 0 CTA decoder, 1 skip (error already reported / table error), 2 warp decoder
  uint8_t sumb;
  uint8_t fast_mask;  // bit a: magic-constant midpoint valid (q < 2^51)
  uint8_t geo_bits;   // bit 2a: axis range overflow, bit 2a+1: N inconsistent
  uint8_t chk_mask;   // bit a: reconstruction may be non-finite -> per-element check
  uint8_t pn_big;     // Π N > 2^32 (64-bit delinearisation)
  uint8_t pn_all;     // Π N >= 2^64 (every id in range)
  uint8_t fast_body;  // 32-bit decode body applies (see k_decode); 2: with the midpoint table; 3: 32-bit q
  uint16_t lut1, lut2;  // fast_body 2: table offsets of axes 1 and 2 (axis 0 starts at 0)
  uint16_t lut_n;       // table entries Σ N_a 2^b_a when <= kLutEntries (else 0); lut1/lut2 valid then
};
static_assert(sizeof(DecRec) == 128, "DecRec layout");

struct DecParams {
  const uint8_t* c;        // container (device)
  uint64_t len;
  uint64_t table_end, payload_len;
  uint64_t nblocks, count;
  uint32_t bs;
  double eb_abs;
  void* out[3];
  uint64_t out_cap;
  const uint64_t* out_offsets;  // null: block i starts at i*bs
  DevResult* res;
  DecRec* rec;
  uint32_t* list;          // K4a: blocks for the CTA decoder (count in res->wide_count)
  uint64_t blk_lo, blk_hi; // this launch decodes blocks [blk_lo, blk_hi) (chunked host pipelines)
  uint8_t* big;            // K4b: per-CTA workspace slices (block_size > 1024)
  uint64_t pf_dist;        // K4w: L2 prefetch distance in payload bytes (0 = off), set at launch
  uint64_t pf_blks;        // K4w: the same distance in blocks
};

constexpr int kDecStageWords = 5120;  // 20 KB payload window (legit blocks <= 19.2 KB)
#ifndef GPZB_LUT_UMAX
#define GPZB_LUT_UMAX 512
#endif
constexpr int kLutEntries = 4096;     // midpoint table (f32 entries) in the window after unpacking

__device__ __forceinline__ uint64_t ld_le(const uint8_t* p, int nbytes) {
  uint64_t v = 0;
  for (int i = 0; i < nbytes; ++i) v |= (uint64_t)p[i] << (8 * i);
  return v;
}

// floor(n / d) for 32-bit n via a multiply-high (Granlund-Montgomery,
// round-up variant); d == 1 is handled by l == 0.
__device__ __forceinline__ uint32_t magic_div(uint32_t n, uint32_t m, uint32_t l) {
  if (l == 0) return n;
  const uint32_t t = __umulhi(m, n);
  return (t + ((n - t) >> 1)) >> (l - 1);
}

// ---------------------------------------------------------------------- K4a
template <int D, bool F64, bool PRES>
__global__ void __launch_bounds__(256) k_decode_plan(const DecParams P) {
  using T = typename std::conditional<F64, double, float>::type;
  constexpr int S = F64 ? 8 : 4;
  constexpr uint32_t HS = 8 + D * (2 * S + 5) + (PRES ? 4 : 3);
  const uint64_t blk = P.blk_lo + blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (blk >= P.blk_hi) return;
  DevResult* R = P.res;
  if (blk == P.blk_lo) R->claim = 0;  // K4w runs after this launch (same stream)
  DecRec rec;
  memset(&rec, 0, sizeof(rec));
  rec.kind = 1;
  const uint8_t* table = P.c + GPZB_GLOBAL_HEADER_SIZE;
  const uint64_t e0 = ld_le(table + 8 * blk, 8);
  const uint64_t e1 = ld_le(table + 8 * blk + 8, 8);
  uint32_t tf = 0;
  if (blk == 0 && e0 != 0) tf |= 1;
  if (e0 > e1) tf |= 2;
  if (blk + 1 == P.nblocks && e1 != P.payload_len) tf |= 4;
  if (tf) atomicOr(&R->table_flags, tf);
  if (tf || e1 > P.payload_len) {  // reported container-wide
    P.rec[blk] = rec;
    return;
  }
  const uint64_t L = e1 - e0;
  const uint8_t* pb = P.c + P.table_end + e0;
  // ---- parse_block header checks, in the reference's order
  uint32_t e = 0, eax = 0, n = 0, U = 0;
  uint32_t w4[4] = {0, 0, 0, 0};
  double lo[D], hi[D];
  if (L < HS) {
    e = R_BLK_SHORT;
  } else {
    n = (uint32_t)ld_le(pb, 4);
    U = (uint32_t)ld_le(pb + 4, 4);
    const uint8_t* wp = pb + 8 + D * (2 * S + 5);
    for (int s = 0; s < (PRES ? 4 : 3); ++s) w4[s] = wp[s];
    if (U > n) e = R_BLK_UNIQUE;
    if (!e && (w4[0] > 64 || w4[1] > 64 || w4[2] > 64 || w4[3] > 64)) e = R_BLK_WIDTH;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const uint8_t* ap = pb + 8 + a * (2 * S + 5);
      if (F64) {
        lo[a] = __longlong_as_double((long long)ld_le(ap, 8));
        hi[a] = __longlong_as_double((long long)ld_le(ap + 8, 8));
      } else {
        lo[a] = (double)__uint_as_float((uint32_t)ld_le(ap, 4));
        hi[a] = (double)__uint_as_float((uint32_t)ld_le(ap + 4, 4));
      }
      rec.b[a] = ap[2 * S];
      rec.N[a] = (uint32_t)ld_le(ap + 2 * S + 1, 4);
      if (!e) {
        if (rec.N[a] < 1 && n > 0) { e = R_BLK_NOSEG; eax = a; }
        else if (rec.b[a] > 63) { e = R_BLK_OFFBITS; eax = a; }
        else if (!(isfinite(lo[a]) && isfinite(hi[a]) && lo[a] <= hi[a])) { e = R_BLK_BOUNDS; eax = a; }
      }
    }
    if (!e) {
      uint64_t cur = HS;
      const uint64_t cnts[4] = {U, U, n, n};
      uint32_t so[4] = {0, 0, 0, 0};
      for (int s = 0; s < (PRES ? 4 : 3) && !e; ++s) {
        const uint64_t nb = (cnts[s] * w4[s] + 7) >> 3;
        so[s] = (uint32_t)cur;
        if (cur + nb > L) e = R_BLK_TRUNC;
        cur += nb;
      }
      if (!e && cur != L) e = R_BLK_TRAILING;
      rec.sd = (uint16_t)so[0]; rec.sc = (uint16_t)so[1]; rec.so = (uint16_t)so[2]; rec.sr = (uint16_t)so[3];
    }
    const __int128 want = (blk + 1 < P.nblocks) ? (__int128)P.bs
                          : (__int128)P.count - (__int128)P.bs * (__int128)(P.nblocks - 1);
    if (P.bs <= (uint32_t)kMaxBs) {  // CTA decoders: the payload window and 1024 particles
      if (!e && L > (uint64_t)(kDecStageWords * 4 - 16)) e = R_BLK_WINDOW;  // only with oversized widths
      if (!e && n > (uint32_t)kMaxBs) e = ((__int128)n == want) ? R_UNSUPPORTED_BS : R_BLK_TOO_BIG;
    } else if (!e && n > P.bs) {  // K4b: per-CTA slices of block_size particles
      e = R_BLK_TOO_BIG;
    }
    // per-block count vs the boundary math (pipeline.py:174-181), ranked
    // behind every decode check of the same block by the host
    if (!e && (__int128)n != want) atomicMax(&R->err_count, err_code(blk, 0, R_BLK_COUNT));
  }
  if (e) {
    atomicMax(&R->err_block, err_code(blk, eax, e));
    P.rec[blk] = rec;
    return;
  }
  rec.kind = 0;
  rec.e0 = e0;
  rec.n = n;
  rec.U = U;
  rec.wd = (uint8_t)w4[0]; rec.wc = (uint8_t)w4[1]; rec.wo = (uint8_t)w4[2]; rec.wr = (uint8_t)w4[3];
  // ---- geometry re-derived from the stored bounds (pipeline.py:128-145)
  unsigned __int128 pn = 1;
  uint32_t sumb = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    bool half;
    const double eb_int = inner_bound(P.eb_abs, lo[a], hi[a], F64, half);
    const double w = __dmul_rn(2.0, eb_int);
    const double span = __dsub_rn(hi[a], lo[a]);
    uint64_t Q = 1;
    if (span > 0.0) {
      const double ratio = __ddiv_rn(span, w);
      if (!(ratio < 18446744073709551616.0)) rec.geo_bits |= (uint8_t)(1u << (2 * a));
      else Q = (uint64_t)__double2ull_rz(ratio) + 1;
    }
    const uint32_t b = rec.b[a];
    if (!(rec.geo_bits & (1u << (2 * a))) && n > 0) {
      const uint64_t m = 1ull << b;
      if (Q / m + (Q % m ? 1 : 0) != rec.N[a]) rec.geo_bits |= (uint8_t)(2u << (2 * a));
    }
    const uint32_t Na = rec.N[a];
    uint32_t l = 0, mg = 0;
    if (Na > 1) {
      l = 32 - __clz((int)(Na - 1));
      mg = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << l) - Na)) / Na + 1);
    }
    rec.mg_m[a] = mg;
    rec.mg_l[a] = (uint8_t)l;
    rec.lo[a] = lo[a];
    rec.w[a] = w;
    if (b < 51 && (uint64_t)Na <= ((1ull << 51) >> b)) rec.fast_mask |= (uint8_t)(1u << a);
    // reconstruction range: q in [0, N*2^b) maps monotonically into
    // [mid(0), mid(N*2^b - 1)]; both ends finite => every output finite
    const unsigned __int128 qmax = ((unsigned __int128)(Na ? Na : 1) << b) - 1;
    const uint64_t q1 = qmax > 0xffffffffffffffffull ? 0xffffffffffffffffull : (uint64_t)qmax;
    const T vmax = (T)__dadd_rn(lo[a], __dmul_rn(__dadd_rn(__ull2double_rn(q1), 0.5), w));
    const T vmin = (T)__dadd_rn(lo[a], __dmul_rn(0.5, w));
    if (!isfinite((double)vmax) || !isfinite((double)vmin) || qmax > 0xffffffffffffffffull)
      rec.chk_mask |= (uint8_t)(1u << a);
    pn *= Na;
    if (pn > ((unsigned __int128)1 << 64)) pn = ((unsigned __int128)1 << 64) + 1;
    sumb += b;
  }
  rec.PN = pn > 0xffffffffffffffffull ? 0xffffffffffffffffull : (uint64_t)pn;
  rec.pn_all = pn >= ((unsigned __int128)1 << 64);
  rec.pn_big = pn > 0xffffffffull;
  rec.sumb = (uint8_t)sumb;
  rec.fast_body = (n == (uint32_t)kMaxBs && P.bs <= (uint32_t)kMaxBs && !PRES && w4[0] <= 32 && w4[1] <= 32 && w4[2] <= 32 && sumb <= 32 &&
                   !rec.pn_big && rec.fast_mask == (1u << D) - 1 && rec.chk_mask == 0 && rec.geo_bits == 0)
                      ? 1 : 0;
  if (rec.fast_body) {
    // every reconstructable value of the block, one table entry per bin
    // (q in [0, N_a 2^b_a) per axis), when the table fits the stage
    uint64_t tot = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (a == 1) rec.lut1 = (uint16_t)tot;
      if (a == 2) rec.lut2 = (uint16_t)tot;
      tot += (uint64_t)rec.N[a] << rec.b[a];
    }
    if (tot <= (uint64_t)kLutEntries / (F64 ? 2 : 1)) rec.lut_n = (uint16_t)tot;  // table offsets valid
    if (rec.lut_n && U <= GPZB_LUT_UMAX) {
      rec.fast_body = 2;
    } else {
      bool q31 = true;
#pragma unroll
      for (int a = 0; a < D; ++a) q31 = q31 && rec.b[a] <= 30 && ((uint64_t)rec.N[a] << rec.b[a]) <= (1ull << 31);
      if (q31) rec.fast_body = 3;  // 32-bit bin indices (k_decode fast body)
    }
  }
  // route: the warp decoder (K4w) takes fast-body blocks whose payload
  // window fits its 4 KB stage; the CTA decoder gets the rest via the list
  {
    const uint32_t al = (uint32_t)((uintptr_t)(P.c + P.table_end + e0) & 15);
    const uint32_t plen = rec.so + ((kMaxBs * (uint32_t)rec.wo + 7) >> 3);
    if (rec.fast_body && al + plen + 16 <= 4096u) {
      rec.kind = 2;
    } else if (P.list) {
      P.list[atomicAdd(&R->wide_count, 1u)] = (uint32_t)blk;
    }
  }
  P.rec[blk] = rec;
}

// ---------------------------------------------------------------------- K4
struct DecSmem {
  unsigned long long scan[2 * kWarps];
  uint32_t red[kWarps];
  uint32_t seen[kMaxBs / 32];
  uint32_t rstart[kMaxBs / 32];  // fast path: bit p set <=> a run starts at position p
  __align__(16) uint32_t words[kDecStageWords];
  __align__(16) uint64_t uniq[kMaxBs];
  __align__(16) uint32_t starts[kMaxBs];
};

__device__ __forceinline__ uint32_t get_bits32(const uint32_t* st, uint32_t pos, uint32_t nbits) {
  const uint32_t sh = pos & 31;
  const uint32_t* w = st + (pos >> 5);
  const uint32_t v = __funnelshift_r(w[0], w[1], sh);
  return nbits >= 32 ? v : (v & ((1u << nbits) - 1u));
}

// Exclusive block scan of two u64 values at once (one barrier pair).
__device__ __forceinline__ void block_excl_scan2(unsigned long long& a, unsigned long long& b,
                                                 unsigned long long& ta, unsigned long long& tb,
                                                 unsigned long long* ws) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long xa = a, xb = b;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long ya = __shfl_up_sync(kFull, xa, o), yb = __shfl_up_sync(kFull, xb, o);
    if (lane >= o) { xa += ya; xb += yb; }
  }
  if (lane == 31) { ws[wid] = xa; ws[kWarps + wid] = xb; }
  __syncthreads();
  unsigned long long sa = (lane < kWarps) ? ws[lane] : 0ull, sb = (lane < kWarps) ? ws[kWarps + lane] : 0ull;
#pragma unroll
  for (int o = 1; o < kWarps; o <<= 1) {
    const unsigned long long ya = __shfl_up_sync(kFull, sa, o), yb = __shfl_up_sync(kFull, sb, o);
    if (lane >= o) { sa += ya; sb += yb; }
  }
  ta = __shfl_sync(kFull, sa, kWarps - 1);
  tb = __shfl_sync(kFull, sb, kWarps - 1);
  const unsigned long long pa = __shfl_sync(kFull, sa, wid) - __shfl_sync(kFull, xa, 31);
  const unsigned long long pb = __shfl_sync(kFull, sb, wid) - __shfl_sync(kFull, xb, 31);
  a = pa + xa - a;
  b = pb + xb - b;
  __syncthreads();
}

#ifndef GPZB_K4_MINB
#define GPZB_K4_MINB 6
#endif

// Load the payload window into shared memory (16B chunks; edges bytewise).
__device__ __forceinline__ void load_window(const DecParams& P, DecSmem& sm, const uint8_t* pay, uint32_t al,
                                            uint32_t plen) {
  const uint8_t* g16 = pay - al;
  const uint8_t* cend = P.c + P.len;
  const uint32_t nch = (al + plen + 15) >> 4;
  for (uint32_t ch = threadIdx.x; ch < nch; ch += kThreads) {
    const uint8_t* src = g16 + 16 * ch;
    uint4 v;
    if (src >= P.c && src + 16 <= cend) {
      v = __ldcs(reinterpret_cast<const uint4*>(src));
    } else {
      uint32_t w[4] = {0, 0, 0, 0};
      for (int j = 0; j < 16; ++j)
        if (src + j >= P.c && src + j < cend) w[j >> 2] |= (uint32_t)src[j] << (8 * (j & 3));
      v = make_uint4(w[0], w[1], w[2], w[3]);
    }
    reinterpret_cast<uint4*>(sm.words)[ch] = v;
  }
}

__device__ __forceinline__ void report_decode_error(DevResult* R, uint64_t blk, uint32_t bits) {
  const int bit = __ffs((int)bits) - 1;
  int reason, ax = 0;
  switch (bit) {
    case 0: reason = R_BLK_PAD_DELTA; break;
    case 1: reason = R_BLK_PAD_COUNT; break;
    case 2: reason = R_BLK_PAD_OFF; break;
    case 3: reason = R_BLK_IDS; break;
    case 4: reason = R_BLK_ZERO_RUN; break;
    case 5: reason = R_BLK_RUN_SUM; break;
    case 6: reason = R_BLK_RUN_MAX; break;
    case 13: reason = R_BLK_SEG_RANGE; break;
    case 14: reason = R_BLK_OFF_RANGE; break;
    case 15: reason = R_BLK_PAD_RANK; break;
    case 16: reason = R_BLK_RANKS; break;
    default: ax = (bit - 7) >> 1; reason = ((bit - 7) & 1) ? R_BLK_SEGCOUNT : R_BLK_AXIS_RANGE; break;
  }
  atomicMax(&R->err_block, err_code(blk, ax, reason));
}

// 32-bit decode body (K4a fast_body): a full 1024-particle block, every
// stream width <= 32, Σ log2 m <= 32, Π N <= 2^32, magic-constant midpoints
// on every axis and a reconstruction range proven finite.  Same checks and
// results as decode_general, fewer instructions.
template <int D, bool F64>
__device__ __forceinline__ void decode_fast(const DecParams& P, DecSmem& sm, const uint64_t blk, const DecRec* rec) {
  using T = typename std::conditional<F64, double, float>::type;
  const int tid = threadIdx.x;
  DevResult* R = P.res;
  const uint32_t U = rec->U;
  const uint32_t wd = rec->wd, wc = rec->wc, wo = rec->wo;
  const uint32_t sd = rec->sd, sc = rec->sc, so = rec->so;
  const uint8_t* pay = P.c + P.table_end + rec->e0;
  const uint32_t al = (uint32_t)((uintptr_t)pay & 15);
  const uint32_t plen = so + ((kMaxBs * wo + 7) >> 3);
  load_window(P, sm, pay, al, plen);
  if (tid < kMaxBs / 32) sm.rstart[tid] = 0;
  __syncthreads();
  const uint8_t* pb = reinterpret_cast<const uint8_t*>(sm.words) + al;
  const uint32_t pbit = 8 * al;
  const int p0 = tid * kItems;
  uint32_t fl = 0;
  if (tid < 3) {  // zero padding (codec.py:147-148)
    const uint32_t cnt = tid < 2 ? U : (uint32_t)kMaxBs;
    const uint32_t w = tid == 0 ? wd : tid == 1 ? wc : wo;
    const uint32_t st = tid == 0 ? sd : tid == 1 ? sc : so;
    const uint32_t used = cnt * w, nb = (used + 7) >> 3;
    if (w && cnt && (used & 7) && (pb[st + nb - 1] >> (used & 7))) fl |= 1u << tid;
  }
  unsigned long long dsum = 0;
  uint32_t csum = 0;
  uint32_t dl[kItems], cn[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t r = p0 + j;
    dl[j] = cn[j] = 0;
    if (r < U) {
      dl[j] = get_bits32(sm.words, pbit + 8 * sd + r * wd, wd);
      cn[j] = get_bits32(sm.words, pbit + 8 * sc + r * wc, wc);
    }
    dsum += dl[j];
    csum += cn[j];
  }
  uint32_t off[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) off[k] = get_bits32(sm.words, pbit + 8 * so + (p0 + k) * wo, wo);
  const bool lut = rec->fast_body == 2;
  // one u64 scan for both sums: Σ deltas < 1024 * 2^32 = 2^42 (widths <= 32)
  // in the low 43 bits, run lengths above them, clamped per thread at 1025
  // (a valid block sums to exactly 1024, so clamping never hides an error)
  constexpr int kDBits = 43;
  constexpr unsigned long long kDMask = (1ull << kDBits) - 1;
  unsigned long long tot;
  const unsigned long long ex =
      block_excl_scan<unsigned long long>(((unsigned long long)min(csum, 1025u) << kDBits) | dsum, tot, sm.scan);
  const unsigned long long ctot = tot >> kDBits;
  {
    uint64_t prev = ex & kDMask;
    uint32_t cex = (uint32_t)(ex >> kDBits);
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t r = p0 + j;
      if (r < U) {
        const uint64_t u = prev + dl[j];
        if (r > 0 && u <= prev) fl |= 1u << 3;   // pipeline.py:116-117
        if (cn[j] < 1) fl |= 1u << 4;             // pipeline.py:118-119
        if (u >= rec->PN) fl |= 1u << 13;         // quantizer.py:262-263
        sm.uniq[r] = u;
        if (cex < (uint32_t)kMaxBs) red_or_shared(&sm.rstart[cex >> 5], 1u << (cex & 31));
        cex += cn[j];
        prev = u;
      }
    }
  }
  if (ctot != (unsigned long long)kMaxBs) fl |= 1u << 5;  // pipeline.py:120-123
  {
    const uint32_t sb = rec->sumb;
    if (sb < 32) {
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (off[k] >> sb) fl |= 1u << 14;  // quantizer.py:264-265
    }
  }
  if (__syncthreads_or(fl != 0)) {
    uint32_t v[1] = {fl};
    block_or<1>(v, sm.red);
    if (tid == 0) report_decode_error(R, blk, v[0]);
    return;
  }
  // run index of every position = (run starts at or before it) - 1: a rank
  // in the 1024-bit run-start map (counts are validated: >= 1, summing to
  // 1024, so the starts are distinct and in range)
  uint32_t run[kItems];
  {
    const int lane = tid & 31;
    const uint32_t c = __popc(sm.rstart[lane]);
    uint32_t incl = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const int wsel = p0 >> 5;  // this thread's 4 positions share one map word
    const uint32_t base = __shfl_sync(kFull, incl - c, wsel);
    const uint32_t word = sm.rstart[wsel];
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint32_t b = (uint32_t)(p0 + k) & 31;
      run[k] = base + __popc(word & (0xffffffffu >> (31 - b))) - 1;
    }
  }
  T vals[D][kItems];
  if (lut) {
    // midpoint table over the (now consumed) payload window, then one lookup per coordinate
    T* tab = reinterpret_cast<T*>(sm.words);
    const uint32_t nt = rec->lut_n, l1 = rec->lut1, l2 = rec->lut2;
    for (uint32_t i = tid; i < nt; i += kThreads) {
      const int a = (D > 2 && i >= l2) ? 2 : (D > 1 && i >= l1) ? 1 : 0;
      const uint32_t q = i - (a == 0 ? 0u : a == 1 ? l1 : l2);
      const double h = __longlong_as_double((long long)(0x4320000000000000ull + 2 * (uint64_t)q + 1));
      const double aq = __dsub_rn(h, 2251799813685248.0);
      tab[i] = (T)__dadd_rn(rec->lo[a], __dmul_rn(aq, rec->w[a]));
    }
    // each run's table bases (bin seg_a << b_a per axis, 16 bits per axis),
    // spread over all threads (U may be far below the thread count)
    for (uint32_t r = tid; r < U; r += kThreads) {
      uint32_t rest = (uint32_t)sm.uniq[r];
      uint64_t pk = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        uint32_t sa;
        if (a + 1 < D) {
          const uint32_t qd = magic_div(rest, rec->mg_m[a], rec->mg_l[a]);
          sa = rest - qd * rec->N[a];
          rest = qd;
        } else {
          sa = rest;
        }
        const uint32_t base = (a == 0 ? 0u : a == 1 ? l1 : l2) + (sa << rec->b[a]);
        pk |= (uint64_t)(base & 0xffffu) << (16 * a);
      }
      sm.uniq[r] = pk;
    }
    __syncthreads();
    uint32_t shifts[D], masks[D];
    {
      uint32_t sft = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        shifts[a] = sft;
        masks[a] = (1u << rec->b[a]) - 1u;
        sft += rec->b[a];
      }
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const uint64_t pk = sm.uniq[run[k]];
#pragma unroll
      for (int a = 0; a < D; ++a)
        vals[a][k] = tab[((uint32_t)(pk >> (16 * a)) & 0xffffu) + ((off[k] >> shifts[a]) & masks[a])];
    }
  } else {
  double lo[D], w[D];
  uint32_t bsh[D], shifts[D], Nn[D], mgm[D], mgl[D], omask[D];
  {
    uint32_t s = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      lo[a] = rec->lo[a];
      w[a] = rec->w[a];
      bsh[a] = rec->b[a];
      omask[a] = bsh[a] >= 32 ? 0xffffffffu : (1u << bsh[a]) - 1u;
      shifts[a] = s;
      s += bsh[a];
      Nn[a] = rec->N[a];
      mgm[a] = rec->mg_m[a];
      mgl[a] = rec->mg_l[a];
    }
  }
  if (rec->fast_body == 3) {
    // every bin index < 2^31 (K4a): 32-bit q and the 2^51 magic constant from one word
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      uint32_t rest = (uint32_t)sm.uniq[run[k]];
#pragma unroll
      for (int a = 0; a < D; ++a) {
        uint32_t sa;
        if (a + 1 < D) {
          const uint32_t qd = magic_div(rest, mgm[a], mgl[a]);
          sa = rest - qd * Nn[a];
          rest = qd;
        } else {
          sa = rest;
        }
        const uint32_t q = (sa << bsh[a]) | ((off[k] >> shifts[a]) & omask[a]);
        const double h = __hiloint2double(0x43200000, (int)(2u * q + 1u));
        const double aq = __dsub_rn(h, 2251799813685248.0);
        vals[a][k] = (T)__dadd_rn(lo[a], __dmul_rn(aq, w[a]));
      }
    }
  } else {
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    uint32_t rest = (uint32_t)sm.uniq[run[k]];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      uint32_t sa;
      if (a + 1 < D) {
        const uint32_t qd = magic_div(rest, mgm[a], mgl[a]);
        sa = rest - qd * Nn[a];
        rest = qd;
      } else {
        sa = rest;
      }
      const uint32_t oa = bsh[a] ? (off[k] >> shifts[a]) & ((1u << bsh[a]) - 1u) : 0u;
      const uint64_t q = ((uint64_t)sa << bsh[a]) | oa;
      // RN(q + 0.5) exactly: 2^51 + q + 0.5 has ulp 0.5 (q < 2^51)
      const double h = __longlong_as_double((long long)(0x4320000000000000ull + 2 * q + 1));
      const double aq = __dsub_rn(h, 2251799813685248.0);
      vals[a][k] = (T)__dadd_rn(lo[a], __dmul_rn(aq, w[a]));
    }
  }
  }
  }
  const uint64_t idx0 = (P.out_offsets ? P.out_offsets[blk] : blk * (uint64_t)P.bs) + p0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    T* out = reinterpret_cast<T*>(P.out[a]);
    if (idx0 + kItems <= P.out_cap && ((reinterpret_cast<uintptr_t>(out + idx0) & 15) == 0)) {
      if constexpr (sizeof(T) == 4) {
        __stcs(reinterpret_cast<float4*>(out + idx0), make_float4(vals[a][0], vals[a][1], vals[a][2], vals[a][3]));
      } else {
        __stcs(reinterpret_cast<double2*>(out + idx0), make_double2(vals[a][0], vals[a][1]));
        __stcs(reinterpret_cast<double2*>(out + idx0) + 1, make_double2(vals[a][2], vals[a][3]));
      }
    } else {
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (idx0 + k < P.out_cap) out[idx0 + k] = vals[a][k];
    }
  }
}

// General decode body: any widths, 64-bit ids, rank stream, partial blocks.
template <int D, bool F64, bool PRES>
__device__ __forceinline__ void decode_general(const DecParams& P, DecSmem& sm, const uint64_t blk,
                                               const DecRec* rec) {
  using T = typename std::conditional<F64, double, float>::type;
  const int tid = threadIdx.x;
  DevResult* R = P.res;
  const int n = (int)rec->n;
  const uint32_t U = rec->U;
  const uint32_t wd = rec->wd, wc = rec->wc, wo = rec->wo, wr = PRES ? rec->wr : 0u;
  const uint32_t sd = rec->sd, sc = rec->sc, so = rec->so, sr = rec->sr;
  const uint8_t* pay = P.c + P.table_end + rec->e0;
  const uint32_t al = (uint32_t)((uintptr_t)pay & 15);
  // payload length = end of the last stream (validated by K4a)
  const uint32_t plen = PRES ? sr + (uint32_t)(((uint64_t)n * wr + 7) >> 3)
                             : so + (uint32_t)(((uint64_t)n * wo + 7) >> 3);

  // ---- 1. payload window -> shared memory (16B chunks; edges bytewise)
  if (PRES && tid < kMaxBs / 32) sm.seen[tid] = 0;
  {
    const uint8_t* g16 = pay - al;
    const uint8_t* cend = P.c + P.len;
    const uint32_t nch = (al + plen + 15) >> 4;
    for (uint32_t ch = tid; ch < nch; ch += kThreads) {
      const uint8_t* src = g16 + 16 * ch;
      uint4 v;
      if (src >= P.c && src + 16 <= cend) {
        v = __ldcs(reinterpret_cast<const uint4*>(src));
      } else {
        uint32_t w[4] = {0, 0, 0, 0};
        for (int j = 0; j < 16; ++j)
          if (src + j >= P.c && src + j < cend) w[j >> 2] |= (uint32_t)src[j] << (8 * (j & 3));
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
      reinterpret_cast<uint4*>(sm.words)[ch] = v;
    }
  }
  __syncthreads();
  const uint8_t* pb = reinterpret_cast<const uint8_t*>(sm.words) + al;  // payload byte 0
  const uint64_t pbit = 8ull * al;
  const int p0 = tid * kItems;
  uint32_t fl = 0;  // check bits in the reference's order (see the reason table below)

  // ---- 2. unpack (codec.unpack_fixed): padding, deltas + counts, offsets, ranks
  if (tid < (PRES ? 4 : 3)) {
    const uint32_t s = tid;
    const uint64_t cnt = s < 2 ? U : (uint64_t)n;
    const uint32_t w = s == 0 ? wd : s == 1 ? wc : s == 2 ? wo : wr;
    const uint32_t st = s == 0 ? sd : s == 1 ? sc : s == 2 ? so : sr;
    const uint64_t used = cnt * w, nb = (used + 7) >> 3;
    if (w && cnt && (used & 7) && (pb[st + nb - 1] >> (used & 7))) fl |= (s == 3) ? (1u << 15) : (1u << s);
  }
  unsigned long long dsum = 0, csum = 0;
  uint64_t dl[kItems], cn[kItems];
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t r = p0 + j;
    dl[j] = cn[j] = 0;
    if (r < U) {
      dl[j] = get_bits(sm.words, pbit + 8ull * sd + (uint64_t)r * wd, wd);
      cn[j] = get_bits(sm.words, pbit + 8ull * sc + (uint64_t)r * wc, wc);
    }
    dsum += dl[j];
    csum += cn[j];
  }
  uint64_t off[kItems];
  uint32_t rk[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    off[k] = (p0 + k < n) ? get_bits(sm.words, pbit + 8ull * so + (uint64_t)(p0 + k) * wo, wo) : 0ull;
    rk[k] = (PRES && p0 + k < n) ? (uint32_t)get_bits(sm.words, pbit + 8ull * sr + (uint64_t)(p0 + k) * wr, wr)
                                 : 0u;
  }

  // ---- 3. delta decode (wrapping cumsum) + run starts, with the decoder checks
  unsigned long long dtot, ctot;
  block_excl_scan2(dsum, csum, dtot, ctot, sm.scan);
  {
    uint64_t prev = dsum;
    unsigned long long cex = csum;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t r = p0 + j;
      if (r < U) {
        const uint64_t u = prev + dl[j];
        if (r > 0 && u <= prev) fl |= 1u << 3;           // pipeline.py:116-117
        if (cn[j] < 1) fl |= 1u << 4;                     // pipeline.py:118-119
        if (cn[j] >= (1ull << 63)) fl |= 1u << 6;         // codec.py:88-89
        if (!rec->pn_all && u >= rec->PN) fl |= 1u << 13;  // quantizer.py:262-263
        sm.uniq[r] = u;
        sm.starts[r] = (uint32_t)cex;
        cex += cn[j];
        prev = u;
      }
    }
  }
  if (ctot != (unsigned long long)n) fl |= 1u << 5;       // pipeline.py:120-123
  fl |= (uint32_t)rec->geo_bits << 7;                      // pipeline.py:128-138
  {
    const uint32_t sb = rec->sumb;
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (p0 + k < n && sb < 64 && (off[k] >> sb)) fl |= 1u << 14;  // quantizer.py:264-265
  }
  if (PRES) {  // the rank stream must be a permutation (pipeline.py:149-154)
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (p0 + k < n) {
        if (rk[k] >= (uint32_t)n) fl |= 1u << 16;
        else if (atomicOr(&sm.seen[rk[k] >> 5], 1u << (rk[k] & 31)) & (1u << (rk[k] & 31))) fl |= 1u << 16;
      }
  }
  if (__syncthreads_or(fl != 0)) {
    uint32_t v[1] = {fl};
    block_or<1>(v, sm.red);
    if (tid == 0) {
      const int bit = __ffs((int)v[0]) - 1;
      int reason, ax = 0;
      switch (bit) {
        case 0: reason = R_BLK_PAD_DELTA; break;
        case 1: reason = R_BLK_PAD_COUNT; break;
        case 2: reason = R_BLK_PAD_OFF; break;
        case 3: reason = R_BLK_IDS; break;
        case 4: reason = R_BLK_ZERO_RUN; break;
        case 5: reason = R_BLK_RUN_SUM; break;
        case 6: reason = R_BLK_RUN_MAX; break;
        case 13: reason = R_BLK_SEG_RANGE; break;
        case 14: reason = R_BLK_OFF_RANGE; break;
        case 15: reason = R_BLK_PAD_RANK; break;
        case 16: reason = R_BLK_RANKS; break;
        default: ax = (bit - 7) >> 1; reason = ((bit - 7) & 1) ? R_BLK_SEGCOUNT : R_BLK_AXIS_RANGE; break;
      }
      atomicMax(&R->err_block, err_code(blk, ax, reason));
    }
    return;
  }

  // ---- 4. run expansion + delinearize + midpoint reconstruction
  uint32_t r;
  {
    uint32_t lo_i = 0, hi_i = U ? U - 1 : 0;
    const uint32_t p = (uint32_t)p0;
    while (lo_i < hi_i) {  // last run whose start <= p
      const uint32_t mid = (lo_i + hi_i + 1) >> 1;
      if (sm.starts[mid] <= p) lo_i = mid; else hi_i = mid - 1;
    }
    r = lo_i;
  }
  const uint64_t obase = P.out_offsets ? P.out_offsets[blk] : blk * (uint64_t)P.bs;
  const bool big = rec->pn_big;
  const uint32_t fast = rec->fast_mask, chk = rec->chk_mask;
  double lo[D], w[D];
  uint32_t bsh[D], shifts[D], Nn[D], mgm[D], mgl[D];
  {
    uint32_t s = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      lo[a] = rec->lo[a];
      w[a] = rec->w[a];
      bsh[a] = rec->b[a];
      shifts[a] = s;
      s += bsh[a];
      Nn[a] = rec->N[a];
      mgm[a] = rec->mg_m[a];
      mgl[a] = rec->mg_l[a];
    }
  }
  T vals[D][kItems];
  uint32_t nf = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    const int p = p0 + k;
    if (p >= n) {
#pragma unroll
      for (int a = 0; a < D; ++a) vals[a][k] = T(0);
      continue;
    }
    while (r + 1 < U && sm.starts[r + 1] <= (uint32_t)p) ++r;
    uint64_t rest = sm.uniq[r];
#pragma unroll
    for (int a = 0; a < D; ++a) {
      uint64_t sa;
      if (a + 1 < D) {
        if (!big) {
          const uint32_t qd = magic_div((uint32_t)rest, mgm[a], mgl[a]);
          sa = (uint32_t)rest - qd * Nn[a];
          rest = qd;
        } else {
          sa = rest % Nn[a];
          rest /= Nn[a];
        }
      } else {
        sa = rest;
      }
      const uint64_t oa = shr64(off[k], shifts[a]) & mask64(bsh[a]);
      const uint64_t q = shl64(sa, bsh[a]) | oa;
      double v;
      if (fast & (1u << a)) {
        // RN(q + 0.5) exactly: 2^51 + q + 0.5 has ulp 0.5 (q < 2^51)
        const double h = __longlong_as_double((long long)(0x4320000000000000ull + 2 * q + 1));
        const double aq = __dsub_rn(h, 2251799813685248.0);
        v = __dadd_rn(lo[a], __dmul_rn(aq, w[a]));
      } else {
        const double aq = __dadd_rn(__ull2double_rn(q), 0.5);
        v = __dadd_rn(lo[a], __dmul_rn(aq, w[a]));
      }
      const T tv = (T)v;  // RN to the output precision (quantizer.py:271)
      if ((chk & (1u << a)) && !isfinite((double)tv)) nf |= 1u << a;
      vals[a][k] = tv;
    }
  }
  if (nf) atomicOr(&R->nonfinite_mask, nf);

  // ---- 5. store: sorted order, or scattered by the rank stream
#pragma unroll
  for (int a = 0; a < D; ++a) {
    T* out = reinterpret_cast<T*>(P.out[a]);
    if (PRES) {
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        const uint64_t idx = obase + rk[k];
        if (p0 + k < n && idx < P.out_cap) out[idx] = vals[a][k];
      }
    } else {
      const uint64_t idx0 = obase + p0;
      const bool full = p0 + kItems <= n && idx0 + kItems <= P.out_cap &&
                        ((reinterpret_cast<uintptr_t>(out + idx0) & 15) == 0);
      if (full) {
        if constexpr (sizeof(T) == 4) {
          __stcs(reinterpret_cast<float4*>(out + idx0), make_float4(vals[a][0], vals[a][1], vals[a][2], vals[a][3]));
        } else {
          __stcs(reinterpret_cast<double2*>(out + idx0), make_double2(vals[a][0], vals[a][1]));
          __stcs(reinterpret_cast<double2*>(out + idx0) + 1, make_double2(vals[a][2], vals[a][3]));
        }
      } else {
#pragma unroll
        for (int k = 0; k < kItems; ++k)
          if (p0 + k < n && idx0 + k < P.out_cap) out[idx0 + k] = vals[a][k];
      }
    }
  }
}

// Particle count of each block (iter_decompressed_blocks output offsets).
__global__ void k_block_counts(const uint8_t* c, uint64_t len, uint64_t table_end, uint64_t payload_len,
                               uint64_t nblocks, uint32_t bs, uint64_t* counts) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nblocks) return;
  const uint8_t* table = c + GPZB_GLOBAL_HEADER_SIZE;
  const uint64_t e0 = ld_le(table + 8 * i, 8), e1 = ld_le(table + 8 * i + 8, 8);
  uint64_t n = 0;
  if (e0 + 4 <= e1 && e1 <= payload_len) n = ld_le(c + table_end + e0, 4);
  counts[i] = min(n, (uint64_t)max(bs, (uint32_t)kMaxBs));
}

}  // namespace gpzb
