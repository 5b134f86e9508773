// K4: fused block decoder for the GPZ B200 decompressor.
//
// One CTA per block restates pipeline._decode_block (pipeline.py:106-157):
// offset-table checks (container.py:282-290), parse_block (container.py:128-200),
// unpack_fixed (codec.py:132-151), delta/RLE decode (codec.py:82-104) with the
// decoder's consistency checks (pipeline.py:116-145), _delinearize +
// dequantize_block (quantizer.py:194-272) and the rank scatter
// (pipeline.py:149-156).  The first failing check of the lowest failing block
// is reported, matching the reference's serial first-error order.
#pragma once

#include <type_traits>

#include "gpzb_common.cuh"

namespace gpzb {

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
};

constexpr int kDecStageWords = 6144;  // 24 KB payload window

struct DecSmem {
  uint64_t e0;             // payload start within the payload region
  uint64_t L;              // payload length
  uint32_t n, U, err, sh;
  uint32_t b[3];
  uint32_t wd, wc, wo, wr;
  uint32_t sumb;
  uint64_t N[3];
  uint64_t PN;             // Π N (saturated at 2^64-1 when larger)
  int pn_big;              // Π N > 2^32
  uint32_t sd, sc, so, sr; // stream byte offsets within the payload
  double lo[3], w[3];
  uint32_t mg_m[3], mg_l[3];
  int fast[3];
  uint32_t flags;
  uint32_t red[kWarps * 2];
  unsigned long long scan64[kWarps];
  uint32_t seen[kMaxBs / 32];
  __align__(16) uint32_t words[kDecStageWords];
  __align__(16) uint64_t uniq[kMaxBs];
  __align__(16) uint32_t starts[kMaxBs];
};

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

template <int D, bool F64, bool PRES>
__global__ void __launch_bounds__(kThreads) k_decode(const DecParams P) {
  using T = typename std::conditional<F64, double, float>::type;
  constexpr int S = F64 ? 8 : 4;
  constexpr uint32_t HS = 8 + D * (2 * S + 5) + (PRES ? 4 : 3);
  __shared__ DecSmem sm;
  const int tid = threadIdx.x;
  const uint64_t blk = blockIdx.x;
  DevResult* R = P.res;
  const uint8_t* table = P.c + GPZB_GLOBAL_HEADER_SIZE;

  // ---- 1. offset-table entries and the payload window
  if (tid == 0) {
    const uint64_t e0 = ld_le(table + 8 * blk, 8);
    const uint64_t e1 = ld_le(table + 8 * blk + 8, 8);
    uint32_t tf = 0;
    if (blk == 0 && e0 != 0) tf |= 1;
    if (e0 > e1) tf |= 2;
    if (blk + 1 == P.nblocks && e1 != P.payload_len) tf |= 4;
    if (tf) atomicOr(&R->table_flags, tf);
    const bool ok = !tf && e1 <= P.payload_len;
    sm.err = ok ? 0u : 0xffffffffu;  // table problems are reported container-wide
    sm.L = ok ? (e1 - e0) : 0;
    sm.e0 = e0;
  }
  __syncthreads();
  if (sm.err) return;
  const uint64_t L = sm.L;
  const uint8_t* pay = P.c + P.table_end + sm.e0;
  const uint32_t al = (uint32_t)((uintptr_t)pay & 15);
  const uint64_t avail = min(L, (uint64_t)(kDecStageWords * 4 - 16));
  {
    const uint8_t* g16 = pay - al;
    const uint8_t* cend = P.c + P.len;
    const uint32_t nch = (uint32_t)((al + avail + 15) >> 4);
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

  // ---- 2. parse_block header checks (container.py:128-193), serial order
  if (tid == 0) {
    uint32_t e = 0, eax = 0;
    uint32_t n = 0, U = 0;
    if (L < HS) {
      e = R_BLK_SHORT;
    } else {
      n = (uint32_t)ld_le(pb, 4);
      U = (uint32_t)ld_le(pb + 4, 4);
      const uint8_t* wp = pb + 8 + D * (2 * S + 5);
      sm.wd = wp[0]; sm.wc = wp[1]; sm.wo = wp[2]; sm.wr = PRES ? wp[3] : 0;
      if (U > n) e = R_BLK_UNIQUE;
      if (!e && (sm.wd > 64 || sm.wc > 64 || sm.wo > 64 || sm.wr > 64)) e = R_BLK_WIDTH;
      for (int a = 0; a < D && !e; ++a) {
        const uint8_t* ap = pb + 8 + a * (2 * S + 5);
        double lo, hi;
        if (F64) {
          lo = __longlong_as_double((long long)ld_le(ap, 8));
          hi = __longlong_as_double((long long)ld_le(ap + 8, 8));
        } else {
          lo = (double)__uint_as_float((uint32_t)ld_le(ap, 4));
          hi = (double)__uint_as_float((uint32_t)ld_le(ap + 4, 4));
        }
        const uint32_t b = ap[2 * S];
        const uint64_t N = ld_le(ap + 2 * S + 1, 4);
        sm.lo[a] = lo;
        sm.w[a] = hi;  // hi stashed in w until the geometry step
        sm.b[a] = b;
        sm.N[a] = N;
        if (N < 1 && n > 0) { e = R_BLK_NOSEG; eax = a; }
        else if (b > 63) { e = R_BLK_OFFBITS; eax = a; }
        else if (!(isfinite(lo) && isfinite(hi) && lo <= hi)) { e = R_BLK_BOUNDS; eax = a; }
      }
      if (!e) {
        uint64_t cur = HS;
        const uint64_t cnts[4] = {U, U, n, n};
        const uint32_t ws[4] = {sm.wd, sm.wc, sm.wo, sm.wr};
        uint32_t so[4];
        for (int s = 0; s < (PRES ? 4 : 3) && !e; ++s) {
          const uint64_t nb = (cnts[s] * ws[s] + 7) >> 3;
          so[s] = (uint32_t)cur;
          if (cur + nb > L) e = R_BLK_TRUNC;
          cur += nb;
        }
        if (!e && cur != L) e = R_BLK_TRAILING;
        if (!e) { sm.sd = so[0]; sm.sc = so[1]; sm.so = so[2]; sm.sr = PRES ? so[3] : 0; }
      }
      if (!e && L > avail) e = R_BLK_WINDOW;  // only with oversized stream widths
      if (!e && n > (uint32_t)kMaxBs) {
        // a block the 1024-particle kernels cannot hold: unsupported when the
        // header's boundary math says it is legitimately that large
        const __int128 want = (blk + 1 < P.nblocks) ? (__int128)P.bs
                              : (__int128)P.count - (__int128)P.bs * (__int128)(P.nblocks - 1);
        e = ((__int128)n == want) ? R_UNSUPPORTED_BS : R_BLK_TOO_BIG;
      }
    }
    if (e) atomicMax(&R->err_block, err_code(blk, eax, e));
    sm.err = e;
    sm.n = n;
    sm.U = U;
    sm.flags = 0;
  }
  if (tid < kMaxBs / 32) sm.seen[tid] = 0;
  __syncthreads();
  if (sm.err) return;
  const int n = (int)sm.n;
  const uint32_t U = sm.U;
  const int p0 = tid * kItems;
  const uint32_t wd = sm.wd, wc = sm.wc, wo = sm.wo;
  const uint64_t pbit = 8ull * al;  // bit position of payload byte 0 in words
  uint32_t fl = 0;  // check bits in reference order

  // ---- 3. unpack (codec.unpack_fixed) with padding checks
  if (tid < (PRES ? 4 : 3)) {
    const uint32_t s = tid;
    const uint64_t cnt = s < 2 ? U : (uint64_t)n;
    const uint32_t w = s == 0 ? wd : s == 1 ? wc : s == 2 ? wo : sm.wr;
    const uint32_t so = s == 0 ? sm.sd : s == 1 ? sm.sc : s == 2 ? sm.so : sm.sr;
    const uint64_t used = cnt * w, nb = (used + 7) >> 3;
    if (w && cnt && (used & 7)) {
      const uint8_t last = pb[so + nb - 1];
      if (last >> (used & 7)) fl |= (s == 3) ? (1u << 15) : (1u << s);
    }
  }
  uint64_t dl[kItems], cn[kItems];
  uint64_t dsum = 0, csum = 0;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t r = p0 + j;
    dl[j] = cn[j] = 0;
    if (r < U) {
      dl[j] = get_bits(sm.words, pbit + 8ull * sm.sd + (uint64_t)r * wd, wd);
      cn[j] = get_bits(sm.words, pbit + 8ull * sm.sc + (uint64_t)r * wc, wc);
    }
    dsum += dl[j];
    csum += cn[j];
  }
  uint64_t off[kItems];
  uint32_t rk[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    off[k] = (p0 + k < n) ? get_bits(sm.words, pbit + 8ull * sm.so + (uint64_t)(p0 + k) * wo, wo) : 0ull;
    rk[k] = (PRES && p0 + k < n) ? (uint32_t)get_bits(sm.words, pbit + 8ull * sm.sr + (uint64_t)(p0 + k) * sm.wr, sm.wr) : 0u;
  }

  // ---- 4. delta decode (wrapping cumsum) + run lengths, with the decoder checks
  unsigned long long dtot, ctot;
  unsigned long long dex = block_excl_scan<unsigned long long>(dsum, dtot, sm.scan64);
  unsigned long long cex = block_excl_scan<unsigned long long>(csum, ctot, sm.scan64);
  {
    uint64_t prev = dex;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t r = p0 + j;
      if (r < U) {
        const uint64_t u = prev + dl[j];
        if (r > 0 && u <= prev) fl |= 1u << 3;          // pipeline.py:116-117
        if (cn[j] < 1) fl |= 1u << 4;                    // pipeline.py:118-119
        if (cn[j] >= (1ull << 63)) fl |= 1u << 6;        // codec.py:88-89
        sm.uniq[r] = u;
        sm.starts[r] = (uint32_t)cex;
        cex += cn[j];
        prev = u;
      }
    }
  }
  if (ctot != (unsigned long long)n) fl |= 1u << 5;       // pipeline.py:120-123

  // ---- 5. geometry re-derived from the stored bounds (pipeline.py:128-145)
  if (tid < D) {
    const int a = tid;
    const double lo = sm.lo[a], hi = sm.w[a];
    bool half;
    const double eb_int = inner_bound(P.eb_abs, lo, hi, F64, half);
    const double w = __dmul_rn(2.0, eb_int);
    const double span = __dsub_rn(hi, lo);
    uint64_t Q = 1;
    bool ovf = false;
    if (span > 0.0) {
      const double ratio = __ddiv_rn(span, w);
      if (!(ratio < 18446744073709551616.0)) ovf = true;
      else Q = (uint64_t)__double2ull_rz(ratio) + 1;
    }
    if (ovf) fl |= 1u << (7 + 2 * a);
    else if (n > 0) {
      const uint32_t b = sm.b[a];
      const uint64_t m = 1ull << b;
      const uint64_t need = Q / m + (Q % m ? 1 : 0);
      if (need != sm.N[a]) fl |= 1u << (8 + 2 * a);
    }
    const uint32_t Na = (uint32_t)(sm.N[a] > 0xffffffffull ? 0xffffffffull : sm.N[a]);
    uint32_t l = 0, mg = 0;
    if (Na > 1) {
      l = 32 - __clz((int)(Na - 1));
      mg = (uint32_t)((((uint64_t)1 << 32) * (((uint64_t)1 << l) - Na)) / Na + 1);
    }
    sm.mg_m[a] = mg;
    sm.mg_l[a] = l;
    sm.lo[a] = lo;
    sm.w[a] = w;
    // q = seg_a * m + off_a < N * m; the magic-constant midpoint needs q < 2^51
    sm.fast[a] = (sm.b[a] < 51) && (sm.N[a] <= ((1ull << 51) >> sm.b[a]));
  }
  if (tid == 0) {
    unsigned __int128 pn = 1;
    uint32_t sb = 0;
    for (int a = 0; a < D; ++a) {
      pn *= sm.N[a];
      if (pn > ((unsigned __int128)1 << 64)) pn = ((unsigned __int128)1 << 64) + 1;
      sb += sm.b[a];
    }
    sm.PN = pn > 0xffffffffffffffffull ? 0xffffffffffffffffull : (uint64_t)pn;
    sm.pn_big = pn > 0xffffffffull;
    sm.sumb = sb;
    // PN saturated: a true product >= 2^64 admits every u64 id
    sm.flags = (pn >= ((unsigned __int128)1 << 64)) ? 1u : 0u;
  }
  __syncthreads();
  {
    const bool pn_all = sm.flags & 1u;
    const uint64_t PN = sm.PN;
    const uint32_t sb = sm.sumb;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t r = p0 + j;
      if (r < U && !pn_all && sm.uniq[r] >= PN) fl |= 1u << 13;  // quantizer.py:262-263
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (p0 + k < n && sb < 64 && (off[k] >> sb)) fl |= 1u << 14;  // quantizer.py:264-265
  }
  // ---- 6. rank stream must be a permutation (pipeline.py:149-154)
  if (PRES) {
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (p0 + k < n) {
        if (rk[k] >= (uint32_t)n) fl |= 1u << 16;
        else if (atomicOr(&sm.seen[rk[k] >> 5], 1u << (rk[k] & 31)) & (1u << (rk[k] & 31))) fl |= 1u << 16;
      }
  }
  {
    uint32_t v[1] = {fl};
    block_or<1>(v, sm.red);
    fl = v[0];
  }
  if (fl) {
    if (tid == 0) {
      const int bit = __ffs((int)fl) - 1;
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

  // ---- 7. per-block particle count vs the boundary math (pipeline.py:174-181)
  if (tid == 0) {
    const __int128 want = (blk + 1 < P.nblocks)
                              ? (__int128)P.bs
                              : (__int128)P.count - (__int128)P.bs * (__int128)(P.nblocks - 1);
    if ((__int128)n != want) atomicMax(&R->err_count, err_code(blk, 0, R_BLK_COUNT));
  }

  // ---- 8. run expansion + delinearize + midpoint reconstruction
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
  T vals[D][kItems];
  uint32_t nf = 0;
  uint32_t shifts[D];
  {
    uint32_t s = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) { shifts[a] = s; s += sm.b[a]; }
  }
  const bool big = sm.pn_big;
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
          const uint32_t qd = magic_div((uint32_t)rest, sm.mg_m[a], sm.mg_l[a]);
          sa = (uint32_t)rest - qd * (uint32_t)sm.N[a];
          rest = qd;
        } else {
          sa = rest % sm.N[a];
          rest /= sm.N[a];
        }
      } else {
        sa = rest;
      }
      const uint32_t b = sm.b[a];
      const uint64_t oa = (off[k] >> shifts[a]) & mask64(b);
      const uint64_t q = shl64(sa, b) | oa;
      double v;
      if (sm.fast[a]) {
        // RN(q + 0.5) exactly: 2^51 + q + 0.5 has ulp 0.5 (q < 2^51)
        const double h = __longlong_as_double((long long)(0x4320000000000000ull + 2 * q + 1));
        const double aq = __dsub_rn(h, 2251799813685248.0);
        v = __dadd_rn(sm.lo[a], __dmul_rn(aq, sm.w[a]));
      } else {
        const double aq = __dadd_rn(__ull2double_rn(q), 0.5);
        v = __dadd_rn(sm.lo[a], __dmul_rn(aq, sm.w[a]));
      }
      T tv = (T)v;  // RN to the output precision (quantizer.py:271)
      if (!isfinite((double)tv)) nf |= 1u << a;
      vals[a][k] = tv;
    }
  }
  if (nf) atomicOr(&R->nonfinite_mask, nf);

  // ---- 9. store: sorted order, or scattered by the rank stream
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
                               uint64_t nblocks, uint64_t* counts) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= nblocks) return;
  const uint8_t* table = c + GPZB_GLOBAL_HEADER_SIZE;
  const uint64_t e0 = ld_le(table + 8 * i, 8), e1 = ld_le(table + 8 * i + 8, 8);
  uint64_t n = 0;
  if (e0 + 4 <= e1 && e1 <= payload_len) n = ld_le(c + table_end + e0, 4);
  counts[i] = min(n, (uint64_t)kMaxBs);
}

}  // namespace gpzb
