// K2b / K4b: blocks of more than 1024 particles.
//
// CompressConfig accepts any positive multiple of 32 as block_size
// (model.py:118-119).  Every other encoder and decoder holds a whole block in
// one CTA's registers and shared memory (<= 1024 particles); a larger block
// keeps its state in a per-CTA slice of the workspace instead, and one CTA of
// 256 threads walks it in chunks.  This is the correctness path for those
// configurations (the benchmarked ones use 1024): same bytes and the same
// errors as pipeline._encode_block / _decode_block (pipeline.py:38-70,
// 106-157), not tuned for speed.
//
// K2b per block (K1.5 puts every block of such a call on the general list,
// with a side-buffer slot sized by payload_bound):
//   quantize each particle (quantize_coord: every quantizer mode of
//   quantizer.py:142-191) and linearise -> (seg, off, index) in the slice,
//   padded to a power of two with all-ones keys; a bitonic sort on the triple
//   (the index breaks ties, so the order is np.lexsort's stable one,
//   blocksort.py:17-28); run starts by a chunked block scan (rle_encode,
//   codec.py:53-79); stream widths by OR (codec.py:107-112); the header and
//   streams OR-ed bit by bit into the zeroed slot with 64-bit atomics
//   (serialize_block / pack_fixed, container.py:98-121, codec.py:115-129).
// K4b per block (K4a lists them all): the streams read straight from the
//   container, the decoder's checks in _decode_block's order as the same
//   ordered bits as decode_general, run ids and starts in the slice, then
//   every particle's run by binary search, delinearisation and the midpoint
//   (quantizer.py:194-272), stored in order or through the rank stream.
#pragma once

#include "gpzb_decode.cuh"
#include "gpzb_encode.cuh"

namespace gpzb {

// Workspace slice per CTA: encoder (seg u64, off u64, index u32) per padded
// particle + (run id u64, run start u32) per particle; decoder (run id u64,
// run start u32) per particle + the rank bitmap.
__host__ __device__ inline uint64_t big_pad(uint32_t bs) {
  uint64_t p = 1;
  while (p < bs) p <<= 1;
  return p;
}
__host__ __device__ inline uint64_t big_enc_slice(uint32_t bs) { return 32ull * big_pad(bs); }
__host__ __device__ inline uint64_t big_dec_slice(uint32_t bs) { return (12ull * bs + bs / 8 + 64 + 255) & ~255ull; }

__device__ __forceinline__ bool big_less(uint64_t s1, uint64_t o1, uint32_t i1, uint64_t s2, uint64_t o2,
                                         uint32_t i2) {
  return s1 < s2 || (s1 == s2 && (o1 < o2 || (o1 == o2 && i1 < i2)));
}

// OR the low `nbits` (<= 64) bits of v at bit `pos` of a zeroed u64 array.
__device__ __forceinline__ void or_bits_global(unsigned long long* w, uint64_t pos, uint64_t v, uint32_t nbits) {
  if (nbits == 0 || v == 0) return;
  const uint32_t sh = (uint32_t)(pos & 63);
  atomicOr(w + (pos >> 6), (unsigned long long)(v << sh));
  if (sh && sh + nbits > 64) atomicOr(w + (pos >> 6) + 1, (unsigned long long)(v >> (64 - sh)));
}

// `nbits` (<= 64) bits at bit `pos` of a byte array (little-endian, LSB first).
__device__ __forceinline__ uint64_t get_bits_bytes(const uint8_t* p, uint64_t pos, uint32_t nbits) {
  if (nbits == 0) return 0;
  const uint8_t* b = p + (pos >> 3);
  const uint32_t sh = (uint32_t)(pos & 7), nby = (sh + nbits + 7) >> 3;
  uint64_t lo = 0, hi = 0;
  for (uint32_t i = 0; i < nby && i < 8; ++i) lo |= (uint64_t)b[i] << (8 * i);
  if (nby > 8) hi = b[8];
  const uint64_t v = (lo >> sh) | (sh ? hi << (64 - sh) : 0ull);
  return v & mask64(nbits);
}

template <int D, bool F64, bool PRES>
__global__ void __launch_bounds__(kThreads) k_encode_big(const EncParams P, uint8_t* scratch) {
  using T = typename std::conditional<F64, double, float>::type;
  constexpr int S = F64 ? 8 : 4;
  constexpr int H = 8 + D * (2 * S + 5) + (PRES ? 4 : 3);  // block header bytes (container.py:62-67)
  __shared__ AxisGeo geo[3];
  __shared__ int ax_err[3];
  __shared__ uint32_t scan32[kWarps];
  __shared__ uint32_t red[kWarps * 8];
  const int tid = threadIdx.x;
  DevResult* R = P.res;
  const uint64_t npad = big_pad(P.bs);
  uint8_t* base = scratch + blockIdx.x * big_enc_slice(P.bs);
  uint64_t* seg = reinterpret_cast<uint64_t*>(base);
  uint64_t* off = seg + npad;
  uint64_t* uniq = off + npad;
  uint32_t* idx = reinterpret_cast<uint32_t*>(uniq + npad);
  uint32_t* start = idx + npad;
  const uint32_t nlist = R->wide_count;
  for (uint32_t item = blockIdx.x; item < nlist; item += gridDim.x) {
    __syncthreads();  // the slice and shared state are reused across blocks
    const uint64_t blk = P.wide_list[item];
    const uint64_t first = blk * (uint64_t)P.bs;
    const uint32_t n = (uint32_t)min((uint64_t)P.bs, P.count - first);
    const double eb_abs = R->eb_abs;
    if (tid < D) {
      const T* b = reinterpret_cast<const T*>(P.bounds) + blk * 2 * D;
      ax_err[tid] = axis_geometry((double)b[2 * tid], (double)b[2 * tid + 1], eb_abs, F64, P.target, geo[tid]);
    }
    __syncthreads();
    bool bad = !(eb_abs > 0.0);
    uint64_t stride[D];
    uint32_t shift[D];
    {
      unsigned __int128 pn = 1;
      uint32_t sb = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        bad = bad || ax_err[a] != 0;
        stride[a] = (uint64_t)pn;
        shift[a] = sb;
        pn *= geo[a].N;
        bad = bad || pn > ((unsigned __int128)1 << 64);
        sb += geo[a].b;
      }
      bad = bad || sb > 64;
    }
    if (bad) continue;  // cannot happen: K1.5 reported the block and routed it away

    // ---- quantize + linearise (quantizer.py:142-191, 176-191), padded keys
    for (uint64_t i = tid; i < npad; i += kThreads) {
      uint64_t s = ~0ull, o = ~0ull;
      uint32_t ix = ~0u;
      if (i < n) {
        s = 0;
        o = 0;
        ix = (uint32_t)i;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const T x = reinterpret_cast<const T*>(P.axes[a])[first + i];
          const AxisGeo g = geo[a];
          const uint64_t q = quantize_coord((double)x, g, eb_abs, F64);
          s += shr64(q, g.b) * stride[a];
          o |= shl64(q & mask64(g.b), shift[a]);
        }
      }
      seg[i] = s;
      off[i] = o;
      idx[i] = ix;
    }
    __syncthreads();
    // ---- bitonic sort on (seg, off, index)
    for (uint64_t k = 2; k <= npad; k <<= 1) {
      for (uint64_t j = k >> 1; j > 0; j >>= 1) {
        for (uint64_t i = tid; i < npad; i += kThreads) {
          const uint64_t l = i ^ j;
          if (l > i) {
            const uint64_t s1 = seg[i], o1 = off[i], s2 = seg[l], o2 = off[l];
            const uint32_t i1 = idx[i], i2 = idx[l];
            const bool asc = (i & k) == 0;
            if (asc ? big_less(s2, o2, i2, s1, o1, i1) : big_less(s1, o1, i1, s2, o2, i2)) {
              seg[i] = s2; off[i] = o2; idx[i] = i2;
              seg[l] = s1; off[l] = o1; idx[l] = i1;
            }
          }
        }
        __syncthreads();
      }
    }
    // ---- runs: unique ids and starts (rle_encode), offset OR
    uint32_t U = 0;
    uint64_t off_or = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += kThreads) {
      const uint32_t i = c0 + tid;
      const uint32_t flag = i < n && (i == 0 || seg[i] != seg[i - 1]);
      if (i < n) off_or |= off[i];
      uint32_t tot;
      const uint32_t r = U + block_excl_scan<uint32_t>(flag, tot, scan32);
      if (flag) {
        uniq[r] = seg[i];
        start[r] = i;
      }
      U += tot;
    }
    __syncthreads();
    uint64_t del_or = 0;
    uint32_t cnt_or = 0;
    for (uint32_t r = tid; r < U; r += kThreads) {
      del_or |= uniq[r] - (r ? uniq[r - 1] : 0ull);
      cnt_or |= (r + 1 < U ? start[r + 1] : n) - start[r];
    }
    uint32_t rv[5] = {(uint32_t)off_or, (uint32_t)(off_or >> 32), cnt_or, (uint32_t)del_or, (uint32_t)(del_or >> 32)};
    block_or<5>(rv, red);
    const uint32_t w_off = bitlen64((uint64_t)rv[0] | ((uint64_t)rv[1] << 32));
    const uint32_t w_cnt = bitlen32(rv[2]);
    const uint32_t w_del = bitlen64((uint64_t)rv[3] | ((uint64_t)rv[4] << 32));
    const uint32_t w_rank = PRES ? (uint32_t)bitlen32(n - 1) : 0u;
    const uint64_t Ld = ((uint64_t)U * w_del + 7) >> 3, Lc = ((uint64_t)U * w_cnt + 7) >> 3;
    const uint64_t Lo = ((uint64_t)n * w_off + 7) >> 3, Lr = PRES ? (((uint64_t)n * w_rank + 7) >> 3) : 0;
    const uint64_t L = (uint64_t)H + Ld + Lc + Lo + Lr;
    BlkRec* rec = reinterpret_cast<BlkRec*>(P.rec) + blk;
    if (rec->side_off + ((L + 15) & ~15ull) > P.side_cap) {
      // the caller's side buffer is too small: report the bytes K1.5 reserved
      if (tid == 0) atomicMax(&R->side_need, R->side_bytes);
      continue;
    }
    unsigned long long* dst = reinterpret_cast<unsigned long long*>(P.side + rec->side_off);  // 16B aligned
    for (uint64_t w = tid; w < (L + 7) >> 3; w += kThreads) dst[w] = 0ull;
    __syncthreads();
    // ---- header (container.serialize_block, container.py:107-121) and streams
    if (tid < 2 + 4 * D + (PRES ? 4 : 3)) {
      const int f = tid;
      uint64_t bpos = 0, val = 0;
      uint32_t bits = 8;
      if (f == 0) { bpos = 0; val = n; bits = 32; }
      else if (f == 1) { bpos = 4; val = U; bits = 32; }
      else if (f < 2 + 4 * D) {
        const int a = (f - 2) >> 2, which = (f - 2) & 3;
        const uint64_t ab = 8 + (uint64_t)a * (2 * S + 5);
        const AxisGeo& g = geo[a];
        if (which < 2) {
          const double v = which ? g.hi : g.lo;
          bpos = ab + which * S;
          val = F64 ? (uint64_t)__double_as_longlong(v) : (uint64_t)__float_as_uint((float)v);
          bits = 8 * S;
        } else if (which == 2) { bpos = ab + 2 * S; val = g.b; }
        else { bpos = ab + 2 * S + 1; val = (uint32_t)g.N; bits = 32; }
      } else {
        const int wi = f - 2 - 4 * D;
        bpos = 8 + (uint64_t)D * (2 * S + 5) + wi;
        val = wi == 0 ? w_del : wi == 1 ? w_cnt : wi == 2 ? w_off : w_rank;
      }
      or_bits_global(dst, 8 * bpos, val, bits);
    }
    const uint64_t bd = 8ull * H, bc = bd + 8 * Ld, bo = bc + 8 * Lc, br = bo + 8 * Lo;
    for (uint32_t r = tid; r < U; r += kThreads) {
      or_bits_global(dst, bd + (uint64_t)r * w_del, uniq[r] - (r ? uniq[r - 1] : 0ull), w_del);
      or_bits_global(dst, bc + (uint64_t)r * w_cnt, (r + 1 < U ? start[r + 1] : n) - start[r], w_cnt);
    }
    for (uint32_t p = tid; p < n; p += kThreads) {
      or_bits_global(dst, bo + (uint64_t)p * w_off, off[p], w_off);
      if (PRES) or_bits_global(dst, br + (uint64_t)p * w_rank, idx[p], w_rank);  // quantizer.py:240-241
    }
    __syncthreads();
    if (tid == 0) {
      rec->side_len = (uint32_t)L;
      rec->path = 4;  // diagnostics: the general encoder
      P.status[blk] = L;  // payload length for the K3 scan
    }
  }
}

template <int D, bool F64, bool PRES>
__global__ void __launch_bounds__(kThreads) k_decode_big(const DecParams P, uint8_t* scratch) {
  using T = typename std::conditional<F64, double, float>::type;
  constexpr int S = F64 ? 8 : 4;
  constexpr uint32_t HS = 8 + D * (2 * S + 5) + (PRES ? 4 : 3);
  __shared__ unsigned long long scan[2 * kWarps];
  __shared__ uint32_t red[kWarps * 8];
  const int tid = threadIdx.x;
  DevResult* R = P.res;
  uint8_t* base = scratch + blockIdx.x * big_dec_slice(P.bs);
  uint64_t* uniq = reinterpret_cast<uint64_t*>(base);
  uint32_t* start = reinterpret_cast<uint32_t*>(uniq + P.bs);
  uint32_t* seen = start + P.bs;
  const uint32_t cnt = *reinterpret_cast<volatile const uint32_t*>(&R->wide_count);
  for (uint32_t item = blockIdx.x; item < cnt; item += gridDim.x) {
    __syncthreads();
    const uint64_t blk = P.list[item];
    const DecRec* rec = P.rec + blk;
    const uint32_t n = rec->n, U = rec->U;
    const uint32_t wd = rec->wd, wc = rec->wc, wo = rec->wo, wr = PRES ? rec->wr : 0u;
    // stream offsets (K4a checked them; DecRec keeps only 16 bits of each)
    const uint64_t sd = HS, sc = sd + (((uint64_t)U * wd + 7) >> 3), so = sc + (((uint64_t)U * wc + 7) >> 3);
    const uint64_t sr = so + (((uint64_t)n * wo + 7) >> 3);
    const uint8_t* pb = P.c + P.table_end + rec->e0;
    uint32_t fl = 0;  // check bits in the reference's order (report_decode_error)
    if (tid < (PRES ? 4 : 3)) {  // zero padding (codec.py:147-148)
      const uint64_t c = tid < 2 ? U : (uint64_t)n;
      const uint32_t w = tid == 0 ? wd : tid == 1 ? wc : tid == 2 ? wo : wr;
      const uint64_t st = tid == 0 ? sd : tid == 1 ? sc : tid == 2 ? so : sr;
      const uint64_t used = c * w, nb = (used + 7) >> 3;
      if (w && c && (used & 7) && (pb[st + nb - 1] >> (used & 7))) fl |= (tid == 3) ? (1u << 15) : (1u << tid);
    }
    if (PRES)
      for (uint32_t i = tid; i < (n + 31) / 32; i += kThreads) seen[i] = 0;
    // ---- deltas + run lengths: ids (wrapping cumsum) and run starts
    unsigned long long dcarry = 0, ccarry = 0;
    for (uint32_t c0 = 0; c0 < U; c0 += kThreads) {
      const uint32_t r = c0 + tid;
      unsigned long long dl = 0, cn = 0;
      if (r < U) {
        dl = get_bits_bytes(pb, 8 * sd + (uint64_t)r * wd, wd);
        cn = get_bits_bytes(pb, 8 * sc + (uint64_t)r * wc, wc);
      }
      unsigned long long dx = dl, cx = cn, dt, ct;
      block_excl_scan2(dx, cx, dt, ct, scan);
      if (r < U) {
        const uint64_t prev = dcarry + dx, u = prev + dl;
        if (r > 0 && u <= prev) fl |= 1u << 3;            // pipeline.py:116-117
        if (cn < 1) fl |= 1u << 4;                        // pipeline.py:118-119
        if (cn >= (1ull << 63)) fl |= 1u << 6;            // codec.py:88-89
        if (!rec->pn_all && u >= rec->PN) fl |= 1u << 13;  // quantizer.py:262-263
        uniq[r] = u;
        start[r] = (uint32_t)min(ccarry + cx, (unsigned long long)0xffffffffu);
      }
      dcarry += dt;
      ccarry += ct;
    }
    if (ccarry != (unsigned long long)n) fl |= 1u << 5;   // pipeline.py:120-123
    fl |= (uint32_t)rec->geo_bits << 7;                   // pipeline.py:128-138
    __syncthreads();
    for (uint32_t p = tid; p < n; p += kThreads) {
      const uint64_t o = get_bits_bytes(pb, 8 * so + (uint64_t)p * wo, wo);
      if (rec->sumb < 64 && (o >> rec->sumb)) fl |= 1u << 14;  // quantizer.py:264-265
      if (PRES) {  // the rank stream must be a permutation (pipeline.py:149-154)
        const uint64_t rk = get_bits_bytes(pb, 8 * sr + (uint64_t)p * wr, wr);
        if (rk >= n) fl |= 1u << 16;
        else if (atomicOr(&seen[rk >> 5], 1u << (rk & 31)) & (1u << (rk & 31))) fl |= 1u << 16;
      }
    }
    uint32_t v[1] = {fl};
    block_or<1>(v, red);
    if (v[0]) {
      if (tid == 0) report_decode_error(R, blk, v[0]);
      continue;
    }
    // ---- particles: run (binary search), delinearise, midpoint (quantizer.py:194-272)
    const uint64_t obase = P.out_offsets ? P.out_offsets[blk] : blk * (uint64_t)P.bs;
    uint32_t nf = 0;
    for (uint32_t p = tid; p < n; p += kThreads) {
      uint32_t lo_i = 0, hi_i = U - 1;
      while (lo_i < hi_i) {  // last run whose start <= p
        const uint32_t mid = (lo_i + hi_i + 1) >> 1;
        if (start[mid] <= p) lo_i = mid; else hi_i = mid - 1;
      }
      const uint64_t o = get_bits_bytes(pb, 8 * so + (uint64_t)p * wo, wo);
      const uint64_t rk = PRES ? get_bits_bytes(pb, 8 * sr + (uint64_t)p * wr, wr) : p;
      uint64_t rest = uniq[lo_i];
      uint32_t sh = 0;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        uint64_t sa;
        if (a + 1 < D) {
          sa = rest % rec->N[a];
          rest /= rec->N[a];
        } else {
          sa = rest;
        }
        const uint32_t b = rec->b[a];
        const uint64_t q = shl64(sa, b) | (shr64(o, sh) & mask64(b));
        sh += b;
        double aq;
        if (rec->fast_mask & (1u << a)) {  // RN(q + 0.5) exactly: 2^51 + q + 0.5 has ulp 0.5
          aq = __dsub_rn(__longlong_as_double((long long)(0x4320000000000000ull + 2 * q + 1)), 2251799813685248.0);
        } else {
          aq = __dadd_rn(__ull2double_rn(q), 0.5);
        }
        const T tv = (T)__dadd_rn(rec->lo[a], __dmul_rn(aq, rec->w[a]));  // RN to the output precision
        if ((rec->chk_mask & (1u << a)) && !isfinite((double)tv)) nf |= 1u << a;
        const uint64_t at = obase + rk;
        if (at < P.out_cap) reinterpret_cast<T*>(P.out[a])[at] = tv;
      }
    }
    if (nf) atomicOr(&R->nonfinite_mask, nf);
  }
}

}  // namespace gpzb
