// K2: the 32-bit fast block encoder.
//
// One CTA (256 threads x 4 particles) per block, in launch order.  For
// "narrow" blocks (K1.5: every axis on the certified-reciprocal quantizer,
// Π N <= 2^16, Σ log2 m <= 32, no rank stream) it does the whole of
// pipeline._encode_block (pipeline.py:38-70):
//
//   quantize (quantizer.py:142-191)  -> 32-bit (segment, offset) per particle
//   pass A: presence bitmap over [0, Π N) -> distinct-segment ranks, run
//           lengths and unique ids in one pass (RLE, codec.py:53-79)
//   widths (codec.width_for) by OR-reduction -> payload length
//   offset order (blocksort.py:17-28): per-segment (offset, tie) masks, or a
//           presence bitmap over (segment rank, offset), or in-group
//           comparison ranks, or a stable 5-bit LSD (ties are identical
//           pairs, so any tie order serialises to the same bytes)
//   bit-pack header + streams into shared memory, then 16-byte stores of the
//           payload into the block's staging slot and its length into
//           sizes[blk] for the K3 scan + copy (gpzb_compact.cuh).
//
// General blocks (staged by K2w) and error blocks only report their length.
#pragma once

#include "gpzb_compact.cuh"

namespace gpzb {

#ifndef GPZB_K2_MINB
#define GPZB_K2_MINB 6
#endif
constexpr int kNarrowStageWords = 2048 + 32;  // narrow payload <= 7.7 KB
constexpr uint32_t kGroupMaskWords = 3584;    // path 5: per-segment (offset, tie) masks

struct NarrowSmem {
  BlkRec rec;  // this block's geometry record (K1.5), staged once
  uint32_t red[kWarps * 4];
  uint32_t scan32[kWarps];
  __align__(16) uint32_t cnt[kMaxBs];   // run length per distinct segment rank
  __align__(16) uint32_t soff[kMaxBs];  // offsets in sorted order
  __align__(16) uint16_t uniqp[kMaxBs + 8];  // [0] = 0 sentinel, [r + 1] = unique id r (Π N <= 2^16)
  union U {
    struct { uint32_t bm[2048]; uint16_t wp[2048]; } a;
    struct { uint32_t bm[2048]; uint16_t wp[2048]; uint32_t cnt2[kMaxBs]; } b;
    struct { uint16_t segstart[kMaxBs]; uint32_t tmp[kMaxBs]; } c;
    struct { uint32_t gm[kGroupMaskWords]; uint16_t segstart[kMaxBs]; } g;
    struct { uint32_t off[kMaxBs]; uint16_t sr[kMaxBs]; uint32_t bm[1024]; uint16_t wp[1024]; } l;
    uint32_t stage[kNarrowStageWords];
  };
  __align__(16) U u;
};

// Vectorised loads of a full block's 4 particles per thread (16-byte aligned axes).
template <int D, typename T>
__device__ __forceinline__ void load_full(const EncParams& P, uint64_t first, int p0, T (&x)[D][kItems]) {
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const T* base = reinterpret_cast<const T*>(P.axes[a]) + first + p0;
    if constexpr (sizeof(T) == 4) {
      const float4 v = __ldcs(reinterpret_cast<const float4*>(base));
      x[a][0] = v.x; x[a][1] = v.y; x[a][2] = v.z; x[a][3] = v.w;
    } else {
      const double2 v0 = __ldcs(reinterpret_cast<const double2*>(base));
      const double2 v1 = __ldcs(reinterpret_cast<const double2*>(base) + 1);
      x[a][0] = v0.x; x[a][1] = v0.y; x[a][2] = v1.x; x[a][3] = v1.y;
    }
  }
}

// Exact-division (segment, offset) of one particle: the rare fallback of the
// certified quantizer, out of line so the fast path keeps no temporaries
// alive for it.  Returns seg << 32 | off.
template <int D, typename T>
__device__ __noinline__ uint64_t redo_exact(T x0, T x1, T x2, const BlkRec* rec) {
  uint32_t sk = 0, ok = 0, st = 1, sh = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const T xa = a == 0 ? x0 : (a == 1 ? x1 : x2);
    const double t = __dsub_rn((double)xa, rec->lo[a]);
    const uint32_t q = (uint32_t)__double2ull_rz(__ddiv_rn(t, rec->w[a]));
    const uint32_t b = rec->b[a];
    sk += (q >> b) * st;
    ok |= (q & ((1u << b) - 1u)) << (sh & 31);
    st *= rec->N[a];
    sh += b;
  }
  return ((uint64_t)sk << 32) | ok;
}

template <int D, bool F64, bool FULL>
__device__ __forceinline__ void narrow_body(const EncParams& P, NarrowSmem& sm, const uint64_t blk,
                                            const BlkRec* rec, const int n,
                                            typename std::conditional<F64, double, float>::type (&x)[D][kItems]) {
  using T = typename std::conditional<F64, double, float>::type;
  constexpr int S = F64 ? 8 : 4;
  constexpr uint32_t H = 8 + D * (2 * S + 5) + 3;  // block header bytes (container.py:62-67)
  const int tid = threadIdx.x;
  const uint64_t first = blk * (uint64_t)P.bs;
  const int p0 = tid * kItems;
#define VALID(k) (FULL || p0 + (k) < n)

  // ---- 1. load (full blocks: already issued by the caller) + quantize to 32-bit (segment, offset)
  if constexpr (!FULL) load_particles<D, T>(P, first, n, p0, x);
  const uint32_t PN = rec->PN, sumb = rec->sumb;
  uint32_t seg[kItems], off[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) { seg[k] = 0; off[k] = 0; }
  {
    // certified reciprocal quantizer (gpzb_common.cuh quantize_coord, mode 0);
    // coordinates whose certificate fails are redone exactly in one
    // warp-uniform pass (rare: t == 0 or RN(t/w) within an ulp of an integer)
    uint32_t redo = 0;
    uint32_t stride = 1, shift = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const double lo = rec->lo[a], rinv = rec->rinv[a];
      const uint32_t b = rec->b[a];
      const uint32_t mk = (1u << b) - 1u;
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        const double t = __dsub_rn((double)x[a][k], lo);
        const double r = __dmul_rn(t, rinv);
        const uint32_t rl = (uint32_t)__double2loint(r), rh = (uint32_t)__double2hiint(r);
        const uint32_t q = (uint32_t)__double2loint(__dadd_rz(r, 4503599627370496.0));
        redo |= ((rl + 1u) <= 1u && (rl | rh) != 0u) ? (1u << k) : 0u;  // r == 0 is exact
        seg[k] += (q >> b) * stride;
        off[k] |= (q & mk) << (shift & 31);  // b == 0 -> mk == 0
      }
      stride *= rec->N[a];
      shift += b;
    }
    if (__any_sync(kFull, redo != 0) && redo) {
      // re-linearise all four particles of this thread with exact division
      // (identical wherever the certificate held): the fast path's seg / off
      // are then dead in this branch and need not survive the calls
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        const uint64_t so = redo_exact<D, T>(x[0][k], D > 1 ? x[D > 1 ? 1 : 0][k] : T(0),
                                             D > 2 ? x[D > 2 ? 2 : 0][k] : T(0), rec);
        seg[k] = (uint32_t)(so >> 32);
        off[k] = (uint32_t)so;
      }
    }
  }
  uint32_t off_or = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) off_or |= VALID(k) ? off[k] : 0u;

  // ---- 2. pass A: distinct-segment ranks, run lengths, unique ids
  const int nwA = (int)((PN + 31) >> 5);
  bm_zero(sm.u.a.bm, nwA);
  reinterpret_cast<uint4*>(sm.cnt)[tid] = make_uint4(0, 0, 0, 0);
  if (tid == 0) sm.uniqp[0] = 0;
  if (tid < 3) sm.red[tid] = 0;  // block_or_z accumulators
  __syncthreads();
#pragma unroll
  for (int k = 0; k < kItems; ++k)
    if (VALID(k)) red_or_shared(&sm.u.a.bm[seg[k] >> 5], 1u << (seg[k] & 31));
  __syncthreads();
  const uint32_t U = bm_prefix(sm.u.a.bm, sm.u.a.wp, nwA, sm.scan32);
  __syncthreads();
  uint32_t srank[kItems], tie[kItems];
#pragma unroll
  for (int k = 0; k < kItems; ++k) {
    srank[k] = tie[k] = 0;
    if (VALID(k)) {
      srank[k] = bm_rank(sm.u.a.bm, sm.u.a.wp, seg[k]);
      tie[k] = atomicAdd(&sm.cnt[srank[k]], 1u);
      sm.uniqp[srank[k] + 1] = (uint16_t)seg[k];
    }
  }
  __syncthreads();

  // ---- 3. stream widths (width_for == bit length of the OR) and payload size
  // this thread's runs p0..p0+3 are also the ones it packs in step 5: keep
  // each run's delta | count << 16 (delta < 2^16, count <= 1024) in registers
  // (vector loads: counts p0..p0+3 in one 16-byte word, ids p0..p0+4 in an
  // 8-byte word + one; runs >= U are masked, no branches)
  uint32_t dc[kItems], csum = 0, c_or = 0, d_or = 0;
  {
    const uint4 c4 = reinterpret_cast<const uint4*>(sm.cnt)[tid];
    const uint2 u4 = reinterpret_cast<const uint2*>(sm.uniqp)[tid];
    const uint32_t u[5] = {u4.x & 0xffffu, u4.x >> 16, u4.y & 0xffffu, u4.y >> 16, (uint32_t)sm.uniqp[p0 + 4]};
    const uint32_t cc[4] = {c4.x, c4.y, c4.z, c4.w};
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const bool in = (uint32_t)(p0 + j) < U;
      const uint32_t c = in ? cc[j] : 0u, d = in ? u[j + 1] - u[j] : 0u;
      c_or |= c;
      d_or |= d;
      csum += c;
      dc[j] = d | (c << 16);
    }
  }
  uint32_t red[3] = {off_or, c_or, d_or};
  block_or_z<3>(red, sm.red);
  const uint32_t w_off = bitlen32(red[0]), w_cnt = bitlen32(red[1]), w_del = bitlen32(red[2]);
  const uint32_t Ld = (U * w_del + 7) >> 3, Lc = (U * w_cnt + 7) >> 3, Lo = ((uint32_t)n * w_off + 7) >> 3;
  const uint32_t L = H + Ld + Lc + Lo;
  if (tid == 0) P.status[blk] = L;  // payload length for the K3 scan

  // ---- 4. order the offsets: (segment rank, offset) composite ranks
  int path = 0;
  if (w_off) {
    uint32_t pos[kItems];
    // (offset, tie) codes are unique inside a segment group, so a per-group
    // presence mask ranks them directly; ties are identical (seg, off)
    // pairs, any order of which serialises to the same bytes
    const uint32_t cb = sumb + w_cnt;  // tie < max run length < 2^w_cnt
    const uint32_t W = cb <= 5 ? 1u : (1u << (cb - 5));
    if (cb <= 7 && U * W <= kGroupMaskWords) {
      path = 5;
      uint32_t* gm = sm.u.g.gm;
      for (uint32_t w = tid; w < (U * W + 3) >> 2; w += kThreads)
        reinterpret_cast<uint4*>(gm)[w] = make_uint4(0, 0, 0, 0);
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(csum, tot, sm.scan32);  // its barriers order the zeroing
      {  // the four run starts in one 8-byte store (entries past U are never read)
        const uint32_t e0 = ex, e1 = e0 + (dc[0] >> 16), e2 = e1 + (dc[1] >> 16), e3 = e2 + (dc[2] >> 16);
        if (p0 < (int)U) reinterpret_cast<uint2*>(sm.u.g.segstart)[tid] = make_uint2(e0 | (e1 << 16), e2 | (e3 << 16));
      }
      uint32_t code[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        code[k] = (off[k] << w_cnt) | tie[k];
        if VALID(k) red_or_shared(&gm[srank[k] * W + (code[k] >> 5)], 1u << (code[k] & 31));
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        pos[k] = 0;
        if VALID(k) {
          // codes below mine in the group's 32 / 64 / 128-bit mask (W is block-uniform)
          const uint32_t c = code[k];
          uint32_t r;
          if (W == 1) {
            r = __popc(gm[srank[k]] & ((1u << c) - 1u));
          } else if (W == 2) {
            const uint2 m = reinterpret_cast<const uint2*>(gm)[srank[k]];
            r = __popcll((((uint64_t)m.y << 32) | m.x) & ((1ull << c) - 1ull));
          } else {
            const uint4 m = reinterpret_cast<const uint4*>(gm)[srank[k]];
            const uint64_t lo = ((uint64_t)m.y << 32) | m.x, hi = ((uint64_t)m.w << 32) | m.z;
            const uint32_t ch = c & 63;
            r = c < 64 ? __popcll(lo & ((1ull << ch) - 1ull))
                       : __popcll(lo) + __popcll(hi & ((1ull << ch) - 1ull));
          }
          pos[k] = sm.u.g.segstart[srank[k]] + r;
        }
      }
    } else if (w_cnt > 3 && sumb <= 16 && (U << sumb) <= 65536u) {
      path = 1;
      const int nw = (int)(((U << sumb) + 31) >> 5);
      bm_zero(sm.u.b.bm, nw);
      reinterpret_cast<uint4*>(sm.u.b.cnt2)[tid] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      uint32_t c[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        c[k] = (srank[k] << sumb) | off[k];
        if VALID(k) red_or_shared(&sm.u.b.bm[c[k] >> 5], 1u << (c[k] & 31));
      }
      __syncthreads();
      const uint32_t nd = bm_prefix(sm.u.b.bm, sm.u.b.wp, nw, sm.scan32);
      __syncthreads();
      uint32_t cr[kItems], t2[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        cr[k] = t2[k] = 0;
        if VALID(k) {
          cr[k] = bm_rank(sm.u.b.bm, sm.u.b.wp, c[k]);
          t2[k] = atomicAdd(&sm.u.b.cnt2[cr[k]], 1u);
        }
      }
      __syncthreads();
      uint32_t v[kItems], loc = 0;
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        v[j] = (p0 + j < (int)nd) ? sm.u.b.cnt2[p0 + j] : 0u;
        loc += v[j];
      }
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(loc, tot, sm.scan32);
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        if (p0 + j < (int)nd) sm.u.b.cnt2[p0 + j] = ex;
        ex += v[j];
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kItems; ++k) pos[k] = VALID(k) ? sm.u.b.cnt2[cr[k]] + t2[k] : 0u;
    } else if (w_cnt <= 6) {
      // segment groups of <= 63 particles: rank by comparison inside the group
      path = 2;
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(csum, tot, sm.scan32);
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        if (p0 + j < (int)U) sm.u.c.segstart[p0 + j] = (uint16_t)ex;
        ex += dc[j] >> 16;
      }
      __syncthreads();
      uint32_t g0[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        g0[k] = 0;
        if VALID(k) {
          g0[k] = sm.u.c.segstart[srank[k]];
          sm.u.c.tmp[g0[k] + tie[k]] = off[k];
        }
      }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        pos[k] = 0;
        if VALID(k) {
          const uint32_t gs = sm.cnt[srank[k]], me = g0[k] + tie[k];
          uint32_t rr = 0;
          for (uint32_t j = g0[k]; j < g0[k] + gs; ++j) {
            const uint32_t o = sm.u.c.tmp[j];
            rr += (o < off[k]) || (o == off[k] && j < me);
          }
          pos[k] = g0[k] + rr;
        }
      }
    } else {
      // large groups and a wide composite: stable LSD, 5-bit digits
      path = 3;
      const uint32_t total_bits = sumb + (uint32_t)bitlen32(U - 1);
      for (uint32_t s = 0; s < total_bits; s += 5) {
        const int dlen = (int)min(5u, total_bits - s);
        uint32_t dig[kItems], np[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          const uint64_t key = ((uint64_t)srank[k] << sumb) | off[k];
          dig[k] = (uint32_t)(key >> s) & ((1u << dlen) - 1u);
        }
        lsd_ranks(dig, dlen, n, p0, sm.u.l.bm, sm.u.l.wp, sm.scan32, np);
#pragma unroll
        for (int k = 0; k < kItems; ++k)
          if (p0 + k < n) { sm.u.l.off[np[k]] = off[k]; sm.u.l.sr[np[k]] = (uint16_t)srank[k]; }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kItems; ++k)
          if (p0 + k < n) { off[k] = sm.u.l.off[p0 + k]; srank[k] = sm.u.l.sr[p0 + k]; }
        __syncthreads();
      }
#pragma unroll
      for (int k = 0; k < kItems; ++k) pos[k] = p0 + k;
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if VALID(k) sm.soff[pos[k]] = off[k];
  }
  __syncthreads();  // soff complete; union free for the stage

  // ---- 5. bit-pack header + streams into the stage (payload byte 0 = stage byte 0)
  uint32_t* st = sm.u.stage;
  if (tid == 0) P.rec[blk].path = (uint8_t)path;  // diagnostics: gpzb_encode_path_counts
  const uint32_t nquads = (L + 15) >> 4;
  for (uint32_t w = tid; w < nquads; w += kThreads) reinterpret_cast<uint4*>(st)[w] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  {
    const int t = tid, nt = kThreads;
    if (t < 32) {
      // block header fields, one per lane (container.serialize_block, container.py:107-121)
      const int f = t;
      uint32_t bpos = 0;
      uint64_t val = 0;
      bool act = true;
      if (f == 0) { bpos = 0; val = (uint32_t)n; }
      else if (f == 1) { bpos = 4; val = U; }
      else if (f < 2 + 4 * D) {
        const int a = (f - 2) >> 2, which = (f - 2) & 3;
        const uint32_t ab = 8 + a * (2 * S + 5);
        const T* bnd = reinterpret_cast<const T*>(P.bounds) + blk * 2 * D;
        if (which < 2) {
          bpos = ab + which * S;
          const T v = bnd[2 * a + which];
          if constexpr (F64) val = (uint64_t)__double_as_longlong(v);
          else val = __float_as_uint(v);
        } else if (which == 2) { bpos = ab + 2 * S; val = rec->b[a]; }
        else { bpos = ab + 2 * S + 1; val = rec->N[a]; }
      } else if (f < 2 + 4 * D + 3) {
        const int wi = f - 2 - 4 * D;
        bpos = 8 + D * (2 * S + 5) + wi;
        val = wi == 0 ? w_del : wi == 1 ? w_cnt : w_off;
      } else {
        act = false;
      }
      if (act) or_bits(st, 8ull * bpos, val);
    }
    const uint64_t bd = 8ull * H, bc = bd + 8ull * Ld, bo = bc + 8ull * Lc;
    // deltas + run lengths, 4 consecutive runs per chunk (32-bit windows
    // when four values fit in 32 bits, else 64-bit ones)
    const bool d32 = 4 * w_del <= 32, c32 = 4 * w_cnt <= 32;
    static_assert(kItems == 4 && kThreads * kItems >= kMaxBs, "one chunk of four runs per thread");
    if (p0 < (int)U) {
      const uint32_t r0 = p0;
      uint32_t d[4], cn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        d[j] = dc[j] & 0xffffu;
        cn[j] = dc[j] >> 16;
      }
      if (d32) {
        if (w_del) or_bits32(st, (uint32_t)bd + r0 * w_del, d[0] | d[1] << w_del | d[2] << (2 * w_del) | d[3] << (3 * w_del));
      } else {
        uint64_t dv = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) dv |= (uint64_t)d[j] << (j * w_del);
        or_bits(st, bd + (uint64_t)r0 * w_del, dv);
      }
      if (c32) {
        if (w_cnt) or_bits32(st, (uint32_t)bc + r0 * w_cnt, cn[0] | cn[1] << w_cnt | cn[2] << (2 * w_cnt) | cn[3] << (3 * w_cnt));
      } else {
        uint64_t cv = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) cv |= (uint64_t)cn[j] << (j * w_cnt);
        or_bits(st, bc + (uint64_t)r0 * w_cnt, cv);
      }
    }
    // offsets in sorted order, 4 per chunk: one 32-bit window when they fit,
    // else two 2-value 64-bit halves
    if (w_off) {
      for (uint32_t p = 4 * t; p < (uint32_t)n; p += 4 * nt) {
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) o[j] = p + j < (uint32_t)n ? sm.soff[p + j] : 0u;
        if (4 * w_off <= 32) {
          or_bits32(st, (uint32_t)bo + p * w_off, o[0] | o[1] << w_off | o[2] << (2 * w_off) | o[3] << (3 * w_off));
        } else {
          or_bits(st, bo + (uint64_t)p * w_off, (uint64_t)o[0] | (uint64_t)o[1] << w_off);
          or_bits(st, bo + (uint64_t)(p + 2) * w_off, (uint64_t)o[2] | (uint64_t)o[3] << w_off);
        }
      }
    }
  }
  __syncthreads();

  // ---- 6. the stage to this block's 16-byte aligned staging slot (K3 moves it into place)
  uint4* slot = reinterpret_cast<uint4*>(P.staging + blk * (uint64_t)kSlotBytes);
  for (uint32_t w = tid; w < nquads; w += kThreads) __stcg(slot + w, reinterpret_cast<const uint4*>(st)[w]);
#undef VALID
}

template <int D, bool F64>
__global__ void __launch_bounds__(kThreads, GPZB_K2_MINB) k_encode(const EncParams P) {
  __shared__ NarrowSmem sm;
  const int tid = threadIdx.x;
  using T = typename std::conditional<F64, double, float>::type;
  // persistent over K1.5's list of narrow blocks (plus the blocks K2s handed
  // back); the list length is read on the device, so the host never waits
  const uint32_t count = *reinterpret_cast<volatile const uint32_t*>(&P.res->cta_count);
  for (uint32_t item = blockIdx.x; item < count; item += gridDim.x) {
    const uint64_t blk = (uint64_t)P.cta_list[item];
    const uint64_t first = blk * (uint64_t)P.bs;
    const int n = (int)min((uint64_t)P.bs, P.count - first);
    const bool full = n == kMaxBs && P.vec;
    T x[D][kItems];
    if (full) load_full<D, T>(P, first, tid * kItems, x);  // in flight while the record is staged
    if (tid < 8) reinterpret_cast<uint4*>(&sm.rec)[tid] = reinterpret_cast<const uint4*>(P.rec + blk)[tid];
    __syncthreads();
    const BlkRec* rec = &sm.rec;
    if (rec->kind == KIND_NARROW) {  // block-uniform
      if (full) narrow_body<D, F64, true>(P, sm, blk, rec, n, x);
      else narrow_body<D, F64, false>(P, sm, blk, rec, n, x);
    }
    __syncthreads();  // the shared state is reused by the next block
  }
}

}  // namespace gpzb
