// K4w: warp-per-block decoder for the common blocks.
//
// The CTA decoder (k_decode, 256 threads x 4 particles) pays its per-thread
// fixed costs — window load, two block scans, barriers, record loads —
// over only four particles and four runs per thread.  Here one warp owns a
// whole 1024-particle block: 32 runs and 32 particles per lane, warp scans
// instead of block scans, no CTA barriers, so the fixed cost is spread over
// 8x more work and independent warps never wait for each other.
//
// Eligible blocks (K4a marks them kind = 2): the fast body (full block,
// stream widths <= 32, Σ log2 m <= 32, Π N <= 2^32, finite reconstruction,
// no rank stream) whose payload window fits kWinBytes.  Everything else goes
// to the CTA decoder through K4a's list.  Checks and their order are those
// of decode_fast (pipeline.py:106-157 semantics; lowest bit = first failure).
#pragma once

#include "gpzb_decode.cuh"

namespace gpzb {

constexpr int kWinBytes = 4096;            // payload window per warp
#ifndef GPZB_K4W_WARPS
#define GPZB_K4W_WARPS 8
#endif
constexpr int kWarpDecWarps = GPZB_K4W_WARPS;  // warps per CTA
#ifndef GPZB_K4W_MINB
#define GPZB_K4W_MINB 3
#endif
#ifndef GPZB_K4W_PF
#define GPZB_K4W_PF 1  // L2 prefetch distance in claim rounds; 0 = off
#endif
#ifndef GPZB_K4W_PF_MIN
#define GPZB_K4W_PF_MIN 512  // average payload bytes below which the prefetch is off (position blocks: 268 B, 0.65 -> 0.80 ms with it)
#endif
#ifndef GPZB_K4W_LUT_UMAX
#define GPZB_K4W_LUT_UMAX 256  // <= kWarpLutBase
#endif
// blocks with U <= GPZB_K4W_LUT_UMAX runs keep a midpoint table in the unused
// tail of `uniq` (words 256..1023: 768 f32 / 384 f64 entries)
constexpr int kWarpLutBase = 256, kWarpLutWords = kMaxBs - kWarpLutBase;
// blocks without an offset stream (w_off = 0) and few runs keep each run's
// reconstructed values there instead: [axis][run], kWarpRvStride runs per axis
constexpr int kWarpRvStride = 256;
struct WarpDecSmem {
  uint32_t win[kWinBytes / 4 + 8];
  __align__(16) uint32_t uniq[kMaxBs];     // run ids, or packed 10-bit table bases per axis + the table
  uint32_t rstart[kMaxBs / 32];
};
constexpr size_t kWarpDecSmemBytes = sizeof(WarpDecSmem) * kWarpDecWarps;

// The particle phase of K4w: 8 chunks of 128 positions, four consecutive
// per lane (one 16-byte store per axis and chunk).  Q32: every bin index
// < 2^31, so the 2^51 magic midpoint comes from one 32-bit word.
template <int D, bool F64, bool Q32, bool LUT, bool RV = false>
__device__ __forceinline__ uint32_t warp_particles(const DecParams& P, const WarpDecSmem& sm, uint64_t blk,
                                                   uint64_t idx_base, int lane, uint32_t wpre, uint32_t pbit,
                                                   uint32_t so, uint32_t wo, uint32_t sb, const double (&lo)[D],
                                                   const double (&w)[D], const uint32_t (&bsh)[D],
                                                   const uint32_t (&shifts)[D], const uint32_t (&Nn)[D],
                                                   const uint32_t (&mgm)[D], const uint32_t (&mgl)[D],
                                                   const uint32_t (&omask)[D]) {
  using T = typename std::conditional<F64, double, float>::type;
  uint32_t offbad = 0;
  const uint32_t omask4 = wo >= 32 ? 0xffffffffu : (1u << wo) - 1u;
  // a particle's run = run starts at or before it - 1; its bit in the map
  // word is (4 lane + k) mod 32 in every chunk
  uint32_t below[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) below[k] = 0xffffffffu >> (31 - ((4 * lane + k) & 31));
  // Q32: 2q + 1 = (s << (b + 1) | 1) | (o << 1), built as s * 2^(b+1) + 1 and a
  // funnel shift of the particle's offsets already doubled (q < 2^31: no overflow)
  uint32_t mul1[D], om2[D];
#pragma unroll
  for (int a = 0; a < D; ++a) {
    mul1[a] = bsh[a] >= 31 ? 0u : 1u << (bsh[a] + 1);
    om2[a] = omask[a] << 1;
  }
  // whole-block 16-byte stores when every axis is aligned and the block fits
  bool vec_ok = idx_base + kMaxBs <= P.out_cap;
#pragma unroll
  for (int a = 0; a < D; ++a) vec_ok = vec_ok && ((reinterpret_cast<uintptr_t>(reinterpret_cast<T*>(P.out[a]) + idx_base) & 15) == 0);
#pragma unroll 1
  for (int c = 0; c < kMaxBs / 128; ++c) {
    const uint32_t p0 = c * 128 + 4 * lane;
    const uint32_t wsel = p0 >> 5;  // the four share one map word
    const uint32_t word = sm.rstart[wsel];
    const uint32_t base = __shfl_sync(kFull, wpre, wsel) - 1u;
    // the four offsets are adjacent in the stream: one or two 64-bit windows
    uint32_t offs[4] = {0, 0, 0, 0};
    if constexpr (!RV) {
      const uint32_t pos = pbit + 8 * so + p0 * wo;
      const uint32_t* q = sm.win + (pos >> 5);
      const uint32_t sh = pos & 31;
      const uint64_t lo64 = (((uint64_t)q[1] << 32) | q[0]) >> sh | (sh ? (uint64_t)q[2] << (64 - sh) : 0ull);
      if (4 * wo + 0 <= 64) {
#pragma unroll
        for (int k = 0; k < 4; ++k) offs[k] = (uint32_t)(lo64 >> (k * wo)) & omask4;
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) offs[k] = get_bits32(sm.win, pos + k * wo, wo);
      }
      if (sb < 32) offbad |= (offs[0] | offs[1] | offs[2] | offs[3]) >> sb;  // quantizer.py:264-265
    }
    T vals[D][4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t run = base + __popc(word & below[k]);
      const uint32_t off = offs[k];
      if constexpr (RV) {
        // no offset stream: every particle of a run has the run's values
        const T* rvt = reinterpret_cast<const T*>(sm.uniq + kWarpLutBase);
#pragma unroll
        for (int a = 0; a < D; ++a) vals[a][k] = rvt[a * (F64 ? kWarpRvStride / 2 : kWarpRvStride) + run];
        continue;
      }
      if constexpr (LUT) {
        // the run's table bases (bin seg_a << b_a of each axis) + this particle's offsets
        const uint32_t pk = sm.uniq[run];
        const T* tab = reinterpret_cast<const T*>(sm.uniq + kWarpLutBase);
#pragma unroll
        for (int a = 0; a < D; ++a)
          vals[a][k] = tab[((pk >> (10 * a)) & 0x3ffu) + ((off >> shifts[a]) & omask[a])];
        continue;
      }
      uint32_t rest = sm.uniq[run];
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
        double h;
        if constexpr (Q32) {
          const uint32_t o2 = __funnelshift_r(off << 1, off >> 31, shifts[a]) & om2[a];
          h = __hiloint2double(0x43200000, (int)((sa * mul1[a] + 1u) | o2));
        } else {
          const uint32_t oa = (off >> shifts[a]) & omask[a];
          const uint64_t qq = ((uint64_t)sa << bsh[a]) | oa;
          h = __longlong_as_double((long long)(0x4320000000000000ull + 2 * qq + 1));
        }
        // RN(q + 0.5) exactly (2^51 magic), then lo + (q + 0.5) w (quantizer.py:132-139)
        const double aq = __dsub_rn(h, 2251799813685248.0);
        vals[a][k] = (T)__dadd_rn(lo[a], __dmul_rn(aq, w[a]));
      }
    }
    const uint64_t idx0 = idx_base + p0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      T* out = reinterpret_cast<T*>(P.out[a]);
      if (vec_ok) {
        if constexpr (sizeof(T) == 4) {
          __stcs(reinterpret_cast<float4*>(out + idx0), make_float4(vals[a][0], vals[a][1], vals[a][2], vals[a][3]));
        } else {
          __stcs(reinterpret_cast<double2*>(out + idx0), make_double2(vals[a][0], vals[a][1]));
          __stcs(reinterpret_cast<double2*>(out + idx0) + 1, make_double2(vals[a][2], vals[a][3]));
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if (idx0 + k < P.out_cap) out[idx0 + k] = vals[a][k];
      }
    }
  }
  return offbad;
}

// One block of K4w (one warp): window, runs, particles.
//
// pf_dist (bytes, multiple of 16; 0 = off): the blocks the grid decodes next
// lie about one claim round ahead in the container, i.e. at this block's
// payload + (average payload) x (warps x blocks per claim).  Lane 0
// bulk-prefetches this block's window shifted by that distance into L2 (the
// union over all blocks covers the payload region contiguously, one round
// ahead) and the record one round ahead, so the window and record loads at
// the start of a block wait on L2 instead of HBM.
template <int D, bool F64>
__device__ __forceinline__ void warp_decode_block(const DecParams& P, WarpDecSmem& sm, const uint64_t blk,
                                                  const int lane) {
  using T = typename std::conditional<F64, double, float>::type;
  DevResult* R = P.res;
  const uint8_t* cend = P.c + P.len;
  {
    const DecRec* rec = P.rec + blk;
    if (P.pf_dist && lane == 0 && blk + P.pf_blks < P.blk_hi)
      asm volatile("prefetch.global.L2 [%0];" ::"l"(P.rec + blk + P.pf_blks) : "memory");
    if (rec->kind != 2) return;  // warp-uniform
    const uint32_t U = rec->U;
    const uint32_t wd = rec->wd, wc = rec->wc, wo = rec->wo;
    const uint32_t sd = rec->sd, sc = rec->sc, so = rec->so;
    const uint32_t PN = rec->PN;  // held in a register: the run loop's shared-memory REDs would force reloads
    const uint8_t* pay = P.c + P.table_end + rec->e0;
    const uint32_t al = (uint32_t)((uintptr_t)pay & 15);
    const uint32_t plen = so + ((kMaxBs * wo + 7) >> 3);
    {  // payload window: 16-byte chunks, edges bytewise
      const uint8_t* g16 = pay - al;
      const uint32_t nch = (al + plen + 15) >> 4;
      if (P.pf_dist && lane == 0) {
        const uint8_t* pf = g16 + P.pf_dist;
        const uint64_t room = pf < cend ? (uint64_t)(cend - pf) & ~15ull : 0ull;
        const uint32_t n16 = (uint32_t)(room < 16ull * nch ? room : 16ull * nch);
        if (n16 && pf >= P.c)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(pf), "r"(n16) : "memory");
      }
      for (uint32_t ch = lane; ch < nch; ch += 32) {
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
        reinterpret_cast<uint4*>(sm.win)[ch] = v;
      }
      sm.win[((nch * 16) >> 2) + lane % 4] = 0;  // get_bits32 may read one word past the end
      sm.rstart[lane] = 0;
    }
    __syncwarp();
    const uint8_t* pb = reinterpret_cast<const uint8_t*>(sm.win) + al;
    const uint32_t pbit = 8 * al;
    uint32_t fl = 0;
    if (lane < 3) {  // zero padding (codec.py:147-148)
      const uint32_t cnt = lane < 2 ? U : (uint32_t)kMaxBs;
      const uint32_t w = lane == 0 ? wd : lane == 1 ? wc : wo;
      const uint32_t st = lane == 0 ? sd : lane == 1 ? sc : so;
      const uint32_t used = cnt * w, nb = (used + 7) >> 3;
      if (w && cnt && (used & 7) && (pb[st + nb - 1] >> (used & 7))) fl |= 1u << lane;
    }
    const bool rv = wo == 0 && U <= (F64 ? kWarpRvStride / 2 : kWarpRvStride) &&
                    D * (F64 ? kWarpRvStride / 2 : kWarpRvStride) * (F64 ? 2 : 1) <= kWarpLutWords;
    const bool wlut = !rv && U <= GPZB_K4W_LUT_UMAX && rec->lut_n != 0 &&
                      rec->lut_n <= (F64 ? kWarpLutWords / 2 : kWarpLutWords);
    if (wlut) {  // every bin's midpoint, RN_T(lo + RN(RN(q + 0.5) w)) (quantizer.py:132-139)
      T* tab = reinterpret_cast<T*>(sm.uniq + kWarpLutBase);
      const uint32_t nt = rec->lut_n, l1 = rec->lut1, l2 = rec->lut2;
      for (uint32_t i = lane; i < nt; i += 32) {
        const int a = (D > 2 && i >= l2) ? 2 : (D > 1 && i >= l1) ? 1 : 0;
        const uint32_t q = i - (a == 0 ? 0u : a == 1 ? l1 : l2);
        const double h = __hiloint2double(0x43200000, (int)(2u * q + 1u));
        tab[i] = (T)__dadd_rn(rec->lo[a], __dmul_rn(__dsub_rn(h, 2251799813685248.0), rec->w[a]));
      }
    }
    // ---- runs: lane l owns runs [l*RPL, (l+1)*RPL)
    const uint32_t RPL = (U + 31) >> 5;
    const uint32_t r0 = lane * RPL, r1 = min(U, r0 + RPL);
    unsigned long long dsum = 0;
    uint32_t csum = 0;
    // narrow streams: keep each run's (delta, count) from this pass in uniq[r]
    const bool keep = wd <= 16 && wc <= 16;
    if (keep) {
      // two runs per 32-bit funnel window of each stream (widths <= 16)
      const uint32_t md = (1u << wd) - 1u, mc = (1u << wc) - 1u;
      uint32_t pd = pbit + 8 * sd + r0 * wd, pc = pbit + 8 * sc + r0 * wc;
      uint32_t r = r0;
      for (; r + 1 < r1; r += 2, pd += 2 * wd, pc += 2 * wc) {
        const uint32_t vd = __funnelshift_r(sm.win[pd >> 5], sm.win[(pd >> 5) + 1], pd & 31);
        const uint32_t vc = __funnelshift_r(sm.win[pc >> 5], sm.win[(pc >> 5) + 1], pc & 31);
        const uint32_t d0 = vd & md, d1 = (vd >> wd) & md, c0 = vc & mc, c1 = (vc >> wc) & mc;
        dsum += d0 + d1;
        csum += c0 + c1;
        sm.uniq[r] = d0 | (c0 << 16);
        sm.uniq[r + 1] = d1 | (c1 << 16);
      }
      if (r < r1) {
        const uint32_t dl = get_bits32(sm.win, pd, wd), cn = get_bits32(sm.win, pc, wc);
        dsum += dl;
        csum += cn;
        sm.uniq[r] = dl | (cn << 16);
      }
    } else {
      for (uint32_t r = r0; r < r1; ++r) {
        const uint32_t dl = get_bits32(sm.win, pbit + 8 * sd + r * wd, wd);
        const uint32_t cn = get_bits32(sm.win, pbit + 8 * sc + r * wc, wc);
        dsum += dl;
        csum += cn;
      }
    }
    // packed warp scan (Σ deltas < 2^42 in the low 43 bits; run lengths,
    // clamped per lane at 1025, above them: a valid block sums to 1024)
    constexpr int kDBits = 43;
    constexpr unsigned long long kDMask = (1ull << kDBits) - 1;
    const unsigned long long mine = ((unsigned long long)min(csum, 1025u) << kDBits) | dsum;
    unsigned long long incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += y;
    }
    const unsigned long long ctot = __shfl_sync(kFull, incl, 31) >> kDBits;
    {
      const unsigned long long ex = incl - mine;
      // ids are prefix sums of non-negative deltas, so (pipeline.py:116-119,
      // quantizer.py:262-263): a later id not above its predecessor <=> a zero
      // delta; an id >= Π N anywhere <=> this lane's last id >= Π N (checked in
      // 64 bits once; inside the loop 32-bit ids are exact whenever it passes)
      const uint64_t prev0 = ex & kDMask;
      if (r1 > r0 && prev0 + dsum >= PN) fl |= 1u << 13;
      uint32_t uu = (uint32_t)prev0, mn_dl = 0xffffffffu, mn_cn = 0xffffffffu;
      uint32_t cex = (uint32_t)(ex >> kDBits);
      // one loop per block-uniform kind of run record (no per-run branches on
      // the kind): the run's id (plain), its table bases (wlut) or its values (rv)
      auto run_loop = [&](auto&& store_run) {
        for (uint32_t r = r0; r < r1; ++r) {
          uint32_t dl, cn;
          if (keep) {
            const uint32_t v = sm.uniq[r];
            dl = v & 0xffffu;
            cn = v >> 16;
          } else {
            dl = get_bits32(sm.win, pbit + 8 * sd + r * wd, wd);
            cn = get_bits32(sm.win, pbit + 8 * sc + r * wc, wc);
          }
          uu += dl;
          mn_dl = min(mn_dl, r ? dl : 0xffffffffu);
          mn_cn = min(mn_cn, cn);
          store_run(r, uu);
          red_or_shared_if(cex < (uint32_t)kMaxBs, &sm.rstart[cex >> 5], 1u << (cex & 31));
          cex += cn;
        }
      };
      if (rv) {
        run_loop([&](uint32_t r, uint32_t u) {
          // the run's reconstruction per axis, as the midpoint table would hold it
          T* rvt = reinterpret_cast<T*>(sm.uniq + kWarpLutBase);
          uint32_t rest = u;  // u < Π N <= 2^32 (else the block is reported below)
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
            const uint64_t qq = (uint64_t)sa << rec->b[a];
            const double h = __longlong_as_double((long long)(0x4320000000000000ull + 2 * qq + 1));
            rvt[a * (F64 ? kWarpRvStride / 2 : kWarpRvStride) + r] =
                (T)__dadd_rn(rec->lo[a], __dmul_rn(__dsub_rn(h, 2251799813685248.0), rec->w[a]));
          }
          sm.uniq[r] = u;
        });
      } else if (wlut) {
        run_loop([&](uint32_t r, uint32_t u) {
          uint32_t rest = u, pk = 0;
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
            const uint32_t lb = a == 0 ? 0u : a == 1 ? (uint32_t)rec->lut1 : (uint32_t)rec->lut2;
            pk |= ((lb + (sa << rec->b[a])) & 0x3ffu) << (10 * a);
          }
          sm.uniq[r] = pk;
        });
      } else {
        run_loop([&](uint32_t r, uint32_t u) { sm.uniq[r] = u; });
      }
      if (mn_dl == 0) fl |= 1u << 3;  // pipeline.py:116-117
      if (mn_cn == 0) fl |= 1u << 4;  // pipeline.py:118-119
    }
    if (ctot != (unsigned long long)kMaxBs) fl |= 1u << 5;  // pipeline.py:120-123
    fl = __reduce_or_sync(kFull, fl);
    if (fl) {
      if (lane == 0) report_decode_error(R, blk, fl);
      __syncwarp();
      return;
    }
    __syncwarp();
    // ---- run-start map prefix: lane w holds the starts before word w
    const uint32_t wcount = __popc(sm.rstart[lane]);
    uint32_t wpre = wcount;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(kFull, wpre, o);
      if (lane >= o) wpre += y;
    }
    wpre -= wcount;
    // ---- geometry constants (warp-uniform)
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
    const bool q32 = rec->fast_body != 1;  // every bin index < 2^31 (fast bodies 2 and 3)
    const uint32_t sb = rec->sumb;
    const uint64_t idx_base = P.out_offsets ? P.out_offsets[blk] : blk * (uint64_t)P.bs;
    const uint32_t offbad =
        rv    ? warp_particles<D, F64, true, false, true>(P, sm, blk, idx_base, lane, wpre, pbit, so, wo, sb, lo, w,
                                                          bsh, shifts, Nn, mgm, mgl, omask)
        : wlut  ? warp_particles<D, F64, true, true>(P, sm, blk, idx_base, lane, wpre, pbit, so, wo, sb, lo, w, bsh,
                                                   shifts, Nn, mgm, mgl, omask)
        : q32 ? warp_particles<D, F64, true, false>(P, sm, blk, idx_base, lane, wpre, pbit, so, wo, sb, lo, w, bsh,
                                                    shifts, Nn, mgm, mgl, omask)
              : warp_particles<D, F64, false, false>(P, sm, blk, idx_base, lane, wpre, pbit, so, wo, sb, lo, w,
                                                     bsh, shifts, Nn, mgm, mgl, omask);
    if (__any_sync(kFull, offbad != 0) && lane == 0) report_decode_error(R, blk, 1u << 14);
    __syncwarp();
  }
}

// K4w: one warp per fast-body block, persistent CTAs.  Blocks are claimed in
// chunks of k from a counter (one chunk ahead, so the atomic's latency hides
// behind the current chunk): CTAs that start late (another kernel holds the
// SMs) still leave the work balanced.  k grows with the blocks per warp
// (1 below 128 per warp, up to 8): same-address atomics serialise in L2,
// and a container of ~10^6 cheap blocks would otherwise wait on its claims
// (1B particles at rel-eb 1e-2: 3.22 -> 2.05 ms).
#ifndef GPZB_K4W_CLAIM_K
#define GPZB_K4W_CLAIM_K 0  // 0: adaptive
#endif
__host__ __device__ inline uint32_t warp_claim_chunk(uint32_t nblk, uint32_t grid) {
  if (GPZB_K4W_CLAIM_K) return GPZB_K4W_CLAIM_K;
  const uint32_t k = nblk / (64u * grid * kWarpDecWarps);
  return k < 1u ? 1u : k > 8u ? 8u : k;
}

template <int D, bool F64>
__global__ void __launch_bounds__(32 * kWarpDecWarps, GPZB_K4W_MINB) k_decode_warp(const DecParams P) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpDecSmem& sm = reinterpret_cast<WarpDecSmem*>(dsm)[wid];
  unsigned int* claim = &P.res->claim;
  const uint32_t nblk = (uint32_t)(P.blk_hi - P.blk_lo);
  const uint32_t k = warp_claim_chunk(nblk, gridDim.x);
  uint32_t i = lane == 0 ? atomicAdd(claim, k) : 0u, nxt = 0;
  for (i = __shfl_sync(kFull, i, 0); i < nblk; i = __shfl_sync(kFull, nxt, 0)) {
    if (lane == 0) nxt = atomicAdd(claim, k);
    const uint32_t e = min(i + k, nblk);
    for (uint32_t b = i; b < e; ++b) warp_decode_block<D, F64>(P, sm, P.blk_lo + b, lane);
  }
}

// The CTA decoder over K4a's list of the remaining blocks (persistent CTAs).
template <int D, bool F64, bool PRES>
__global__ void __launch_bounds__(kThreads, GPZB_K4_MINB) k_decode_list(const DecParams P, const uint32_t* list) {
  __shared__ DecSmem sm;
  const uint32_t cnt = *reinterpret_cast<volatile const uint32_t*>(&P.res->wide_count);
  for (uint32_t i = blockIdx.x; i < cnt; i += gridDim.x) {
    const uint64_t blk = list[i];
    const DecRec* rec = P.rec + blk;
    if (!PRES && rec->fast_body) decode_fast<D, F64>(P, sm, blk, rec);
    else decode_general<D, F64, PRES>(P, sm, blk, rec);
    __syncthreads();
  }
}

}  // namespace gpzb
