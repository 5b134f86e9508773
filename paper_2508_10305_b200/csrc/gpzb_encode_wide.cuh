// K2w: the general block encoder for blocks outside the 32-bit fast path
// (wide keys, exact-division or half-bound quantizer axes, preserve_order,
// Π N > 2^16).  Same four stages as pipeline._encode_block (pipeline.py:38-70);
// payloads go to a side buffer that K2 copies into the container in block
// order.  Persistent CTAs loop over the K1.5 wide list.
#pragma once

#include "gpzb_encode.cuh"

namespace gpzb {

struct WideSmem {
  uint64_t blk;
  uint64_t excl;
  AxisGeo geo[3];
  int ax_err[3];
  int pad_;
  __align__(16) double redd[3 * 2 * kWarps];
  uint32_t red[kWarps * 8];
  uint32_t scan32[kWarps];
  unsigned long long scan64[kWarps];
  __align__(16) uint32_t cnt[kMaxBs];   // run length per distinct segment rank
  __align__(16) uint64_t uniq[kMaxBs];  // unique segment ids (increasing)
  union U {
    struct { uint32_t bm[2048]; uint16_t wp[2048]; } a;  // pass A: segment bitmap
    struct {
      uint32_t bm[2048]; uint16_t wp[2048]; uint32_t cnt2[kMaxBs];
    } b;                                                  // pass B: (rank, offset) bitmap
    struct { uint16_t segstart[kMaxBs]; uint64_t tmp[kMaxBs]; } c;  // in-group compare
    struct {
      uint64_t off[kMaxBs]; uint16_t sr[kMaxBs]; uint16_t rk[kMaxBs]; uint32_t bm[2048]; uint16_t wp[2048];
    } l;                                                  // LSD on (rank, offset)
    struct {
      uint64_t off[kMaxBs]; uint64_t seg[kMaxBs]; uint16_t rk[kMaxBs]; uint32_t bm[1024]; uint16_t wp[1024];
    } g;                                                  // LSD on (segment, offset)
    uint32_t stage[6144];                                 // payload staging (24 KB)
  };
  __align__(16) U u;
};

template <int D, bool F64, bool PRES>
__global__ void __launch_bounds__(kThreads) k_encode_wide(const EncParams P) {
  using T = typename std::conditional<F64, double, float>::type;
  constexpr int S = F64 ? 8 : 4;
  constexpr int H = 8 + D * (2 * S + 5) + (PRES ? 4 : 3);  // block header bytes (container.py:62-67)
  __shared__ WideSmem sm;
  const int tid = threadIdx.x, lane = tid & 31;
  DevResult* R = P.res;
  const uint32_t nwide = R->wide_count;
  for (uint32_t item = blockIdx.x; item < nwide; item += gridDim.x) {
  __syncthreads();  // smem reuse across items
  const uint64_t blk = P.wide_list[item];
  const uint64_t first = blk * (uint64_t)P.bs;
  const int n = (int)min((uint64_t)P.bs, P.count - first);
  const int p0 = tid * kItems;

  // ---- 1. load the block (coalesced 16B loads, evict-first)
  T x[D][kItems];
  load_particles<D, T>(P, first, n, p0, x);

  // ---- 2. block bounds from K1, eb_abs from K1.5
  double lo[D], hi[D];
  {
    const T* b = reinterpret_cast<const T*>(P.bounds) + blk * 2 * D;
#pragma unroll
    for (int a = 0; a < D; ++a) { lo[a] = (double)b[2 * a]; hi[a] = (double)b[2 * a + 1]; }
  }
  const double eb_abs = R->eb_abs;

  // ---- 3. geometry (one thread per axis)
  if (tid < D) sm.ax_err[tid] = axis_geometry(lo[tid], hi[tid], eb_abs, F64, P.target, sm.geo[tid]);
  __syncthreads();
  int err = R_NONE, err_axis = 0;
  if (!(eb_abs > 0.0)) {
    err = R_EB_NOT_POSITIVE;
  } else {
#pragma unroll
    for (int a = D - 1; a >= 0; --a)
      if (sm.ax_err[a]) { err = R_AXIS_RANGE; err_axis = a; }
  }
  unsigned __int128 PN = 1;
  uint32_t sumb = 0;
  uint64_t stride[D];
  uint32_t shift[D];
  if (!err) {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      stride[a] = (uint64_t)PN;  // Π N of earlier axes (<= 2^64 checked below)
      shift[a] = sumb;
      PN *= sm.geo[a].N;
      if (PN > ((unsigned __int128)1 << 64)) { err = R_GEOMETRY; break; }
      sumb += sm.geo[a].b;
    }
    if (sumb > 64) err = R_GEOMETRY;
  }

  // ---- 4. quantize + linearize (quantizer.py:142-191)
  uint64_t seg[kItems], off[kItems];
  uint64_t off_or = 0;
  if (!err) {
#pragma unroll
    for (int k = 0; k < kItems; ++k) { seg[k] = 0; off[k] = 0; }
#pragma unroll
    for (int a = 0; a < D; ++a) {
      const AxisGeo g = sm.geo[a];
      const uint64_t mk = mask64(g.b);
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        if (p0 + k < n) {
          uint64_t q = quantize_coord((double)x[a][k], g, eb_abs, F64);
          seg[k] += shr64(q, g.b) * stride[a];
          off[k] |= shl64(q & mk, shift[a]);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < kItems; ++k) off_or |= (p0 + k < n) ? off[k] : 0ull;
  }

  // ---- 5. counting sort + run-length statistics
  const bool passA = !err && PN <= 65536;
  uint32_t srank[kItems], tie[kItems], pos[kItems];
  uint32_t rk[kItems];  // original intra-block index (rank stream)
  uint32_t U = 0;
  int path = 0;
#pragma unroll
  for (int k = 0; k < kItems; ++k) { srank[k] = tie[k] = 0; pos[k] = p0 + k; rk[k] = p0 + k; }

  if (passA) {
    // distinct-segment ranks from a presence bitmap over [0, ΠN)
    const int nw = (int)(((uint32_t)PN + 31) >> 5);
    bm_zero(sm.u.a.bm, nw);
    reinterpret_cast<uint4*>(sm.cnt)[tid] = make_uint4(0, 0, 0, 0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (p0 + k < n) atomicOr(&sm.u.a.bm[seg[k] >> 5], 1u << (seg[k] & 31));
    __syncthreads();
    U = bm_prefix(sm.u.a.bm, sm.u.a.wp, nw, sm.scan32);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (p0 + k < n) {
        srank[k] = bm_rank(sm.u.a.bm, sm.u.a.wp, (uint32_t)seg[k]);
        tie[k] = atomicAdd(&sm.cnt[srank[k]], 1u);
        sm.uniq[srank[k]] = seg[k];
      }
    __syncthreads();
  } else if (!err) {
    // general key width: stable LSD over (segment, offset) with 5-bit digits
    path = 4;
    const uint32_t segbits = (uint32_t)bitlen64((uint64_t)(PN - 1));
    const uint32_t total_bits = sumb + segbits;
    for (uint32_t s = 0; s < total_bits; s += 5) {
      const int dlen = (int)min(5u, total_bits - s);
      uint32_t dig[kItems], np[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        uint64_t v = s < sumb ? shr64(off[k], s) : shr64(seg[k], s - sumb);
        if (s < sumb && s + dlen > sumb) v = (off[k] >> s) | shl64(seg[k], sumb - s);
        dig[k] = (uint32_t)(v & ((1u << dlen) - 1u));
      }
      lsd_ranks(dig, dlen, n, p0, sm.u.g.bm, sm.u.g.wp, sm.scan32, np);
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (p0 + k < n) { sm.u.g.off[np[k]] = off[k]; sm.u.g.seg[np[k]] = seg[k]; sm.u.g.rk[np[k]] = (uint16_t)rk[k]; }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (p0 + k < n) { off[k] = sm.u.g.off[p0 + k]; seg[k] = sm.u.g.seg[p0 + k]; rk[k] = sm.u.g.rk[p0 + k]; }
      __syncthreads();
    }
    // run-length factorisation of the sorted segment ids (codec.py:53-79)
    uint32_t flag[kItems], nflag = 0;
#pragma unroll
    for (int k = 0; k < kItems; ++k) {
      const int p = p0 + k;
      uint64_t prev = (k > 0) ? seg[k - 1] : (p > 0 ? sm.u.g.seg[p - 1] : 0);
      flag[k] = (p < n) && (p == 0 || seg[k] != prev);
      nflag += flag[k];
    }
    uint32_t tot;
    uint32_t run = block_excl_scan<uint32_t>(nflag, tot, sm.scan32);
    U = tot;
#pragma unroll
    for (int k = 0; k < kItems; ++k)
      if (flag[k]) { sm.uniq[run] = seg[k]; sm.cnt[run] = (uint32_t)(p0 + k); ++run; }
    __syncthreads();
    uint32_t cs[kItems];
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
      const uint32_t r = p0 + j;
      cs[j] = (r < U) ? ((r + 1 < U ? sm.cnt[r + 1] : (uint32_t)n) - sm.cnt[r]) : 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kItems; ++j)
      if (p0 + j < (int)U) sm.cnt[p0 + j] = cs[j];
    __syncthreads();
  }

  // ---- 6. stream widths (codec.width_for == bit length of the OR) and size
  uint32_t cnt_or = 0, cmax_dummy = 0;
  uint64_t del_or = 0;
  uint32_t cloc[kItems], csum = 0;
  (void)cmax_dummy;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t r = p0 + j;
    cloc[j] = 0;
    if (!err && r < U) {
      cloc[j] = sm.cnt[r];
      cnt_or |= cloc[j];
      del_or |= sm.uniq[r] - (r ? sm.uniq[r - 1] : 0ull);
      csum += cloc[j];
    }
  }
  uint32_t red[5] = {(uint32_t)off_or, (uint32_t)(off_or >> 32), cnt_or, (uint32_t)del_or,
                     (uint32_t)(del_or >> 32)};
  block_or<5>(red, sm.red);
  const uint32_t w_off = bitlen64((uint64_t)red[0] | ((uint64_t)red[1] << 32));
  const uint32_t w_cnt = bitlen32(red[2]);
  const uint32_t w_del = bitlen64((uint64_t)red[3] | ((uint64_t)red[4] << 32));
  const uint32_t w_rank = PRES ? (uint32_t)bitlen32((uint32_t)(n - 1)) : 0u;
  const uint64_t Ld = ((uint64_t)U * w_del + 7) >> 3;
  const uint64_t Lc = ((uint64_t)U * w_cnt + 7) >> 3;
  const uint64_t Lo = ((uint64_t)n * w_off + 7) >> 3;
  const uint64_t Lr = PRES ? (((uint64_t)n * w_rank + 7) >> 3) : 0;
  const uint64_t L = err ? 0 : (uint64_t)H + Ld + Lc + Lo + Lr;


  // ---- 7. order the offset (and rank) stream
  if (passA) {
    const bool need = PRES || w_off != 0;
    if (!need) {
      path = 0;
    } else if (!PRES && sumb <= 16 && ((uint64_t)U << sumb) <= 65536) {
      // pass B: ranks of (segment rank, offset) composites
      path = 1;
      const uint32_t range = U << sumb;
      const int nw = (int)((range + 31) >> 5);
      bm_zero(sm.u.b.bm, nw);
      reinterpret_cast<uint4*>(sm.u.b.cnt2)[tid] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      uint32_t c[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k) {
        c[k] = (srank[k] << sumb) | (uint32_t)off[k];
        if (p0 + k < n) atomicOr(&sm.u.b.bm[c[k] >> 5], 1u << (c[k] & 31));
      }
      __syncthreads();
      const uint32_t nd = bm_prefix(sm.u.b.bm, sm.u.b.wp, nw, sm.scan32);
      __syncthreads();
      uint32_t cr[kItems], t2[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (p0 + k < n) {
          cr[k] = bm_rank(sm.u.b.bm, sm.u.b.wp, c[k]);
          t2[k] = atomicAdd(&sm.u.b.cnt2[cr[k]], 1u);
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
      for (int k = 0; k < kItems; ++k)
        if (p0 + k < n) pos[k] = sm.u.b.cnt2[cr[k]] + t2[k];
      __syncthreads();
    } else if (!PRES && w_cnt <= 6) {
      // small groups: rank by comparison inside each segment's group
      path = 2;
      uint32_t tot;
      uint32_t ex = block_excl_scan<uint32_t>(csum, tot, sm.scan32);
#pragma unroll
      for (int j = 0; j < kItems; ++j) {
        if (p0 + j < (int)U) sm.u.c.segstart[p0 + j] = (uint16_t)ex;
        ex += cloc[j];
      }
      __syncthreads();
      uint32_t g0[kItems];
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (p0 + k < n) {
          g0[k] = sm.u.c.segstart[srank[k]];
          sm.u.c.tmp[g0[k] + tie[k]] = off[k];
        }
      __syncthreads();
#pragma unroll
      for (int k = 0; k < kItems; ++k)
        if (p0 + k < n) {
          const uint32_t gs = sm.cnt[srank[k]], me = g0[k] + tie[k];
          uint32_t r = 0;
          for (uint32_t j = g0[k]; j < g0[k] + gs; ++j) {
            const uint64_t o = sm.u.c.tmp[j];
            r += (o < off[k]) || (o == off[k] && j < me);
          }
          pos[k] = g0[k] + r;
        }
      __syncthreads();
    } else {
      // stable LSD over (segment rank, offset) with 6-bit digits
      path = 3;
      const uint32_t srbits = (uint32_t)bitlen32(U - 1);
      const uint32_t total_bits = sumb + srbits;
      for (uint32_t s = 0; s < total_bits; s += 6) {
        const int dlen = (int)min(6u, total_bits - s);
        uint32_t dig[kItems], np[kItems];
#pragma unroll
        for (int k = 0; k < kItems; ++k) {
          uint64_t v = s < sumb ? shr64(off[k], s) : (uint64_t)(srank[k] >> (s - sumb));
          if (s < sumb && s + dlen > sumb) v |= (uint64_t)srank[k] << (sumb - s);
          dig[k] = (uint32_t)(v & ((1u << dlen) - 1u));
        }
        lsd_ranks(dig, dlen, n, p0, sm.u.l.bm, sm.u.l.wp, sm.scan32, np);
#pragma unroll
        for (int k = 0; k < kItems; ++k)
          if (p0 + k < n) {
            sm.u.l.off[np[k]] = off[k];
            sm.u.l.sr[np[k]] = (uint16_t)srank[k];
            sm.u.l.rk[np[k]] = (uint16_t)rk[k];
          }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < kItems; ++k)
          if (p0 + k < n) {
            off[k] = sm.u.l.off[p0 + k];
            srank[k] = sm.u.l.sr[p0 + k];
            rk[k] = sm.u.l.rk[p0 + k];
          }
        __syncthreads();
      }
#pragma unroll
      for (int k = 0; k < kItems; ++k) pos[k] = p0 + k;
    }
  }

  BlkRec* rec = reinterpret_cast<BlkRec*>(P.rec) + blk;
  if (tid == 0) rec->path = (uint8_t)(err ? 5 : 4);  // diagnostics: gpzb_encode_path_counts
  if (err) continue;  // cannot happen: K1.5 routes error blocks elsewhere

  // ---- 9. bit-pack header + streams into the realigned stage
  if (rec->side_off + ((L + 15) & ~15ull) > P.side_cap) {
    // the caller's side buffer is too small: report the bytes K1.5 reserved
    // (the host grows the buffer and encodes again); nothing is written
    if (tid == 0) atomicMax(&R->side_need, R->side_bytes);
    continue;
  }
  uint8_t* dst = P.side + rec->side_off;  // 16B aligned
  const uint32_t al = 0;
  const uint32_t nbytes = al + (uint32_t)L;
  const uint32_t nch = (nbytes + 15) >> 4;
  uint32_t* st = sm.u.stage;
  for (uint32_t c = tid; c < nch; c += kThreads) reinterpret_cast<uint4*>(st)[c] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  const uint64_t base = 8ull * al;
  if (tid < 32) {
    // header fields, one per lane (container.serialize_block, container.py:107-121)
    int f = lane;
    uint64_t bpos = 0, val = 0;
    bool act = true;
    if (f == 0) { bpos = 0; val = (uint32_t)n; }
    else if (f == 1) { bpos = 4; val = U; }
    else if (f < 2 + 4 * D) {
      const int a = (f - 2) >> 2, which = (f - 2) & 3;
      const uint64_t ab = 8 + (uint64_t)a * (2 * S + 5);
      const AxisGeo& g = sm.geo[a];
      if (which == 0) { bpos = ab; val = F64 ? (uint64_t)__double_as_longlong(g.lo) : (uint64_t)__float_as_uint((float)g.lo); }
      else if (which == 1) { bpos = ab + S; val = F64 ? (uint64_t)__double_as_longlong(g.hi) : (uint64_t)__float_as_uint((float)g.hi); }
      else if (which == 2) { bpos = ab + 2 * S; val = g.b; }
      else { bpos = ab + 2 * S + 1; val = (uint32_t)g.N; }
    } else if (f < 2 + 4 * D + (PRES ? 4 : 3)) {
      const int wi = f - 2 - 4 * D;
      bpos = 8 + (uint64_t)D * (2 * S + 5) + wi;
      val = wi == 0 ? w_del : wi == 1 ? w_cnt : wi == 2 ? w_off : w_rank;
    } else {
      act = false;
    }
    if (act) or_bits(st, base + 8 * bpos, val);
  }
  const uint64_t bd = base + 8ull * H;
  const uint64_t bc = bd + 8ull * Ld;
  const uint64_t bo = bc + 8ull * Lc;
  const uint64_t br = bo + 8ull * Lo;
#pragma unroll
  for (int j = 0; j < kItems; ++j) {
    const uint32_t r = p0 + j;
    if (r < U) {
      if (w_del) or_bits(st, bd + (uint64_t)r * w_del, sm.uniq[r] - (r ? sm.uniq[r - 1] : 0ull));
      if (w_cnt) or_bits(st, bc + (uint64_t)r * w_cnt, cloc[j]);
    }
  }
#pragma unroll
  for (int k = 0; k < kItems; ++k)
    if (p0 + k < n) {
      if (w_off) or_bits(st, bo + (uint64_t)pos[k] * w_off, off[k]);
      if (PRES && w_rank) or_bits(st, br + (uint64_t)pos[k] * w_rank, rk[k]);
    }
  __syncthreads();

  // ---- 10. stage -> side buffer (16B aligned, whole chunks)
  for (uint32_t c = tid; c < nch; c += kThreads)
    reinterpret_cast<uint4*>(dst)[c] = reinterpret_cast<const uint4*>(st)[c];
  if (tid == 0) {
    rec->side_len = (uint32_t)L;
    P.status[blk] = L;  // payload length for the K3 scan
  }
  }
}

}  // namespace gpzb
