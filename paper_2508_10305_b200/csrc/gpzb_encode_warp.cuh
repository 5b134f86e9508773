// K2p: warp-per-block encoder for offset-free blocks.
//
// When every axis has log2 m == 0 (one bin per segment, so the offset stream
// is empty and the (seg, off) sort is the segment sort alone) and Π N <=
// 16384, a block's whole state — presence bitmap, word prefixes, run lengths,
// unique ids, the payload stage — fits ~10 KB, so one warp can own a block:
// 32 particles per lane, warp scans and __syncwarp instead of CTA barriers.
// Same steps and bytes as the CTA encoder (gpzb_encode_narrow.cuh):
//
//   quantize (certified reciprocal, quantizer.py:142-191) -> seg per particle
//   presence bitmap over [0, Π N) -> word prefixes -> rank of each particle's
//   segment; RED.ADD per rank -> run lengths; unique ids by rank
//   (rle_encode(sort(seg)), codec.py:53-79, blocksort.py:17-28)
//   widths by OR (codec.width_for), payload length -> sizes[blk]
//   header + delta + count streams bit-packed in shared memory
//   (container.serialize_block, container.py:102-121), 16-byte stores into
//   the block's staging slot for K3.
#pragma once

#include "gpzb_encode_narrow.cuh"

namespace gpzb {

#ifndef GPZB_K2P_WARPS
#define GPZB_K2P_WARPS 4
#endif
#ifndef GPZB_K2P_MINB
#define GPZB_K2P_MINB 5
#endif
#ifndef GPZB_K2P_L2PF
#define GPZB_K2P_L2PF 1  // blocks ahead (in this warp's sequence) to bulk-prefetch into L2; 0 = off
#endif
constexpr int kWarpEncWarps = GPZB_K2P_WARPS;
// payload <= 74 + 1024 * (14 + 11) / 8 + 2 = 3,276 bytes (widths <= bitlen(16383), bitlen(1024))
constexpr int kWarpStageWords = 832;
struct WarpEncSmem {
  // the geometry record (128 B) and stored bounds (<= 48 B) of this and the
  // warp's next block, brought in by 4-byte cp.async one block ahead
  __align__(16) uint32_t recw[2][32 + 12];
  __align__(16) uint32_t bm[kWarpStageWords];  // presence bitmap (<= 512 words), then the payload stage
  uint16_t wp[kWarpEncMaxPN / 32];             // set bits before each bitmap word
  __align__(16) uint32_t cnt[kMaxBs];          // run length per segment rank
  uint16_t uniqp[kMaxBs + 2];                  // [0] = 0 sentinel, [r + 1] = unique id r
};
constexpr size_t kWarpEncSmemBytes = sizeof(WarpEncSmem) * kWarpEncWarps;

template <int D, bool F64, bool LIST>
__global__ void __launch_bounds__(32 * kWarpEncWarps, GPZB_K2P_MINB) k_encode_warp(const EncParams P) {
  using T = typename std::conditional<F64, double, float>::type;
  constexpr int S = F64 ? 8 : 4;
  constexpr uint32_t H = 8 + D * (2 * S + 5) + 3;  // block header bytes (container.py:62-67)
  constexpr int VE = 16 / S;                        // coordinates per 16-byte load
  extern __shared__ __align__(16) unsigned char esm[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  WarpEncSmem& sm = reinterpret_cast<WarpEncSmem*>(esm)[wid];

  uint4 raw[D][4 / VE];      // 16-byte loads of the chunk being (or about to be) quantized
  uint64_t raw_blk = ~0ull;  // block whose chunk 0 sits in raw
  const uint64_t stride = (uint64_t)gridDim.x * kWarpEncWarps;
  // the geometry record (one word per lane) and the stored block bounds of
  // the warp's next block are copied to shared memory one block ahead, so no
  // block starts (or writes its header) waiting on global memory
  static_assert(sizeof(BlkRec) == 128, "one record word per lane");
  constexpr int kBW = 2 * D * (S / 4);  // bound words per block
  auto prefetch_rec = [&](uint64_t b, int buf) {
    if (b < P.nblocks) {
      cp_async4(&sm.recw[buf][lane], reinterpret_cast<const uint32_t*>(P.rec + b) + lane);
      if (lane < kBW) cp_async4(&sm.recw[buf][32 + lane], reinterpret_cast<const uint32_t*>(P.bounds) + b * kBW + lane);
    }
    cp_async_commit();
  };
  // LIST (the velocity field: fewer than half the blocks are this kernel's):
  // K1.5's list of them, entry item + 2 stride read one block ahead of its
  // use; else every block in order, skipping the others.  Both variants are
  // launched; the one that does not match the device-side count exits.
  const uint32_t nlist = *reinterpret_cast<volatile const uint32_t*>(&P.res->warp_count);
  if ((2ull * nlist < P.nblocks) != LIST) return;
  // one block: blk, with nxt the block this warp encodes next (>= nblocks: none)
  auto encode_one = [&](const uint64_t blk, const uint64_t nxt, const int buf) {
    const BlkRec* rec = P.rec + blk;
    cp_async_wait_all();
    __syncwarp();
    const uint32_t* recw = sm.recw[buf];
    prefetch_rec(nxt, buf ^ 1);
    if ((reinterpret_cast<const uint8_t*>(recw)[offsetof(BlkRec, kind)]) != KIND_WARP) return;  // dense: warp-uniform skip
    const uint64_t first = blk * (uint64_t)P.bs;
#if GPZB_K2P_L2PF
    // the next block's coordinates into L2 (one bulk prefetch per axis): its
    // loads then wait on L2, not HBM, while this block ranks and packs
    if (lane < D && nxt < P.nblocks && P.vec) {
      const uint64_t nf = nxt * (uint64_t)P.bs;
      const uint32_t nbytes = (uint32_t)((min((uint64_t)P.bs, P.count - nf) * S) & ~15ull);
      if (nbytes)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<const T*>(P.axes[lane]) + nf),
                     "r"(nbytes)
                     : "memory");
    }
#endif
    const uint32_t PN = recw[offsetof(BlkRec, PN) / 4];
    const uint32_t nw = (PN + 31) >> 5;
    // ---- zero the bitmap and the run counters
    for (uint32_t w = lane; w < (nw + 3) >> 2; w += 32) reinterpret_cast<uint4*>(sm.bm)[w] = make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int j = 0; j < kMaxBs / 128; ++j) reinterpret_cast<uint4*>(sm.cnt)[j * 32 + lane] = make_uint4(0, 0, 0, 0);
    if (lane == 0) sm.uniqp[0] = 0;
    double lo[D], rinv[D];
    uint32_t Nst[D];
    {
      uint32_t st = 1;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        constexpr int kLo = offsetof(BlkRec, lo) / 4, kRi = offsetof(BlkRec, rinv) / 4, kN = offsetof(BlkRec, N) / 4;
        lo[a] = __hiloint2double((int)recw[kLo + 2 * a + 1], (int)recw[kLo + 2 * a]);
        rinv[a] = __hiloint2double((int)recw[kRi + 2 * a + 1], (int)recw[kRi + 2 * a]);
        Nst[a] = st;
        st *= recw[kN + a];
      }
    }
    __syncwarp();
    // ---- quantize: chunk c, lane l -> particles c*128 + 4l .. +3 (b == 0: q_a is the segment digit)
    uint32_t segpk[kMaxBs / 64];  // 32 segment ids, two 16-bit ids per register
    // software pipeline: chunk c + 1's loads are in flight while chunk c
    // quantizes; chunk 0 was prefetched while the previous block packed
    if (raw_blk != blk) {
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(P.axes[a]) + first + 4 * lane);
#pragma unroll
        for (int v = 0; v < 4 / VE; ++v) raw[a][v] = __ldcs(base + v);
      }
    }
#pragma unroll
    for (int c = 0; c < kMaxBs / 128; ++c) {
      T x[D][4];
#pragma unroll
      for (int a = 0; a < D; ++a) {
#pragma unroll
        for (int v = 0; v < 4 / VE; ++v) {
          const T* e = reinterpret_cast<const T*>(&raw[a][v]);
#pragma unroll
          for (int j = 0; j < VE; ++j) x[a][v * VE + j] = e[j];
        }
      }
      if (c + 1 < kMaxBs / 128) {
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(P.axes[a]) + first +
                                                             (c + 1) * 128 + 4 * lane);
#pragma unroll
          for (int v = 0; v < 4 / VE; ++v) raw[a][v] = __ldcs(base + v);
        }
      }
      uint32_t seg[4] = {0, 0, 0, 0};
      uint32_t mn = ~0u, mx = 0u;  // extremes of the low words: 0 or ~0 flags a possible failure
#pragma unroll
      for (int a = 0; a < D; ++a) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          // certified reciprocal quantizer with the FMA nudge (K2s, DESIGN.md
          // §3.1): t == 0 gives r = nudge, whose low word passes
          const double t = __dsub_rn((double)x[a][k], lo[a]);
          const double r = __fma_rn(t, rinv[a], __longlong_as_double((long long)kCertNudgeBits));
          const uint32_t rl = (uint32_t)__double2loint(r);
          const uint32_t q = (uint32_t)__double2loint(__dadd_rz(r, 4503599627370496.0));
          mn = min(mn, rl);
          mx = max(mx, rl);
          seg[k] += q * Nst[a];
        }
      }
      const bool bad = mn == 0u || mx == ~0u;
      if (__any_sync(kFull, bad)) {
        if (bad) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t so = redo_exact<D, T>(x[0][k], D > 1 ? x[D > 1 ? 1 : 0][k] : T(0),
                                                 D > 2 ? x[D > 2 ? 2 : 0][k] : T(0), rec);
            seg[k] = (uint32_t)(so >> 32);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) red_or_shared(&sm.bm[seg[k] >> 5], 1u << (seg[k] & 31));
      segpk[2 * c] = seg[0] | (seg[1] << 16);
      segpk[2 * c + 1] = seg[2] | (seg[3] << 16);
    }
    // prefetch the next block's chunk 0 (full blocks: always in bounds)
    raw_blk = ~0ull;
    if (nxt < P.nblocks && (nxt + 1) * (uint64_t)P.bs <= P.count) {
      raw_blk = nxt;
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const uint4* base = reinterpret_cast<const uint4*>(reinterpret_cast<const T*>(P.axes[a]) +
                                                           raw_blk * (uint64_t)P.bs + 4 * lane);
#pragma unroll
        for (int v = 0; v < 4 / VE; ++v) raw[a][v] = __ldcs(base + v);
      }
    }
    __syncwarp();
    // ---- word prefixes: lane l owns bitmap words [16l, 16l + 16)
    uint32_t U;
    {
      uint32_t local = 0;
      const uint32_t w0 = 16 * lane;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (w0 + 4 * j < nw) {
          const uint4 q = reinterpret_cast<const uint4*>(sm.bm)[4 * lane + j];
          local += __popc(q.x) + __popc(q.y) + __popc(q.z) + __popc(q.w);
        }
      }
      uint32_t incl = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += y;
      }
      U = __shfl_sync(kFull, incl, 31);
      uint32_t run = incl - local;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (w0 + 4 * j < nw) {
          const uint4 q = reinterpret_cast<const uint4*>(sm.bm)[4 * lane + j];
          const uint32_t a = run, b = a + __popc(q.x), c = b + __popc(q.y), d = c + __popc(q.z);
          reinterpret_cast<uint2*>(sm.wp)[4 * lane + j] = make_uint2(a | (b << 16), c | (d << 16));
          run = d + __popc(q.w);
        }
      }
    }
    __syncwarp();
    // ---- ranks -> run lengths and unique ids
#pragma unroll
    for (int i = 0; i < kMaxBs / 64; ++i) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t sg = (segpk[i] >> (16 * h)) & 0xffffu;
        const uint32_t w = sg >> 5;
        const uint32_t rk = (uint32_t)sm.wp[w] + __popc(sm.bm[w] & ((1u << (sg & 31)) - 1u));
        atomicAdd(&sm.cnt[rk], 1u);  // no return value used: RED
        sm.uniqp[rk + 1] = (uint16_t)sg;
      }
    }
    __syncwarp();
    // ---- widths (width_for == bit length of the OR) and the payload length
    uint32_t c_or = 0, d_or = 0;
    for (uint32_t r = lane; r < U; r += 32) {
      c_or |= sm.cnt[r];
      d_or |= (uint32_t)sm.uniqp[r + 1] - (uint32_t)sm.uniqp[r];
    }
    c_or = __reduce_or_sync(kFull, c_or);
    d_or = __reduce_or_sync(kFull, d_or);
    const uint32_t w_cnt = bitlen32(c_or), w_del = bitlen32(d_or);
    const uint32_t Ld = (U * w_del + 7) >> 3, Lc = (U * w_cnt + 7) >> 3;
    const uint32_t L = H + Ld + Lc;
    if (lane == 0) {
      P.status[blk] = L;  // payload length for the K3 scan
      P.rec[blk].path = 0;  // diagnostics: gpzb_encode_path_counts
    }
    // ---- bit-pack into the stage (the bitmap is dead now)
    uint32_t* st = sm.bm;
    const uint32_t nquads = (L + 15) >> 4;
    for (uint32_t w = lane; w < nquads; w += 32) reinterpret_cast<uint4*>(st)[w] = make_uint4(0, 0, 0, 0);
    __syncwarp();
    {
      // block header fields, one per lane (container.serialize_block, container.py:107-121)
      const int f = lane;
      uint32_t bpos = 0;
      uint64_t val = 0;
      bool act = true;
      // the stored bounds and N of this lane's field, from the prefetched words
      const int fa = f >= 2 && f < 2 + 4 * D ? (f - 2) >> 2 : 0, fw = (f - 2) & 3;
      const int bw = (2 * fa + (fw & 1)) * (S / 4);
      const uint32_t b_lo = recw[32 + bw], b_hi = recw[32 + (S / 4 == 2 ? bw + 1 : bw)];
      const uint32_t n_a = recw[offsetof(BlkRec, N) / 4 + fa];
      if (f == 0) { bpos = 0; val = (uint32_t)kMaxBs; }
      else if (f == 1) { bpos = 4; val = U; }
      else if (f < 2 + 4 * D) {
        const int a = (f - 2) >> 2, which = (f - 2) & 3;
        const uint32_t ab = 8 + a * (2 * S + 5);
        if (which < 2) {
          bpos = ab + which * S;
          if constexpr (F64) val = (uint64_t)b_hi << 32 | b_lo;
          else val = b_lo;
        } else if (which == 2) { bpos = ab + 2 * S; val = 0; }  // log2 m == 0
        else { bpos = ab + 2 * S + 1; val = n_a; }
      } else if (f < 2 + 4 * D + 3) {
        const int wi = f - 2 - 4 * D;
        bpos = 8 + D * (2 * S + 5) + wi;
        val = wi == 0 ? w_del : wi == 1 ? w_cnt : 0u;  // w_off == 0
      } else {
        act = false;
      }
      if (act) or_bits(st, 8ull * bpos, val);
    }
    {
      const uint64_t bd = 8ull * H, bc = bd + 8ull * Ld;
      for (uint32_t r0 = 4 * lane; r0 < U; r0 += 128) {
        uint64_t dv = 0, cv = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t r = r0 + j;
          if (r < U) {
            dv |= (uint64_t)((uint32_t)sm.uniqp[r + 1] - (uint32_t)sm.uniqp[r]) << (j * w_del);
            cv |= (uint64_t)sm.cnt[r] << (j * w_cnt);
          }
        }
        if (w_del) or_bits(st, bd + (uint64_t)r0 * w_del, dv);
        if (w_cnt) or_bits(st, bc + (uint64_t)r0 * w_cnt, cv);
      }
    }
    __syncwarp();
    uint4* slot = reinterpret_cast<uint4*>(P.staging + blk * (uint64_t)kSlotBytes);
    for (uint32_t w = lane; w < nquads; w += 32) __stcg(slot + w, reinterpret_cast<const uint4*>(st)[w]);
    __syncwarp();  // the next block reuses the shared state
  };
  int buf = 0;
  if constexpr (LIST) {
    auto entry = [&](uint64_t j) -> uint64_t { return j < nlist ? (uint64_t)P.warp_list[j] : ~0ull; };
    uint64_t item = (uint64_t)blockIdx.x * kWarpEncWarps + wid;
    uint64_t blk = entry(item), nxt = entry(item + stride), nn = ~0ull;
    prefetch_rec(blk, 0);
    for (; item < nlist; item += stride, buf ^= 1, blk = nxt, nxt = nn) {
      nn = entry(item + 2 * stride);
      encode_one(blk, nxt, buf);
    }
  } else {
    const uint64_t blk0 = (uint64_t)blockIdx.x * kWarpEncWarps + wid;
    prefetch_rec(blk0, 0);
    for (uint64_t blk = blk0; blk < P.nblocks; blk += stride, buf ^= 1) encode_one(blk, blk + stride, buf);
  }
}

}  // namespace gpzb
