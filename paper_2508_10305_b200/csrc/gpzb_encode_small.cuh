// K2s: persistent CTA encoder for full float32 blocks with at most four
// offset bits per particle (Σ log2 m <= 4, Π N <= 2^16) — the bulk of
// HACC-like snapshots at rel-eb 1e-3 (velocities: log2 m = 1 or 2 per axis;
// positions: log2 m = 0).  Same bytes as pipeline._encode_block
// (pipeline.py:38-70).  One CTA of 128 threads per block, 8 particles and 8
// runs per thread, CTAs persistent over K1.5's block list.
//
// Per block (9 barriers with offsets, 7 without):
//   quantize (certified reciprocal, quantizer.py:142-191) -> 32-bit key
//        seg | off << 16 per particle                                  | Bz
//        (the previous block's stage is out; the next block's bulk copy starts)
//   RED.OR into a presence bitmap over [0, Π N)                        | B1
//   word prefixes of the bitmap (up to four 16-byte groups per thread) | B2 B3
//   segment rank r of each particle = prefix + popc below its bit; the
//        rank's counter word gets 1 << 4*off (ATOMS: the returned nibble is
//        the particle's tie index among identical (seg, off) pairs); the
//        unique id of rank r goes to uniq[r + 1]                      | B4
//        == rle_encode(sort_block(...)) (codec.py:53-79, blocksort.py:17-28)
//   thread t owns runs 8t..8t+7: count = nibble sum of the counter word,
//        delta = uniq[r + 1] - uniq[r] (delta_encode, codec.py:93-100);
//        one scan of the counts (run starts) + OR of the widths
//        (width_for, codec.py:107-112)                                | B5
//   header + delta + count streams bit-packed into the shared stage
//        (serialize_block / pack_fixed, container.py:102-121,
//        codec.py:115-129); run starts published                      | B6
//   each particle's place in (seg, off) order = run start + particles of
//        its run with a smaller offset (nibble sum below its nibble) + tie;
//        its offset goes there                                        | B7
//   the offset stream packed from the ordered offsets                 | B8
//   the stage to the block's staging slot (K3 concatenates), zeroed behind
//        the copy (it is the next block's bitmap)
//
// A (segment, offset) pair held by >= 16 particles overflows its nibble; the
// counts then sum to less than 1024 and the block is handed to the general
// CTA encoder K2 (gpzb_encode_narrow.cuh) through its list — exact in every
// case.
#pragma once

#include "gpzb_encode_narrow.cuh"

namespace gpzb {

#ifndef GPZB_K2S_MINB
#define GPZB_K2S_MINB 7
#endif
#ifndef GPZB_K2S0_MINB
#define GPZB_K2S0_MINB 7
#endif
constexpr int kST = 128;               // K2s threads per block
constexpr int kSW = kST / 32;          // warps per block
constexpr int kSP = kMaxBs / kST;      // particles (and runs) per thread
// Π N <= 2^15 (t = 32 in 3D: N_a <= 32 per axis), so the presence bitmap and
// the stage it becomes are 4 KB; with 30 KB of shared memory per CTA seven
// CTAs (28 warps) fit an SM
static_assert(kSmallMaxPN == 32768, "bitmap sizing below");
// payload <= 50 + 1024 * 16 / 8 + 1024 * 11 / 8 (no offsets) = 3,506 bytes
// (with offsets: counts <= 8 bits, offsets <= 4 bits: 3,634 bytes)
constexpr int kSmallStageWords = 1024;
// particles of lane l in warp w: two 4-particle groups of the 32-particle
// chunk l, groups g0 = (l + 2w) mod 8 and g0 + 1 (mod 8). One quantize step of
// a warp spans the whole block (stride 32), which spreads spatially ordered
// same-segment particles (LiDAR scan lines) across the counter atomics, and
// each 8-lane phase of a 16-byte load covers all 32 banks
__device__ __forceinline__ uint32_t small_group(uint32_t lane, uint32_t wid, uint32_t h) {
  return 8u * lane + ((lane + 2u * wid + h) & 7u);  // float4 index
}
__device__ __forceinline__ uint32_t small_pidx(uint32_t lane, uint32_t wid, int k) {
  return 4u * small_group(lane, wid, (uint32_t)k >> 2) + ((uint32_t)k & 3u);
}

template <int D, bool HAS_OFF>
struct SmallSmem {
  // this block's coordinates and geometry record, brought in by one bulk
  // copy (TMA, cp.async.bulk) issued while the previous block was encoded
  __align__(128) float x[D][kMaxBs];
  __align__(16) BlkRec rec;
  unsigned long long mbar;               // completion barrier of that copy
  uint32_t blk;                          // the block it holds
  __align__(16) uint32_t scan[2][kSW];   // warp totals of the two block scans
  __align__(16) uint32_t orw[4];         // width ORs: counts, deltas, offsets
  // presence bitmap over segments (quantize .. ranks), then the payload stage
  __align__(16) uint32_t bm[kSmallMaxPN / 32];
  // set bits before each bitmap word (prefix .. ranks), then run starts
  __align__(16) uint16_t wp[kMaxBs + kMaxBs / 2];  // >= kSmallMaxPN / 32 prefixes; run starts (u16) + offsets (u8)
  // per segment rank r: counter word cnt[r] (offsets 0-7, one nibble each)
  // and cnt[1024 + r] (offsets 8-15); offset-free blocks: the run length
  __align__(16) uint32_t cnt[HAS_OFF ? 2 * kMaxBs : kMaxBs];
  __align__(16) uint16_t uniq[kMaxBs + 8];  // [0] = 0 sentinel, [r + 1] = unique id of rank r
};
static_assert(kSmallStageWords <= kSmallMaxPN / 32, "the stage reuses the bitmap");


// Exclusive scan of one value per thread over the (kSW-warp) CTA with a
// single barrier.  `ws` (16-byte aligned) is not rewritten before a later
// barrier.
__device__ __forceinline__ uint32_t small_excl_scan(uint32_t v, uint32_t& total, uint32_t* ws) {
  static_assert(kSW == 4, "one 16-byte read of the warp totals");
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  const uint4 a = *reinterpret_cast<const uint4*>(ws);
  const uint32_t b1 = a.x, b2 = b1 + a.y, b3 = b2 + a.z;
  total = b3 + a.w;
  const uint32_t before = wid == 0 ? 0u : (wid == 1 ? b1 : (wid == 2 ? b2 : b3));
  return before + x - v;
}

// Sum of the nibbles of a counter word (each nibble <= 15).  Exact when the
// sum is <= 15 (one multiply): runs of <= 15 particles.
__device__ __forceinline__ uint32_t nib_sum1(uint32_t x) { return (x * 0x11111111u) >> 28; }
// Exact for any word (byte-wise fold first).
__device__ __forceinline__ uint32_t nib_sum8(uint32_t x) {
  const uint32_t s = (x & 0x0f0f0f0fu) + ((x >> 4) & 0x0f0f0f0fu);  // bytes <= 30
  return (s * 0x01010101u) >> 24;
}

__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One bulk copy of block `blk`'s coordinates and geometry record into shared
// memory, completing on the CTA's mbarrier (one elected thread).
template <int D, bool HAS_OFF>
__device__ __forceinline__ void small_fetch(const EncParams& P, SmallSmem<D, HAS_OFF>& s, uint32_t blk) {
  mbar_expect_tx(reinterpret_cast<uint64_t*>(&s.mbar), D * kMaxBs * 4 + (uint32_t)sizeof(BlkRec));
#pragma unroll
  for (int a = 0; a < D; ++a)
    bulk_g2s(s.x[a], reinterpret_cast<const float*>(P.axes[a]) + (uint64_t)blk * kMaxBs, kMaxBs * 4,
             reinterpret_cast<uint64_t*>(&s.mbar));
  bulk_g2s(&s.rec, P.rec + blk, sizeof(BlkRec), reinterpret_cast<uint64_t*>(&s.mbar));
}

template <int D, bool HAS_OFF>
__global__ void __launch_bounds__(kST, HAS_OFF ? GPZB_K2S_MINB : GPZB_K2S0_MINB) k_encode_small(const EncParams P) {
  static_assert(kSP == 8, "thread t owns runs 8t..8t+7");
  using Smem = SmallSmem<D, HAS_OFF>;
  __shared__ Smem sm;
  constexpr uint32_t H = 8 + D * 13 + 3;  // F32 block header bytes (container.py:62-67)
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  DevResult* R = P.res;
  const uint32_t nlist = HAS_OFF ? *reinterpret_cast<volatile const uint32_t*>(&R->small_count)
                                 : *reinterpret_cast<volatile const uint32_t*>(&R->small0_count);
  if (blockIdx.x >= nlist) return;
  auto list_at = [&](uint32_t i) -> uint32_t {
    return HAS_OFF ? P.small_list[i] : P.small_list[P.nblocks - 1 - i];
  };
  const uint4 z4 = make_uint4(0, 0, 0, 0);
  // invariant at every block start: bitmap (= stage), counters and OR words are zero
  for (int i = tid; i < (int)(kSmallMaxPN / 128); i += kST) reinterpret_cast<uint4*>(sm.bm)[i] = z4;
  for (int i = tid; i < (int)(sizeof(sm.cnt) / 16); i += kST) reinterpret_cast<uint4*>(sm.cnt)[i] = z4;
  if (tid < 4) sm.orw[tid] = 0;
  if (tid == 0) {
    sm.uniq[0] = 0;
    mbar_init(reinterpret_cast<uint64_t*>(&sm.mbar), 1);
    mbar_fence_init();
    sm.blk = list_at(blockIdx.x);
    small_fetch<D, HAS_OFF>(P, sm, sm.blk);
  }
  // thread 0 keeps the list entry of the block after next in a register, read
  // one block ahead, so issuing the next bulk copy never waits on global memory
  uint32_t next_blk = (tid == 0 && blockIdx.x + gridDim.x < nlist) ? list_at(blockIdx.x + gridDim.x) : 0u;
  __syncthreads();

  const uint32_t bm_s = smem_u32(sm.bm);
  const double nudge = __longlong_as_double((long long)kCertNudgeBits);
  uint32_t phase = 0;
  for (uint32_t item = blockIdx.x; item < nlist; item += gridDim.x) {
    mbar_wait(reinterpret_cast<uint64_t*>(&sm.mbar), phase);
    phase ^= 1;
    // everything this block needs from the record, before the next bulk copy replaces it
    const uint32_t blk = sm.blk;
    const uint32_t PN = sm.rec.PN;
    const uint32_t sumb = HAS_OFF ? (uint32_t)sm.rec.sumb : 0u;
    const uint32_t w_hdr_b = HAS_OFF && lane < D ? (uint32_t)sm.rec.b[lane] : 0u;
    const uint32_t w_hdr_n = lane < D ? sm.rec.N[lane] : 0u;
    // warp 0's header lanes 2 + 4a + {0, 1} write the block's stored bounds:
    // load them now so the global-memory latency hides behind the quantizer
    uint32_t w_hdr_bound = 0;
    if (wid == 0 && lane >= 2 && lane < 2 + 4 * D && ((lane - 2) & 3) < 2)
      w_hdr_bound = __float_as_uint(
          reinterpret_cast<const float*>(P.bounds)[(uint64_t)blk * 2 * D + 2 * ((lane - 2) >> 2) + ((lane - 2) & 3)]);

    // ---- quantize -> key = seg | off << 16
    uint32_t key[kSP], off_or = 0;
    {
      uint32_t seg[kSP], off[kSP];
#pragma unroll
      for (int k = 0; k < kSP; ++k) { seg[k] = 0; off[k] = 0; }
      uint32_t mn = ~0u, mx = 0u;  // extremes of the low words: 0 or ~0 flags a possible failure
      uint32_t stride = 1, shift = 0;
      const uint32_t g0 = small_group(lane, wid, 0), g1 = small_group(lane, wid, 1);
#pragma unroll
      for (int a = 0; a < D; ++a) {
        const double lo = sm.rec.lo[a], rinv = sm.rec.rinv[a];
        const uint32_t b = HAS_OFF ? (uint32_t)sm.rec.b[a] : 0u;
        const uint32_t mks = ((1u << b) - 1u) << shift;
        float x[kSP];
        {
          const float4 v0 = reinterpret_cast<const float4*>(sm.x[a])[g0];
          const float4 v1 = reinterpret_cast<const float4*>(sm.x[a])[g1];
          x[0] = v0.x; x[1] = v0.y; x[2] = v0.z; x[3] = v0.w;
          x[4] = v1.x; x[5] = v1.y; x[6] = v1.z; x[7] = v1.w;
        }
#pragma unroll
        for (int k = 0; k < kSP; ++k) {
          // certified reciprocal quantizer (gpzb_common.cuh quantize_coord,
          // mode 0) with the nudge: r > 0 always, t == 0 gives r = nudge
          const double t = __dsub_rn((double)x[k], lo);
          const double r = __fma_rn(t, rinv, nudge);
          const uint32_t rl = (uint32_t)__double2loint(r);
          const uint32_t q = (uint32_t)__double2loint(__dadd_rz(r, 4503599627370496.0));
          mn = min(mn, rl);
          mx = max(mx, rl);
          if (HAS_OFF) {
            seg[k] += (q >> b) * stride;
            off[k] |= (q << shift) & mks;
          } else {
            seg[k] += q * stride;
          }
        }
        stride *= sm.rec.N[a];
        shift += b;
      }
      // rare (a coordinate within an ulp of a bin edge): exact division for
      // this thread's particles (identical wherever the certificate holds)
      const bool bad = mn == 0u || mx == ~0u;
      if (__any_sync(kFull, bad) && bad) {
#pragma unroll
        for (int k = 0; k < kSP; ++k) {
          auto xat = [&](int a) -> float { return sm.x[a][small_pidx(lane, wid, k)]; };
          const uint64_t so = redo_exact<D, float>(xat(0), D > 1 ? xat(D > 1 ? 1 : 0) : 0.f,
                                                   D > 2 ? xat(D > 2 ? 2 : 0) : 0.f, &sm.rec);
          seg[k] = (uint32_t)(so >> 32);
          off[k] = (uint32_t)so;
        }
      }
#pragma unroll
      for (int k = 0; k < kSP; ++k) {
        key[k] = seg[k] | (off[k] << 18);  // seg | (4 * off) << 16: the offset's nibble position
        off_or |= off[k];
      }
    }
    __syncthreads();  // Bz: coordinates and record consumed; the previous stage is out and zeroed
    if (tid == 0 && item + gridDim.x < nlist) {  // the next block's bulk copy overlaps this block's encode
      fence_proxy_async_smem();
      sm.blk = next_blk;
      small_fetch<D, HAS_OFF>(P, sm, next_blk);
      if (item + 2 * gridDim.x < nlist) next_blk = list_at(item + 2 * gridDim.x);
    }
#pragma unroll
    for (int k = 0; k < kSP; ++k) {
      const uint32_t sg = key[k] & 0xffffu;
      asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(bm_s + ((sg >> 3) & ~3u)), "r"(1u << (sg & 31)) : "memory");
    }
    __syncthreads();  // B1: presence bitmap complete

    // ---- bitmap word prefixes: thread t owns the 16-byte groups 2t and 2t + 1
    static_assert(kSmallMaxPN / 128 == 2 * kST, "two bitmap groups per thread");
    const uint32_t ng = (((PN + 31) >> 5) + 3) >> 2;  // <= 256
    uint32_t U;
    {
      const uint4 z = make_uint4(0, 0, 0, 0);
      const uint4 q0 = 2 * tid < ng ? reinterpret_cast<const uint4*>(sm.bm)[2 * tid] : z;
      const uint4 q1 = 2 * tid + 1 < ng ? reinterpret_cast<const uint4*>(sm.bm)[2 * tid + 1] : z;
      const uint32_t p0 = __popc(q0.x), p1 = __popc(q0.y), p2 = __popc(q0.z), p3 = __popc(q0.w);
      const uint32_t p4 = __popc(q1.x), p5 = __popc(q1.y), p6 = __popc(q1.z), p7 = __popc(q1.w);
      const uint32_t e0 = small_excl_scan(p0 + p1 + p2 + p3 + p4 + p5 + p6 + p7, U, sm.scan[0]);  // B2
      const uint32_t e1 = e0 + p0, e2 = e1 + p1, e3 = e2 + p2, e4 = e3 + p3, e5 = e4 + p4, e6 = e5 + p5,
                     e7 = e6 + p6;
      if (2 * tid < ng) reinterpret_cast<uint2*>(sm.wp)[2 * tid] = make_uint2(e0 | (e1 << 16), e2 | (e3 << 16));
      if (2 * tid + 1 < ng)
        reinterpret_cast<uint2*>(sm.wp)[2 * tid + 1] = make_uint2(e4 | (e5 << 16), e6 | (e7 << 16));
    }
    __syncthreads();  // B3

    // ---- segment ranks -> counters (tie index returned), unique ids
    // rk = rank | tie index << 10 | 4 * offset << 14
    uint32_t rk[kSP];
    auto rank_all = [&](auto wide_c) {
      constexpr bool WIDE = decltype(wide_c)::value;
#pragma unroll
      for (int k = 0; k < kSP; ++k) {
        const uint32_t sg = key[k] & 0xffffu, w = sg >> 5;
        const uint32_t r = (uint32_t)sm.wp[w] + __popc(sm.bm[w] & bmsk_wrap(sg));
        sm.uniq[r + 1] = (uint16_t)sg;
        if (HAS_OFF) {
          const uint32_t o4 = key[k] >> 16;  // 4 * offset
          const uint32_t sh = WIDE ? (o4 & 31u) : o4;
          const uint32_t old = atomicAdd(&sm.cnt[WIDE ? (r | (o4 >> 5) << 10) : r], 1u << sh);
          rk[k] = r | ((old >> sh) & 15u) << 10 | o4 << 14;
        } else {
          atomicAdd(&sm.cnt[r], 1u);  // result unused: RED
          rk[k] = r;
        }
      }
    };
    if (HAS_OFF && sumb > 3) rank_all(std::true_type{});  // counters in both words of a rank
    else rank_all(std::false_type{});
    __syncthreads();  // B4: bitmap and word prefixes dead

    // ---- runs 8t..8t+7: counts, deltas; run starts (scan) and stream widths (OR)
    const bool wide = sumb > 3;  // counters in both words of a rank
    uint32_t dc[kSP], csum = 0, c_or = 0, d_or = 0;
    {
      const uint4 u4 = reinterpret_cast<const uint4*>(sm.uniq)[tid];
      const uint32_t u[9] = {u4.x & 0xffffu, u4.x >> 16, u4.y & 0xffffu, u4.y >> 16,
                             u4.z & 0xffffu, u4.z >> 16, u4.w & 0xffffu, u4.w >> 16, (uint32_t)sm.uniq[kSP * tid + kSP]};
      uint32_t cc[kSP];
      {
        const uint4 a0 = reinterpret_cast<const uint4*>(sm.cnt)[2 * tid];
        const uint4 a1 = reinterpret_cast<const uint4*>(sm.cnt)[2 * tid + 1];
        const uint32_t cw[kSP] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
        if (!HAS_OFF) {
#pragma unroll
          for (int j = 0; j < kSP; ++j) cc[j] = cw[j];
          reinterpret_cast<uint4*>(sm.cnt)[2 * tid] = z4;  // counters are dead (offset-free blocks)
          reinterpret_cast<uint4*>(sm.cnt)[2 * tid + 1] = z4;
        } else if (wide) {
          const uint4 b0 = reinterpret_cast<const uint4*>(sm.cnt)[256 + 2 * tid];
          const uint4 b1 = reinterpret_cast<const uint4*>(sm.cnt)[256 + 2 * tid + 1];
          const uint32_t cw2[kSP] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
          for (int j = 0; j < kSP; ++j) cc[j] = nib_sum8(cw[j]) + nib_sum8(cw2[j]);
        } else {
#pragma unroll
          for (int j = 0; j < kSP; ++j) cc[j] = nib_sum8(cw[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < kSP; ++j) {
        // ranks >= U: the counter words are zero; their uniq entries are stale
        const uint32_t c = cc[j];
        const uint32_t d = (uint32_t)(kSP * tid + j) < U ? u[j + 1] - u[j] : 0u;
        csum += c;
        c_or |= c;
        d_or |= d;
        dc[j] = d | (c << 16);
      }
    }
    // the bitmap becomes the payload stage: zero the words it used
    if (2 * tid < ng) reinterpret_cast<uint4*>(sm.bm)[2 * tid] = z4;
    if (2 * tid + 1 < ng) reinterpret_cast<uint4*>(sm.bm)[2 * tid + 1] = z4;
    uint32_t total, ex;
    {
      const uint32_t r0 = __reduce_or_sync(kFull, c_or), r1 = __reduce_or_sync(kFull, d_or);
      const uint32_t r2 = HAS_OFF ? __reduce_or_sync(kFull, off_or) : 0u;
      const uint32_t mine = lane == 0 ? r0 : (lane == 1 ? r1 : r2);
      red_or_shared_if(lane < 3 && mine != 0, &sm.orw[lane < 3 ? lane : 0], mine);
      ex = small_excl_scan(csum, total, sm.scan[1]);  // B5
    }
    if (HAS_OFF && total != (uint32_t)kMaxBs) {
      // a nibble counter overflowed: the general CTA encoder takes this block
      // (block-uniform branch; nothing was written to the stage)
      reinterpret_cast<uint4*>(sm.cnt)[2 * tid] = z4;
      reinterpret_cast<uint4*>(sm.cnt)[2 * tid + 1] = z4;
      reinterpret_cast<uint4*>(sm.cnt)[256 + 2 * tid] = z4;
      reinterpret_cast<uint4*>(sm.cnt)[256 + 2 * tid + 1] = z4;
      __syncthreads();  // every thread has read the OR words
      if (tid < 4) sm.orw[tid] = 0;
      if (tid == 0) {
        P.rec[blk].kind = KIND_NARROW;
        P.cta_list[atomicAdd(&R->cta_count, 1u)] = (uint32_t)blk;
      }
      continue;
    }
    const bool short_runs = sm.orw[0] < 16u;  // every run <= 15 particles
    const uint32_t w_cnt = bitlen32(sm.orw[0]), w_del = bitlen32(sm.orw[1]);
    const uint32_t w_off = HAS_OFF ? bitlen32(sm.orw[2]) : 0u;
    const uint32_t Ld = (U * w_del + 7) >> 3, Lc = (U * w_cnt + 7) >> 3;
    const uint32_t Lo = HAS_OFF ? ((uint32_t)kMaxBs * w_off + 7) >> 3 : 0u;
    const uint32_t L = H + Ld + Lc + Lo;
    const uint32_t bd = 8 * H, bc = bd + 8 * Ld, bo = bc + 8 * Lc;
    if (tid == 0) {
      P.status[blk] = L;  // payload length for the K3 scan
      P.rec[blk].path = HAS_OFF ? 6 : 7;  // diagnostics: gpzb_encode_path_counts
    }
    if (HAS_OFF && kSP * tid < (int)U) {  // run starts of runs 8t..8t+7 (one 16-byte store; wp is dead)
      uint32_t e[kSP];
      e[0] = ex;
#pragma unroll
      for (int j = 1; j < kSP; ++j) e[j] = e[j - 1] + (dc[j - 1] >> 16);
      reinterpret_cast<uint4*>(sm.wp)[tid] =
          make_uint4(e[0] | e[1] << 16, e[2] | e[3] << 16, e[4] | e[5] << 16, e[6] | e[7] << 16);
    }
    uint32_t* st = sm.bm;  // the payload stage
    // block header, one field per lane of warp 0 (container.serialize_block, container.py:107-121)
    if (wid == 0) {
      const int f = lane;
      uint32_t bpos = 0, val = 0;
      const int a = (f - 2) >> 2, which = (f - 2) & 3;
      const uint32_t hb = __shfl_sync(kFull, w_hdr_b, a & 3), hn = __shfl_sync(kFull, w_hdr_n, a & 3);
      if (f == 0) { bpos = 0; val = (uint32_t)kMaxBs; }
      else if (f == 1) { bpos = 4; val = U; }
      else if (f < 2 + 4 * D) {
        const uint32_t ab = 8 + a * 13;
        if (which < 2) {
          bpos = ab + which * 4;
          val = w_hdr_bound;
        } else if (which == 2) { bpos = ab + 8; val = hb; }
        else { bpos = ab + 9; val = hn; }
      } else if (f < 2 + 4 * D + 3) {
        const int wi = f - 2 - 4 * D;
        bpos = 8 + D * 13 + wi;
        val = wi == 0 ? w_del : (wi == 1 ? w_cnt : w_off);
      }
      if (f < 2 + 4 * D + 3) or_bits(st, 8ull * bpos, val);
    }
    // deltas + run lengths of runs 8t..8t+7, four values per 64-bit window
    if (kSP * tid < (int)U) {
      const uint32_t r0 = kSP * tid;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t* v = dc + 4 * h;
        if (w_del)
          or_bits(st, bd + (r0 + 4 * h) * w_del,
                  (uint64_t)(v[0] & 0xffffu) | (uint64_t)(v[1] & 0xffffu) << w_del |
                      (uint64_t)(v[2] & 0xffffu) << (2 * w_del) | (uint64_t)(v[3] & 0xffffu) << (3 * w_del));
        or_bits(st, bc + (r0 + 4 * h) * w_cnt,
                (uint64_t)(v[0] >> 16) | (uint64_t)(v[1] >> 16) << w_cnt | (uint64_t)(v[2] >> 16) << (2 * w_cnt) |
                    (uint64_t)(v[3] >> 16) << (3 * w_cnt));
      }
    }
    if (HAS_OFF) {
      __syncthreads();  // B6: run starts visible
      // ---- each particle's offset to its place in (seg, off) order
      uint8_t* soff = reinterpret_cast<uint8_t*>(sm.wp + kMaxBs);
#pragma unroll
      for (int k = 0; k < kSP; ++k) {
        const uint32_t r = rk[k] & 0x3ffu, o4 = rk[k] >> 14;
        const uint32_t m = bmsk_wrap(o4);  // nibbles below the offset's (mod 32)
        uint32_t below;
        if (wide && short_runs) {  // runs <= 15: every partial nibble sum fits one multiply
          const uint32_t c0 = sm.cnt[r];
          below = o4 < 32 ? nib_sum1(c0 & m) : nib_sum1(c0) + nib_sum1(sm.cnt[1024 | r] & m);
        } else if (wide) {
          const uint32_t c0 = sm.cnt[r];
          below = o4 < 32 ? nib_sum8(c0 & m) : nib_sum8(c0) + nib_sum8(sm.cnt[1024 | r] & m);
        } else if (short_runs) {
          below = nib_sum1(sm.cnt[r] & m);  // runs <= 15: one multiply
        } else {
          below = nib_sum8(sm.cnt[r] & m);
        }
        soff[(uint32_t)sm.wp[r] + below + ((rk[k] >> 10) & 15u)] = (uint8_t)(o4 >> 2);
      }
      __syncthreads();  // B7
      if (w_off) {  // sorted offsets 8t..8t+7 (each < 16): one 32-bit window
        const uint2 o8 = reinterpret_cast<const uint2*>(soff)[tid];
        uint32_t v = 0;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          v |= ((o8.x >> (8 * j)) & 0xffu) << (j * w_off);
          v |= ((o8.y >> (8 * j)) & 0xffu) << ((j + 4) * w_off);
        }
        or_bits32(st, bo + kSP * tid * w_off, v);
      }
    }
    __syncthreads();  // B8: the stage is complete; counters and OR words are dead
    if (tid < 4) sm.orw[tid] = 0;
    if (HAS_OFF) {  // zero this thread's counter words for the next block
      reinterpret_cast<uint4*>(sm.cnt)[2 * tid] = z4;
      reinterpret_cast<uint4*>(sm.cnt)[2 * tid + 1] = z4;
      if (wide) {
        reinterpret_cast<uint4*>(sm.cnt)[256 + 2 * tid] = z4;
        reinterpret_cast<uint4*>(sm.cnt)[256 + 2 * tid + 1] = z4;
      }
    }
    // ---- the stage to this block's 16-byte aligned staging slot (K3 moves it
    // into place); the stage words are zeroed behind the copy (bitmap invariant;
    // the next block's Bz orders this before its bitmap)
    {
      uint4* slot = reinterpret_cast<uint4*>(P.staging + (uint64_t)blk * kSlotBytes);
      const uint32_t nq = (L + 15) >> 4;  // <= 228 (3,634-byte payloads)
#pragma unroll
      for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t w = tid + h * kST;
        if (w < nq) {
          __stcg(slot + w, reinterpret_cast<const uint4*>(st)[w]);
          reinterpret_cast<uint4*>(st)[w] = z4;
        }
      }
    }
  }
}

}  // namespace gpzb
