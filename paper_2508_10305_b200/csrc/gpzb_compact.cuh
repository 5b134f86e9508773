// K3: stream concatenation — container.compact (container.py:203-208) and
// the offset table of write_container (container.py:211-230).
//
// K2 leaves every block's payload in a 16-byte aligned slot (narrow blocks:
// the staging area, one kSlotBytes slot per block; general blocks: the side
// buffer staged by K2w) and its length in sizes[blk].  Then:
//
//   K3a k_scan_sizes     single-pass decoupled look-back scan over the
//                        payload lengths (tiles of 8192 blocks; each tile
//                        publishes its aggregate, warp 0 looks back over the
//                        tile words): exclusive offsets in place and the
//                        total payload length (the container size is known
//                        here, so the caller can allocate it exactly)
//   K3b k_copy_payloads  8-32 lanes per block: its u64 LE offset-table entry,
//                        and the payload moved from its slot to its byte
//                        offset (arbitrary alignment) with funnel-shifted
//                        16-byte stores; edge chunks shared with the
//                        neighbouring payloads use narrower stores; block 0
//                        also writes table entry 0 and the global header
//
// This is the paper's three-step compaction, with the
// prefix sum done as a single-pass look-back scan.  Keeping the look-back
// out of the encoder matters on B200: blocks that reach their look-back
// while their predecessors are still quantizing would hold the SM idle.
#pragma once

#include "gpzb_encode.cuh"

namespace gpzb {

constexpr int kScanThreads = 1024;
constexpr int kScanItems = 8;
constexpr uint64_t kScanTile = (uint64_t)kScanThreads * kScanItems;
constexpr uint32_t kSlotBytes = 7680;  // >= the largest narrow payload (74 + 2048 + 1408 + 4096 B)

struct CompactParams {
  unsigned long long* sizes;  // in: payload bytes per block; out: exclusive offsets
  unsigned long long* tstat;  // one look-back word per scan tile (zeroed)
  uint64_t nblocks;
  uint8_t* table0;            // table entry 0 (or null: not this call's job)
  uint8_t* table;             // table entry 1
  uint64_t table_base;        // added to every table entry (sharded containers)
  DevResult* res;
  const uint8_t* staging;     // narrow blocks: slot blk * kSlotBytes
  const uint8_t* side;        // general blocks: rec.side_off
  const BlkRec* rec;
  uint8_t* payload;           // block 0's payload byte
  // global header (container.py:211-230), written by tile 0 when non-null
  uint8_t* header;
  int dims, f64, preserve, eb_mode_code;
  double eb;
  uint32_t bs;
  uint64_t header_count, header_blocks;
};

__device__ void write_global_header(const CompactParams& P) {
  uint8_t* h = P.header;
  auto put = [](uint8_t* d, uint64_t v, int nb) { for (int i = 0; i < nb; ++i) d[i] = (uint8_t)(v >> (8 * i)); };
  h[0] = 'G'; h[1] = 'P'; h[2] = 'Z'; h[3] = '1';
  put(h + 4, 1, 2);
  h[6] = (uint8_t)P.dims;
  h[7] = P.f64 ? 1 : 0;
  h[8] = P.preserve ? 1 : 0;
  h[9] = (uint8_t)P.eb_mode_code;
  put(h + 10, (uint64_t)__double_as_longlong(P.eb), 8);
  put(h + 18, (uint64_t)__double_as_longlong(P.res->eb_abs), 8);
  put(h + 26, P.bs, 4);
  put(h + 30, P.header_count, 8);
  put(h + 38, P.header_blocks, 8);
}

// Little-endian u64 at an arbitrary (at least 2-byte aligned when `even`) address.
__device__ __forceinline__ void put_u64_le(uint8_t* p, uint64_t v, bool even) {
  if (even) {
    uint16_t* q = reinterpret_cast<uint16_t*>(p);
#pragma unroll
    for (int i = 0; i < 4; ++i) q[i] = (uint16_t)(v >> (16 * i));
  } else {
#pragma unroll
    for (int i = 0; i < 8; ++i) p[i] = (uint8_t)(v >> (8 * i));
  }
}

__global__ void __launch_bounds__(kScanThreads) k_scan_sizes(const CompactParams P) {
  __shared__ unsigned long long warp_tot[kScanThreads / 32];
  __shared__ unsigned long long tile_excl;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint64_t tile = blockIdx.x;
  const uint64_t first = tile * kScanTile + (uint64_t)tid * kScanItems;

  unsigned long long v[kScanItems], sum = 0;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    v[i] = (first + i < P.nblocks) ? P.sizes[first + i] : 0ull;
    sum += v[i];
  }
  // CTA exclusive scan of the per-thread sums
  unsigned long long x = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = warp_tot[lane], s = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned long long y = __shfl_up_sync(kFull, s, o);
      if (lane >= o) s += y;
    }
    warp_tot[lane] = s - w;  // exclusive prefix of each warp
    const unsigned long long total = __shfl_sync(kFull, s, 31);
    // publish the tile aggregate, then look back over the preceding tiles
    if (lane == 0) st_relaxed(&P.tstat[tile], (tile == 0 ? kFlagInc : kFlagAgg) | total);
    unsigned long long excl = 0;
    long long look = (long long)tile - 1;
    while (look >= 0) {
      const long long idx = look - lane;
      unsigned long long t = kFlagInc;
      if (idx >= 0) {
        do { t = ld_relaxed(&P.tstat[idx]); } while ((t >> 62) == 0);
      }
      const unsigned pm = __ballot_sync(kFull, (t >> 62) == 2);
      const int lim = pm ? __ffs(pm) - 1 : 31;
      unsigned long long c = (lane <= lim) ? (t & kValMask) : 0ull;
#pragma unroll
      for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(kFull, c, o);
      excl += c;
      if (pm) break;
      look -= 32;
    }
    if (lane == 0) {
      if (tile > 0) st_relaxed(&P.tstat[tile], kFlagInc | (excl + total));
      tile_excl = excl;
    }
  }
  __syncthreads();
  unsigned long long run = tile_excl + warp_tot[wid] + x - sum;
#pragma unroll
  for (int i = 0; i < kScanItems; ++i) {
    const uint64_t b = first + i;
    if (b < P.nblocks) {
      P.sizes[b] = run;
      run += v[i];
      if (b + 1 == P.nblocks) P.res->total_payload = run;
    }
  }
}

// Move `len` payload bytes from a 16-byte aligned slot to dst (any
// alignment) with lanes [lane, lane + nl, ...) of a warp.  Destination
// chunks that the payload owns outright get one 16-byte store; the first and
// last chunk, shared with the neighbouring payloads, get word / byte stores.
__device__ __forceinline__ void slot_copy(uint8_t* __restrict__ dst, const uint4* __restrict__ src, uint32_t len, int lane,
                                          int nl) {
  const uint32_t al = (uint32_t)((uintptr_t)dst & 15);
  uint8_t* g16 = dst - al;
  const uint32_t nbytes = al + len;
  const uint32_t nch = (nbytes + 15) >> 4;
  // destination chunk c holds payload bytes [16c - al, 16c - al + 16): the
  // tail of source chunk c-1 (from byte 16 - al) and the head of chunk c
  const uint32_t o = (16 - al) & 15;
  const uint32_t k = o >> 2, sh = (o & 3) * 8;
#pragma unroll 2
  for (uint32_t c = lane; c < nch; c += nl) {
    uint32_t w[4];
    if (al == 0) {
      const uint4 b = src[c];
      w[0] = b.x; w[1] = b.y; w[2] = b.z; w[3] = b.w;
    } else {
      const uint4 a = c ? src[c - 1] : make_uint4(0, 0, 0, 0);
      const uint4 b = (16 * c < len) ? src[c] : make_uint4(0, 0, 0, 0);
      const uint32_t t[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
      uint32_t u[5];
#pragma unroll
      for (int i = 0; i < 5; ++i)
        u[i] = k == 0 ? t[i] : k == 1 ? t[i + 1] : k == 2 ? t[i + 2] : t[i + 3];
#pragma unroll
      for (int j = 0; j < 4; ++j) w[j] = sh ? __funnelshift_r(u[j], u[j + 1], sh) : u[j];
    }
    const uint32_t b0 = c * 16;
    if (b0 >= al && b0 + 16 <= nbytes) {
      __stcs(reinterpret_cast<uint4*>(g16 + b0), make_uint4(w[0], w[1], w[2], w[3]));
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t wb = b0 + 4 * j;
        if (wb >= al && wb + 4 <= nbytes) {
          *reinterpret_cast<uint32_t*>(g16 + wb) = w[j];
        } else if (wb + 4 > al && wb < nbytes) {
          for (int q = 0; q < 4; ++q)
            if (wb + q >= al && wb + q < nbytes) g16[wb + q] = (uint8_t)(w[j] >> (8 * q));
        }
      }
    }
  }
}

constexpr int kCopyWarps = 8;

// G lanes per block (8, 16 or 32; the host picks it from the average
// payload): small payloads leave most of a warp idle and every block waits on
// the same two dependent loads, so a warp moves 32 / G blocks at once.
template <int G>
__global__ void __launch_bounds__(32 * kCopyWarps) k_copy_payloads(const CompactParams P) {
  static_assert(G == 8 || G == 16 || G == 32, "lanes per block");
  const int lane = threadIdx.x & (G - 1);
  const uint64_t blk = (uint64_t)blockIdx.x * (kCopyWarps * 32 / G) + (threadIdx.x / G);
  if (blk >= P.nblocks) return;
  // the scan result and the record's kind are independent loads: both in flight at once
  // (also loading this lane's first slot chunks ahead of the scan result was 1% slower)
  const uint8_t kind = P.rec[blk].kind;
  const uint64_t ex = P.sizes[blk];
  const uint64_t end = (blk + 1 < P.nblocks) ? P.sizes[blk + 1] : P.res->total_payload;
  const uint32_t len = (uint32_t)(end - ex);
  // this block's offset-table entry (write_container, container.py:211-230)
  if (lane == 0) put_u64_le(P.table + 8 * blk, P.table_base + end, ((uintptr_t)P.table & 1) == 0);
  if (blk == 0 && lane == 1 && P.table0) put_u64_le(P.table0, P.table_base, false);
  if (blk == 0 && lane == 2 && P.header) write_global_header(P);
  if (len == 0) return;
  const uint8_t* src = kind == KIND_WIDE ? P.side + P.rec[blk].side_off : P.staging + blk * (uint64_t)kSlotBytes;
  slot_copy(P.payload + ex, reinterpret_cast<const uint4*>(src), len, lane, G);
}

// Diagnostics: how many blocks took each offset-order path (BlkRec::path).
__global__ void k_path_counts(const BlkRec* rec, uint64_t nblocks, unsigned long long* counts) {
  __shared__ unsigned int h[8];
  if (threadIdx.x < 8) h[threadIdx.x] = 0;
  __syncthreads();
  for (uint64_t b = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; b < nblocks; b += (uint64_t)gridDim.x * blockDim.x)
    if (rec[b].kind != KIND_ERROR && rec[b].path < 8) atomicAdd(&h[rec[b].path], 1u);
  __syncthreads();
  if (threadIdx.x < 8 && h[threadIdx.x]) atomicAdd(&counts[threadIdx.x], (unsigned long long)h[threadIdx.x]);
}

}  // namespace gpzb
