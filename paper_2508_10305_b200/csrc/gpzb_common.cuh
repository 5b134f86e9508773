// Shared device helpers for the GPZ B200 kernels (sm_100a).
//
// Everything here restates the reference's float64 semantics with explicit
// IEEE-rounded intrinsics (__dadd_rn/__dmul_rn/__ddiv_rn/__drcp_rn), so that
// no FMA contraction or reassociation can change a rounding.  Translation
// units are also compiled with -fmad=false as a second line of defence.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "../../include/gpzb.h"

namespace gpzb {

constexpr int kThreads = 256;             // CTA size of every block-level kernel
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 4;                 // particles per thread
constexpr int kMaxBs = kThreads * kItems; // the block one CTA holds (larger ones: gpzb_big.cuh)
constexpr unsigned kFull = 0xffffffffu;

// ---------------------------------------------------------------- reasons
// Shared with the host (gpzb_reason_message) and the Python layer.
enum Reason : uint32_t {
  R_NONE = 0,
  // compress (pipeline.py:80-83 wraps the block-scoped ones as "block i: ...")
  R_NONFINITE = 1,       // DomainError, dataset-level  (model.py:75-77)
  R_EB_NOT_POSITIVE = 2, // DomainError                 (quantizer.py:102-103)
  R_AXIS_RANGE = 3,      // WidthOverflow               (quantizer.py:82-85)
  R_GEOMETRY = 4,        // WidthOverflow               (quantizer.py:118-122)
  // container-level CorruptData (container.py:249-290)
  R_SHORT = 10, R_MAGIC = 11, R_VERSION = 12, R_DIMS = 13, R_ENUM = 14, R_EB_ABS = 15,
  R_FLAGS = 16, R_TABLE_TRUNC = 17, R_TABLE_START = 18, R_TABLE_ORDER = 19, R_TABLE_END = 20,
  // block-level CorruptData (container.py:150-193, codec.py:132-151, pipeline.py:116-181)
  R_BLK_SHORT = 30, R_BLK_UNIQUE = 31, R_BLK_WIDTH = 32, R_BLK_NOSEG = 33, R_BLK_OFFBITS = 34,
  R_BLK_BOUNDS = 35, R_BLK_TRUNC = 36, R_BLK_TRAILING = 37, R_BLK_PAD_DELTA = 38,
  R_BLK_PAD_COUNT = 39, R_BLK_PAD_OFF = 40, R_BLK_IDS = 41, R_BLK_ZERO_RUN = 42,
  R_BLK_RUN_SUM = 43, R_BLK_RUN_MAX = 44, R_BLK_AXIS_RANGE = 45, R_BLK_SEGCOUNT = 46,
  R_BLK_SEG_RANGE = 47, R_BLK_OFF_RANGE = 48, R_BLK_PAD_RANK = 49, R_BLK_RANKS = 50,
  R_BLK_COUNT = 51, R_BLK_TOO_BIG = 52, R_BLK_WINDOW = 53,
  // after all blocks (pipeline.py:200-205)
  R_NONFINITE_OUT = 60, R_TOTAL = 61,
  R_UNSUPPORTED_BS = 70,
};

// Device-side result record, zeroed per call.  Error words store the
// bitwise complement of (block << 12 | axis << 8 | reason) and are combined
// with atomicMax, so the zero state means "no error" and the smallest block
// index wins (the reference's serial first-error order).
struct DevResult {
  unsigned long long err_block;     // compress: geometry errors; decompress: decode errors
  unsigned long long err_count;     // decompress: count-vs-boundary errors (pipeline.py:174-181)
  unsigned int nonfinite_mask;      // bit a: axis a holds a non-finite value
  unsigned int table_flags;         // bit0 start, bit1 order, bit2 end (container.py:282-290)
  unsigned long long side_need;     // compress: K2w found the side buffer too small (bytes K1.5 reserved)
  unsigned long long total_payload; // inclusive prefix of the last block
  unsigned long long range_w[2];    // ukey(-lo), ukey(hi): joint range (model.py:194-195)
  double eb_abs;
  unsigned long long path_blocks[8];
  unsigned long long side_bytes;    // K1.5: bytes reserved in the side buffer for wide blocks
  unsigned int wide_count;          // K1.5: number of wide blocks (decode: K4a's CTA-list length)
  unsigned int cta_count;           // K1.5: narrow blocks for the CTA encoder (its list length)
  unsigned int warp_count;          // K1.5: blocks for the warp encoder
  unsigned int small_count;         // K1.5: blocks for K2s with offsets (small_list from the front)
  unsigned int small0_count;        // K1.5: blocks for K2s without offsets (small_list from the back)
  unsigned int claim;               // decode: K4w's next block (zeroed by K4a)
};
static_assert(sizeof(DevResult) % 16 == 0, "DevResult alignment");

__host__ __device__ inline unsigned long long err_code(uint64_t blk, int axis, int reason) {
  return ~((blk << 12) | ((uint64_t)(axis & 15) << 8) | (uint64_t)reason);
}

// ------------------------------------------------------ ordered encodings
// u64 whose unsigned order equals the numeric order of the double.
__device__ __forceinline__ unsigned long long ukey(double v) {
  unsigned long long b = (unsigned long long)__double_as_longlong(v);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ inline double ukey_inv(unsigned long long k) {
  unsigned long long b = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
  double d;
  memcpy(&d, &b, 8);
  return d;
}
// i32 whose signed order equals the numeric order of the float.
__device__ __forceinline__ int fkey(float f) {
  int i = __float_as_int(f);
  return i ^ ((i >> 31) & 0x7fffffff);
}
__device__ __forceinline__ float fkey_inv(int k) { return __int_as_float(k ^ ((k >> 31) & 0x7fffffff)); }

// ------------------------------------------------------------ bit helpers
__device__ __forceinline__ uint64_t shr64(uint64_t v, unsigned s) { return s >= 64 ? 0 : v >> s; }
__device__ __forceinline__ uint64_t shl64(uint64_t v, unsigned s) { return s >= 64 ? 0 : v << s; }
__device__ __forceinline__ int bitlen64(uint64_t v) { return v ? 64 - __clzll((long long)v) : 0; }
__device__ __forceinline__ int bitlen32(uint32_t v) { return v ? 32 - __clz((int)v) : 0; }
__device__ __forceinline__ uint64_t mask64(unsigned bits) { return bits >= 64 ? ~0ull : ((1ull << bits) - 1); }

// --------------------------------------------------- memory-order helpers
// Look-back status words carry their own payload (flag + value in one
// 64-bit word), so relaxed gpu-scope accesses are sufficient.
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// ------------------------------------------- TMA bulk copies + mbarriers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
// global -> shared bulk copy (cp.async.bulk, SASS UBLKCP); 16B aligned, size % 16 == 0
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// 4-byte asynchronous global -> shared copies (LDGSTS), committed as a group
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// ------------------------------------------------------- block primitives
// Exclusive scan over the CTA (one value per thread).  `ws` holds kWarps
// entries; the call contains two __syncthreads.
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T& total, T* ws) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(kFull, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[wid] = x;
  __syncthreads();
  // every warp scans the kWarps totals itself (lanes 0..kWarps-1)
  T s = (lane < kWarps) ? ws[lane] : T(0);
#pragma unroll
  for (int o = 1; o < kWarps; o <<= 1) {
    T y = __shfl_up_sync(kFull, s, o);
    if (lane >= o) s += y;
  }
  const T incl_w = __shfl_sync(kFull, s, wid);          // inclusive through this warp
  total = __shfl_sync(kFull, s, kWarps - 1);
  __syncthreads();
  return incl_w - __shfl_sync(kFull, x, 31) + x - v;  // exclusive prefix of this thread
}

// Shared-memory atomic OR without a returned value (RED, no scoreboard wait).
__device__ __forceinline__ void red_or_shared(uint32_t* p, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// The same, issued only where `p` holds (a predicated RED: no branch, no
// convergence barrier around it).
__device__ __forceinline__ void red_or_shared_if(bool p, uint32_t* a, uint32_t v) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %2, 0;\n\t@q red.shared.or.b32 [%0], %1;\n\t}" ::"r"(smem_u32(a)),
      "r"(v), "r"((uint32_t)p)
      : "memory");
}

// OR-reduction over the CTA of NV u32 values; result broadcast to all.
template <int NV>
__device__ __forceinline__ void block_or(uint32_t (&v)[NV], uint32_t* ws /* kWarps*NV */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    uint32_t r = __reduce_or_sync(kFull, v[i]);
    if (lane == 0) ws[wid * NV + i] = r;
  }
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    uint32_t r = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) r |= ws[w * NV + i];
    v[i] = r;
  }
  __syncthreads();
}

// The same with one RED per warp and value and a single barrier: `ws`
// holds NV words that the caller zeroed before an earlier barrier and does
// not touch again until a later one.
template <int NV>
__device__ __forceinline__ void block_or_z(uint32_t (&v)[NV], uint32_t* ws) {
  const int lane = threadIdx.x & 31;
  // lane i (< NV) ORs the warp's value i: one RED instruction per warp
  uint32_t mine = 0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const uint32_t r = __reduce_or_sync(kFull, v[i]);
    mine = lane == i ? r : mine;
  }
  red_or_shared_if(lane < NV && mine != 0, &ws[lane < NV ? lane : 0], mine);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = ws[i];
}

// ---------------------------------------------------------------- geometry
// Per-axis block geometry, restating quantizer.effective_bound
// (quantizer.py:60-68), axis_bin_count (:71-86) and derive_geometry
// (:89-129) with the same IEEE operations in the same order.
struct AxisGeo {
  double lo, hi;       // block bounds (exact)
  double eb_int, w;    // guarded half-width and bin width 2*eb_int
  double rinv;         // RN(1/w) for the certified fast path
  uint64_t Q;          // bin count
  uint64_t N;          // segment count
  uint32_t b;          // log2(m), 0..64
  int mode;            // 0: certified reciprocal, 1: exact divide, 2: exact + snap (half-bound)
};

__device__ __forceinline__ double inner_bound(double eb, double lo, double hi, bool f64, bool& half) {
  // _GUARD_EPS (quantizer.py:41-46); both constants are exact doubles
  const double G = f64 ? (1.0 / 281474976710656.0) : (1.0 / 16777216.0 + 1.0 / 281474976710656.0);
  double scale = __dadd_rn(fmax(fabs(lo), fabs(hi)), __dmul_rn(2.0, eb));
  double margin = __dmul_rn(scale, G);
  double heb = __dmul_rn(0.5, eb);
  half = margin >= heb;
  return half ? heb : __dsub_rn(eb, margin);
}

// Returns R_NONE or R_AXIS_RANGE.
__device__ inline int axis_geometry(double lo, double hi, double eb, bool f64, uint64_t target,
                                    AxisGeo& g) {
  g.lo = lo;
  g.hi = hi;
  bool half;
  g.eb_int = inner_bound(eb, lo, hi, f64, half);
  g.w = __dmul_rn(2.0, g.eb_int);
  double span = __dsub_rn(hi, lo);
  if (span <= 0.0) {
    g.Q = 1;
  } else {
    double ratio = __ddiv_rn(span, g.w);
    if (!(ratio < 18446744073709551616.0)) return R_AXIS_RANGE;
    g.Q = (uint64_t)__double2ull_rz(ratio) + 1;  // floor(ratio) + 1, ratio >= 0
  }
  uint64_t per = g.Q / target + (g.Q % target ? 1 : 0);
  g.b = (uint32_t)bitlen64(per - 1);  // per >= 1
  if (g.b >= 64) {
    g.N = 1;  // m = 2^64 covers any Q < 2^64
  } else {
    uint64_t m = 1ull << g.b;
    g.N = g.Q / m + (g.Q % m ? 1 : 0);
  }
  // Quantizer branch.  Normal branch (not half): q = floor(RN(RN(x-lo)/w))
  // never needs the edge snap and never clips (proof in DESIGN.md §3.2);
  // Q <= 2^20 additionally keeps RN(t*rinv) < 2^21 so the certificate on
  // its low word applies.
  if (half || !(g.w > 0.0) || !isfinite(g.w)) {
    g.mode = 2;
  } else if (g.Q <= (1ull << 20)) {
    g.mode = 0;
  } else {
    g.mode = 1;
  }
  g.rinv = (g.mode == 0) ? __drcp_rn(g.w) : 0.0;
  return R_NONE;
}

// Reconstruction value of bin q as the decoder emits it, in float64
// (quantizer._axis_reconstruction, quantizer.py:132-139), general form.
__device__ __forceinline__ double midpoint_general(uint64_t q, double lo, double w, bool f64) {
  double a = __dadd_rn(__ull2double_rn(q), 0.5);
  double v = __dadd_rn(lo, __dmul_rn(a, w));
  if (!f64) v = (double)__double2float_rn(v);
  return v;
}

// Exact quantization with the edge-snap rule (quantizer.py:142-173); used
// for half-bound axes, where the guard margin does not absorb rounding.
__device__ __noinline__ uint64_t quantize_snap(double x, const AxisGeo& g, double eb, bool f64) {
  double t = __dsub_rn(x, g.lo);
  double qf = floor(__ddiv_rn(t, g.w));
  double top = __ull2double_rn(g.Q - 1);
  qf = fmin(fmax(qf, 0.0), top);
  uint64_t q = (uint64_t)__double2ull_rz(qf);
  double v = midpoint_general(q, g.lo, g.w, f64);
  double err = fabs(__dsub_rn(v, x));
  if (err > eb && g.Q <= (1ull << 62)) {
    long long c = (long long)q + ((v > x) ? -1 : 1);
    long long qmax = (long long)(g.Q - 1);
    c = c < 0 ? 0 : (c > qmax ? qmax : c);
    double v2 = midpoint_general((uint64_t)c, g.lo, g.w, f64);
    double e2 = fabs(__dsub_rn(v2, x));
    if (e2 < err) q = (uint64_t)c;
  }
  return q;
}

// Bin index of one coordinate, bit-identical to quantizer._quantize_axis.
__device__ __forceinline__ uint64_t quantize_coord(double x, const AxisGeo& g, double eb, bool f64) {
  double t = __dsub_rn(x, g.lo);
  if (g.mode == 0) {
    // certified reciprocal path: r' = RN(t * RN(1/w)) is within one ulp of
    // RN(t / w); when r' < 2^21 its low word is pure fraction, and a low word
    // other than 0 / 0xffffffff proves floor(r') == floor(RN(t/w)).
    double r = __dmul_rn(t, g.rinv);
    uint32_t rl = (uint32_t)__double2loint(r);
    uint32_t rh = (uint32_t)__double2hiint(r);
    uint32_t q = (uint32_t)__double2loint(__dadd_rz(r, 4503599627370496.0));
    if ((rl + 1u) <= 1u && (rl | rh) != 0u) {
      q = (uint32_t)__double2ull_rz(__ddiv_rn(t, g.w));
    }
    return q;
  }
  if (g.mode == 1) return (uint64_t)__double2ull_rz(__ddiv_rn(t, g.w));
  return quantize_snap(x, g, eb, f64);
}

// (1 << (w mod 32)) - 1 in one instruction (BMSK)
__device__ __forceinline__ uint32_t bmsk_wrap(uint32_t w) {
  uint32_t d;
  asm("bmsk.wrap.b32 %0, 0, %1;" : "=r"(d) : "r"(w));
  return d;
}

// ------------------------------------------------------ staging bit writer
// OR `nbits` (<= 64) bits of v into a u32 word array at bit position pos.
__device__ __forceinline__ void or_bits(uint32_t* st, uint64_t pos, uint64_t v) {
  const uint32_t sh = (uint32_t)(pos & 31);
  uint32_t* w = st + (pos >> 5);
  const uint64_t lo = v << sh;
  const uint32_t w0 = (uint32_t)lo, w1 = (uint32_t)(lo >> 32);
  const uint32_t w2 = sh ? (uint32_t)(v >> (64 - sh)) : 0u;
  red_or_shared_if(w0 != 0, w, w0);
  red_or_shared_if(w1 != 0, w + 1, w1);
  red_or_shared_if(w2 != 0, w + 2, w2);
}

// The same for a value of at most 32 bits: two predicated REDs, 32-bit shifts.
__device__ __forceinline__ void or_bits32(uint32_t* st, uint32_t pos, uint32_t v) {
  const uint32_t sh = pos & 31;
  uint32_t* w = st + (pos >> 5);
  const uint32_t w0 = v << sh, w1 = sh ? v >> (32 - sh) : 0u;
  red_or_shared_if(w0 != 0, w, w0);
  red_or_shared_if(w1 != 0, w + 1, w1);
}

// Read `nbits` (<= 64) bits at bit position pos from a u32 word array.
__device__ __forceinline__ uint64_t get_bits(const uint32_t* st, uint64_t pos, uint32_t nbits) {
  if (nbits == 0) return 0;
  const uint32_t sh = (uint32_t)(pos & 31);
  const uint32_t* w = st + (pos >> 5);
  uint64_t lo = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  uint64_t v = lo >> sh;
  if (sh && nbits + sh > 64) v |= (uint64_t)w[2] << (64 - sh);
  return v & mask64(nbits);
}

}  // namespace gpzb
