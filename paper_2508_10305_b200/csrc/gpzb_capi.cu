// C ABI of the GPZ B200 path (declared in include/gpzb.h).
//
// Host-side orchestration only: workspace layout, kernel dispatch over
// (dims, precision, preserve_order), the one small result read-back per call,
// and the container's global-header validation (container.py:245-281).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>

#include "gpzb_big.cuh"
#include "gpzb_decode.cuh"
#include "gpzb_decode_warp.cuh"
#include "gpzb_encode.cuh"
#include "gpzb_encode_narrow.cuh"
#include "gpzb_encode_small.cuh"
#include "gpzb_encode_warp.cuh"
#include "gpzb_encode_wide.cuh"
#include "gpzb_metrics.cuh"
#include "gpzb_stages.cuh"

using namespace gpzb;

namespace {

#ifndef GPZB_K1_CTAS
#define GPZB_K1_CTAS 8  // grid-stride CTAs per SM of K1 (16: batched compress step 4.77 +- 0.08 ms, 8: 4.69 +- 0.01)
#endif

constexpr uint64_t kAlign = 256;

// Kernel launches issued by this library (process-wide; gpzb_kernel_launches).
std::atomic<unsigned long long> g_launches{0};
#define GPZB_COUNT_LAUNCH() g_launches.fetch_add(1, std::memory_order_relaxed)
inline uint64_t align_up(uint64_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }

struct EncLayout {
  uint64_t status, tstat, bounds, rec, list, ctalist, slist, wlist, staging, big, total;
};
constexpr uint32_t kMaxBigBs = 1u << 24;  // K2b / K4b: larger blocks are refused (GPZB_UNSUPPORTED)

inline uint64_t nblocks_of(uint64_t count, uint32_t bs) { return bs ? (count + bs - 1) / bs : 0; }

int sm_count();
// CTAs of K2b / K4b: one workspace slice each, at most ~1 GB of slices
uint64_t big_grid(uint64_t nblocks, uint64_t slice) {
  const uint64_t cap = std::max<uint64_t>(1, (1ull << 30) / slice);
  return std::min<uint64_t>(std::min<uint64_t>(nblocks, (uint64_t)sm_count()), cap);
}
EncLayout enc_layout(uint64_t nblocks, int dims, int prec, uint32_t bs = kMaxBs) {
  EncLayout L;
  L.status = align_up(sizeof(DevResult));
  L.tstat = align_up(L.status + 8 * nblocks);
  L.bounds = align_up(L.tstat + 8 * ((nblocks + kScanTile - 1) / kScanTile));
  L.rec = align_up(L.bounds + nblocks * 2ull * dims * (prec ? 8 : 4));
  L.list = align_up(L.rec + nblocks * sizeof(BlkRec));
  L.ctalist = align_up(L.list + 4 * nblocks);
  L.slist = align_up(L.ctalist + 4 * nblocks);
  L.wlist = align_up(L.slist + 4 * nblocks);
  L.staging = align_up(L.wlist + 4 * nblocks);
  // blocks of <= 1024 particles: one staging slot each; larger: K2b's slices
  L.big = align_up(L.staging + (bs <= (uint32_t)kMaxBs ? (uint64_t)kSlotBytes * nblocks : 0));
  L.total = align_up(L.big + (bs > (uint32_t)kMaxBs && nblocks ? big_grid(nblocks, big_enc_slice(bs)) * big_enc_slice(bs) : 0));
  return L;
}

int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// Per-device launch facts, cached per (kernel, device): the dynamic
// shared-memory opt-in is a per-device function attribute, and the occupancy
// query sizes the persistent grids.
std::mutex g_attr_mu;
std::map<std::tuple<const void*, int, int, size_t>, int> g_occ;

template <typename K>
int occupancy(K kern, int threads, size_t smem) {
  int dev = 0;
  cudaGetDevice(&dev);
  const auto key = std::make_tuple(reinterpret_cast<const void*>(kern), dev, threads, smem);
  std::lock_guard<std::mutex> lk(g_attr_mu);
  auto it = g_occ.find(key);
  if (it != g_occ.end()) return it->second;
  if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, threads, smem) != cudaSuccess || per < 1) per = 1;
  g_occ[key] = per;
  return per;
}

inline int cuda_status(cudaError_t e) { return e == cudaSuccess ? GPZB_OK : GPZB_CUDA_ERROR + (int)e; }

int check_args(int dims, int prec, uint32_t bs) {
  if (dims < 1 || dims > 3 || (prec != GPZB_F32 && prec != GPZB_F64)) return GPZB_INVALID_ARGUMENT;
  if (bs == 0 || bs % 32) return GPZB_INVALID_ARGUMENT;
  if (bs > kMaxBigBs) return GPZB_UNSUPPORTED;
  return GPZB_OK;
}

void put_le_host(uint8_t* d, uint64_t v, int n) {
  for (int i = 0; i < n; ++i) d[i] = (uint8_t)(v >> (8 * i));
}
uint64_t get_le_host(const uint8_t* d, int n) {
  uint64_t v = 0;
  for (int i = 0; i < n; ++i) v |= (uint64_t)d[i] << (8 * i);
  return v;
}

void decode_err(unsigned long long w, int64_t* blk, int32_t* axis, int32_t* reason) {
  const unsigned long long c = ~w;
  *blk = (int64_t)(c >> 12);
  *axis = (int32_t)((c >> 8) & 15);
  *reason = (int32_t)(c & 255);
}

int status_of_reason(int r) {
  switch (r) {
    case R_NONE: return GPZB_OK;
    case R_NONFINITE: case R_EB_NOT_POSITIVE: case R_NONFINITE_OUT: return GPZB_DOMAIN_ERROR;
    case R_AXIS_RANGE: case R_GEOMETRY: return GPZB_WIDTH_OVERFLOW;
    case R_UNSUPPORTED_BS: case R_BLK_WINDOW: return GPZB_UNSUPPORTED;
    default: return GPZB_CORRUPT_DATA;
  }
}

void clear_result(gpzb_result* r) {
  memset(r, 0, sizeof(*r));
  r->block = -1;
  r->axis = -1;
  r->decode_block = -1;
  r->count_block = -1;
}

void set_out(EncParams& P, uint8_t* out, uint64_t nb, uint64_t table_base, uint64_t header_count,
             uint64_t header_blocks, int write_header) {
  P.header = out && write_header ? out : nullptr;
  P.table0 = out ? out + GPZB_GLOBAL_HEADER_SIZE : nullptr;
  P.table = out ? out + GPZB_GLOBAL_HEADER_SIZE + 8 : nullptr;
  P.payload = out ? out + GPZB_GLOBAL_HEADER_SIZE + 8 * (nb + 1) : nullptr;
  P.table_base = table_base;
  P.header_count = header_count;
  P.header_blocks = header_blocks;
}

// K3 parameters from the encoder's (payload == null: the container is not
// allocated yet; K3a still runs, K3b waits for gpzb_emit_async).
CompactParams make_compact(const EncParams& P, int dims, bool f64) {
  CompactParams C;
  memset(&C, 0, sizeof(C));
  C.sizes = P.status;
  C.tstat = P.tstat;
  C.nblocks = P.nblocks;
  C.table0 = P.table0;
  C.table = P.table;
  C.table_base = P.table_base;
  C.res = P.res;
  C.staging = P.staging;
  C.side = P.side;
  C.rec = P.rec;
  C.payload = P.payload;
  C.header = P.header;
  C.dims = dims;
  C.f64 = f64 ? 1 : 0;
  C.preserve = P.preserve;
  C.eb_mode_code = P.eb_mode_code;
  C.eb = P.eb;
  C.bs = P.bs;
  C.header_count = P.header_count;
  C.header_blocks = P.header_blocks;
  return C;
}

// K3b: table entries, global header, payload moves; lanes per block from the
// average payload when the caller knows it (0: a full warp per block).
#ifndef GPZB_K3B_G
#define GPZB_K3B_G 0  // 0: by the average payload; else fixed 8 / 16 / 32
#endif
void launch_emit(const CompactParams& C, cudaStream_t s, uint64_t avg_payload = 0) {
  int g = GPZB_K3B_G ? GPZB_K3B_G : avg_payload == 0 || avg_payload >= 1024 ? 32 : avg_payload >= 384 ? 16 : 8;
  const uint64_t per_cta = (uint64_t)kCopyWarps * 32 / g;
  const unsigned grid = (unsigned)((C.nblocks + per_cta - 1) / per_cta);
  GPZB_COUNT_LAUNCH();
  if (g == 8) k_copy_payloads<8><<<grid, 32 * kCopyWarps, 0, s>>>(C);
  else if (g == 16) k_copy_payloads<16><<<grid, 32 * kCopyWarps, 0, s>>>(C);
  else k_copy_payloads<32><<<grid, 32 * kCopyWarps, 0, s>>>(C);
}

template <int D, bool F64>
void launch_range(const EncParams& P, cudaStream_t s) {
  const uint64_t grid = std::min<uint64_t>((P.nblocks + kWarps - 1) / kWarps, (uint64_t)sm_count() * GPZB_K1_CTAS);
  GPZB_COUNT_LAUNCH();
  k_range_w<D, typename std::conditional<F64, double, float>::type><<<(unsigned)grid, kThreads, 0, s>>>(P);
}

template <int D, bool F64>
void launch_geometry(const EncParams& P, cudaStream_t s) {
  GPZB_COUNT_LAUNCH();
  k_geometry<D, typename std::conditional<F64, double, float>::type>
      <<<(unsigned)((P.nblocks + 255) / 256), 256, 0, s>>>(P);
}

template <int D, bool F64>
void launch_encode(const EncParams& P, cudaStream_t s) {
  if (P.bs > (uint32_t)kMaxBs) {  // K2b: every block of the call is on the general list
    const unsigned grid = (unsigned)big_grid(P.nblocks, big_enc_slice(P.bs));
    GPZB_COUNT_LAUNCH();
    if (P.preserve) k_encode_big<D, F64, true><<<grid, kThreads, 0, s>>>(P, P.big);
    else k_encode_big<D, F64, false><<<grid, kThreads, 0, s>>>(P, P.big);
    GPZB_COUNT_LAUNCH();
    const CompactParams C = make_compact(P, D, F64);
    k_scan_sizes<<<(unsigned)((P.nblocks + kScanTile - 1) / kScanTile), kScanThreads, 0, s>>>(C);
    if (P.payload) launch_emit(C, s);
    return;
  }
  {  // K2w: persistent over K1.5's list of general blocks (usually empty)
    const unsigned grid = (unsigned)std::min<uint64_t>(P.nblocks, (uint64_t)sm_count() * 4);
    if (P.preserve) { GPZB_COUNT_LAUNCH(); k_encode_wide<D, F64, true><<<grid, kThreads, 0, s>>>(P); }
    else { GPZB_COUNT_LAUNCH(); k_encode_wide<D, F64, false><<<grid, kThreads, 0, s>>>(P); }
  }
  // K2s first (it may hand blocks back to K2's list), then K2p and K2; every
  // encoder is persistent and reads its block count on the device
  if constexpr (!F64) {
    const uint64_t sm = (uint64_t)sm_count();
    const unsigned g1 = (unsigned)std::min<uint64_t>(P.nblocks, sm * occupancy(k_encode_small<D, true>, kST, 0));
    const unsigned g0 = (unsigned)std::min<uint64_t>(P.nblocks, sm * occupancy(k_encode_small<D, false>, kST, 0));
    GPZB_COUNT_LAUNCH();
    k_encode_small<D, true><<<g1, kST, 0, s>>>(P);
    GPZB_COUNT_LAUNCH();
    k_encode_small<D, false><<<g0, kST, 0, s>>>(P);
  }
  if (!P.small0 || F64) {
    // both variants (K1.5's block list / every block in order); the one that
    // does not match the device-side K2p count exits at once
    const unsigned wgrid = (unsigned)std::min<uint64_t>((P.nblocks + kWarpEncWarps - 1) / kWarpEncWarps,
                                                        (uint64_t)sm_count() * occupancy(k_encode_warp<D, F64, false>, 32 * kWarpEncWarps, kWarpEncSmemBytes));
    occupancy(k_encode_warp<D, F64, true>, 32 * kWarpEncWarps, kWarpEncSmemBytes);  // sets its shared-memory attribute on this device
    GPZB_COUNT_LAUNCH();
    k_encode_warp<D, F64, true><<<wgrid, 32 * kWarpEncWarps, kWarpEncSmemBytes, s>>>(P);
    GPZB_COUNT_LAUNCH();
    k_encode_warp<D, F64, false><<<wgrid, 32 * kWarpEncWarps, kWarpEncSmemBytes, s>>>(P);
  }
  {
    const unsigned cgrid = (unsigned)std::min<uint64_t>(P.nblocks, (uint64_t)sm_count() * occupancy(k_encode<D, F64>, kThreads, 0));
    GPZB_COUNT_LAUNCH();
    k_encode<D, F64><<<cgrid, kThreads, 0, s>>>(P);
  }
  GPZB_COUNT_LAUNCH();
  const CompactParams C = make_compact(P, D, F64);
  k_scan_sizes<<<(unsigned)((P.nblocks + kScanTile - 1) / kScanTile), kScanThreads, 0, s>>>(C);
  if (P.payload) launch_emit(C, s);
}

template <int D, bool F64>
void launch_decode(const DecParams& P, bool pres, cudaStream_t s) {
  const uint64_t nb = P.blk_hi - P.blk_lo;
  const unsigned pgrid = (unsigned)((nb + 255) / 256);
  const unsigned lgrid = (unsigned)std::min<uint64_t>(nb, (uint64_t)sm_count() * GPZB_K4_MINB);
  if (P.bs > (uint32_t)kMaxBs) {  // K4a lists every block for K4b
    const unsigned grid = (unsigned)big_grid(nb, big_dec_slice(P.bs));
    GPZB_COUNT_LAUNCH();
    GPZB_COUNT_LAUNCH();
    if (pres) {
      k_decode_plan<D, F64, true><<<pgrid, 256, 0, s>>>(P);
      k_decode_big<D, F64, true><<<grid, kThreads, 0, s>>>(P, P.big);
    } else {
      k_decode_plan<D, F64, false><<<pgrid, 256, 0, s>>>(P);
      k_decode_big<D, F64, false><<<grid, kThreads, 0, s>>>(P, P.big);
    }
    return;
  }
  if (pres) {
    GPZB_COUNT_LAUNCH();
    k_decode_plan<D, F64, true><<<pgrid, 256, 0, s>>>(P);
    GPZB_COUNT_LAUNCH();
    k_decode_list<D, F64, true><<<lgrid, kThreads, 0, s>>>(P, P.list);
  } else {
    GPZB_COUNT_LAUNCH();
    k_decode_plan<D, F64, false><<<pgrid, 256, 0, s>>>(P);
    const int per_sm = occupancy(k_decode_warp<D, F64>, 32 * kWarpDecWarps, kWarpDecSmemBytes);
    const unsigned wgrid = (unsigned)std::min<uint64_t>((nb + kWarpDecWarps - 1) / kWarpDecWarps,
                                                        (uint64_t)sm_count() * per_sm);
    DecParams Q = P;  // L2 prefetch distance: one claim round of the grid ahead (gpzb_decode_warp.cuh)
    Q.pf_blks = (uint64_t)GPZB_K4W_PF * wgrid * kWarpDecWarps * warp_claim_chunk((uint32_t)nb, wgrid);
    const uint64_t avg = P.nblocks ? P.payload_len / P.nblocks : 0;
    Q.pf_dist = avg >= GPZB_K4W_PF_MIN ? (avg * Q.pf_blks + 15) & ~15ull : 0ull;
    GPZB_COUNT_LAUNCH();
    k_decode_warp<D, F64><<<wgrid, 32 * kWarpDecWarps, kWarpDecSmemBytes, s>>>(Q);
    GPZB_COUNT_LAUNCH();
    k_decode_list<D, F64, false><<<lgrid, kThreads, 0, s>>>(P, P.list);
  }
}

#define DISPATCH_DP(dims, prec, FN, ...)                      \
  do {                                                       \
    if (prec) {                                              \
      if (dims == 1) FN<1, true>(__VA_ARGS__);               \
      else if (dims == 2) FN<2, true>(__VA_ARGS__);          \
      else FN<3, true>(__VA_ARGS__);                         \
    } else {                                                 \
      if (dims == 1) FN<1, false>(__VA_ARGS__);              \
      else if (dims == 2) FN<2, false>(__VA_ARGS__);         \
      else FN<3, false>(__VA_ARGS__);                        \
    }                                                        \
  } while (0)

template <int D, bool F64, bool R64>
void launch_pair_blocks(const PairParams& P, cudaStream_t s) {
  using T = typename std::conditional<F64, double, float>::type;
  using R = typename std::conditional<R64, double, float>::type;
  GPZB_COUNT_LAUNCH();
  if (P.bs > (uint32_t)kMaxBs)
    k_pair_blocks_big<D, T, R><<<P.big_grid, kThreads, 0, s>>>(P, P.big, big_pad(P.bs), big_enc_slice(P.bs));
  else
    k_pair_blocks<D, T, R><<<(unsigned)P.nblocks, kThreads, 0, s>>>(P);
}

template <int D, bool F64, bool R64>
void launch_pair_stats(const PairParams& P, unsigned grid, cudaStream_t s) {
  using T = typename std::conditional<F64, double, float>::type;
  using R = typename std::conditional<R64, double, float>::type;
  GPZB_COUNT_LAUNCH();
  k_pair_stats<D, T, R><<<grid, kThreads, 0, s>>>(P);
  GPZB_COUNT_LAUNCH();
  k_pair_stats_final<D><<<1, 32, 0, s>>>(P, (int)grid);
}

#define DISPATCH_DPR(dims, prec, rprec, FN, ...)                                   \
  do {                                                                             \
    if (prec) {                                                                    \
      if (rprec) { if (dims == 1) FN<1, true, true>(__VA_ARGS__); else if (dims == 2) FN<2, true, true>(__VA_ARGS__); else FN<3, true, true>(__VA_ARGS__); } \
      else { if (dims == 1) FN<1, true, false>(__VA_ARGS__); else if (dims == 2) FN<2, true, false>(__VA_ARGS__); else FN<3, true, false>(__VA_ARGS__); } \
    } else {                                                                       \
      if (rprec) { if (dims == 1) FN<1, false, true>(__VA_ARGS__); else if (dims == 2) FN<2, false, true>(__VA_ARGS__); else FN<3, false, true>(__VA_ARGS__); } \
      else { if (dims == 1) FN<1, false, false>(__VA_ARGS__); else if (dims == 2) FN<2, false, false>(__VA_ARGS__); else FN<3, false, false>(__VA_ARGS__); } \
    }                                                                              \
  } while (0)

unsigned pair_stats_grid(uint64_t count) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((count + kThreads - 1) / kThreads, (uint64_t)sm_count() * 8));
}

EncParams make_enc(const void* const* axes, int dims, int prec, uint64_t count, uint32_t bs,
                   void* ws) {
  EncParams P;
  memset(&P, 0, sizeof(P));
  const uint64_t nb = nblocks_of(count, bs);
  const EncLayout L = enc_layout(nb, dims, prec, bs);
  bool vec = true;
  for (int a = 0; a < dims; ++a) {
    P.axes[a] = axes[a];
    vec = vec && ((reinterpret_cast<uintptr_t>(axes[a]) & 15) == 0);
  }
  P.count = count;
  P.nblocks = nb;
  P.bs = bs;
  P.vec = vec ? 1 : 0;
  P.res = reinterpret_cast<DevResult*>(ws);
  P.status = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + L.status);
  P.tstat = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + L.tstat);
  P.staging = static_cast<uint8_t*>(ws) + L.staging;
  P.bounds = static_cast<uint8_t*>(ws) + L.bounds;
  P.rec = reinterpret_cast<BlkRec*>(static_cast<uint8_t*>(ws) + L.rec);
  P.wide_list = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + L.list);
  P.cta_list = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + L.ctalist);
  P.small_list = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + L.slist);
  P.warp_list = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + L.wlist);
  P.big = static_cast<uint8_t*>(ws) + L.big;
  // routing switches (diagnostics / A-B runs): GPZB_ROUTE=cta sends every
  // narrow block to the general CTA encoder K2, GPZB_ROUTE=small0 sends the
  // offset-free full f32 blocks to K2s instead of the warp encoder K2p
  const char* route = getenv("GPZB_ROUTE");
  P.use_small = !(route && strcmp(route, "cta") == 0);
  P.small0 = route && strcmp(route, "small0") == 0;
  return P;
}

template <int D, bool F64>
void launch_stage_geometry(const EncParams& P, const double* lohi_in, double eb_abs, uint32_t target, AxisGeo* geo,
                           double* lohi, uint64_t* Q, uint64_t* N, uint8_t* bits, cudaStream_t s) {
  using T = typename std::conditional<F64, double, float>::type;
  const unsigned grid = (unsigned)((P.nblocks + 255) / 256);
  GPZB_COUNT_LAUNCH();
  if (lohi_in)
    k_stage_geometry<D, double><<<grid, 256, 0, s>>>(lohi_in, P.nblocks, eb_abs, target, F64, geo, lohi, Q, N, bits, P.res);
  else
    k_stage_geometry<D, T><<<grid, 256, 0, s>>>(reinterpret_cast<const T*>(P.bounds), P.nblocks, eb_abs, target, F64,
                                                geo, lohi, Q, N, bits, P.res);
}

template <int D, bool F64>
void launch_stage_quantize(const EncParams& P, const AxisGeo* geo, double eb_abs, uint64_t* seg, uint64_t* off,
                           cudaStream_t s) {
  using T = typename std::conditional<F64, double, float>::type;
  GPZB_COUNT_LAUNCH();
  k_stage_quantize<D, T><<<(unsigned)((P.count + 255) / 256), 256, 0, s>>>(P, geo, eb_abs, seg, off);
}

// Shared tail of the stage entry points: synchronise, then report the
// dataset-level finiteness error first, then the first failing block.
int stage_result(void* ws, cudaStream_t s, gpzb_result* res) {
  DevResult R;
  cudaError_t e = cudaMemcpyAsync(&R, ws, sizeof(R), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return res->status = cuda_status(e);
  res->nonfinite_mask = R.nonfinite_mask;
  if (R.nonfinite_mask) {
    res->reason = R_NONFINITE;
    res->axis = __builtin_ctz(R.nonfinite_mask);
    return res->status = GPZB_DOMAIN_ERROR;
  }
  if (R.err_block) {
    decode_err(R.err_block, &res->block, &res->axis, &res->reason);
    return res->status = status_of_reason(res->reason);
  }
  return GPZB_OK;
}

}  // namespace

extern "C" {

int gpzb_block_geometry(const void* const* axes, int dims, int prec, uint64_t count, uint32_t bs, uint32_t target,
                        double eb_abs, double* lohi, uint64_t* Q, uint64_t* N, uint8_t* log2m, void* ws,
                        uint64_t ws_bytes, void* stream, gpzb_result* res) {
  clear_result(res);
  int st = check_args(dims, prec, bs);
  if (st) return res->status = st;
  if (target == 0 || (target & (target - 1))) return res->status = GPZB_INVALID_ARGUMENT;
  const uint64_t nb = nblocks_of(count, bs);
  const EncLayout L = enc_layout(nb, dims, prec, bs);
  if (ws_bytes < L.total) return res->status = GPZB_INVALID_ARGUMENT;
  if (nb == 0) return GPZB_OK;
  cudaStream_t s = (cudaStream_t)stream;
  st = gpzb_workspace_reset_async(ws, ws_bytes, count, bs, stream);
  if (st) return res->status = st;
  EncParams P = make_enc(axes, dims, prec, count, bs, ws);
  DISPATCH_DP(dims, prec, launch_range, P, s);  // per-block bounds + finiteness (block_bounds)
  DISPATCH_DP(dims, prec, launch_stage_geometry, P, nullptr, eb_abs, target, nullptr, lohi, Q, N, log2m, s);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return res->status = cuda_status(e);
  return stage_result(ws, s, res);
}

int gpzb_quantize(const void* const* axes, int dims, int prec, uint64_t count, uint32_t bs, uint32_t target,
                  double eb_abs, const double* lohi, uint64_t* seg, uint64_t* off, void* ws, uint64_t ws_bytes,
                  void* stream, gpzb_result* res) {
  clear_result(res);
  int st = check_args(dims, prec, bs);
  if (st) return res->status = st;
  if (target == 0 || (target & (target - 1))) return res->status = GPZB_INVALID_ARGUMENT;
  const uint64_t nb = nblocks_of(count, bs);
  const EncLayout L = enc_layout(nb, dims, prec, bs);
  if (ws_bytes < L.total) return res->status = GPZB_INVALID_ARGUMENT;
  if (nb == 0) return GPZB_OK;
  static_assert(3 * sizeof(AxisGeo) <= kSlotBytes, "geometry records fit the staging slots");
  cudaStream_t s = (cudaStream_t)stream;
  st = gpzb_workspace_reset_async(ws, ws_bytes, count, bs, stream);
  if (st) return res->status = st;
  EncParams P = make_enc(axes, dims, prec, count, bs, ws);
  AxisGeo* geo = reinterpret_cast<AxisGeo*>(static_cast<uint8_t*>(ws) + L.staging);
  if (!lohi) DISPATCH_DP(dims, prec, launch_range, P, s);  // the block's own bounds
  DISPATCH_DP(dims, prec, launch_stage_geometry, P, lohi, eb_abs, target, geo, nullptr, nullptr, nullptr, nullptr, s);
  DISPATCH_DP(dims, prec, launch_stage_quantize, P, geo, eb_abs, seg, off, s);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return res->status = cuda_status(e);
  return stage_result(ws, s, res);
}

int gpzb_scan_workspace(uint64_t nblocks, uint64_t* ws_bytes) {
  *ws_bytes = enc_layout(nblocks, 1, 0).bounds;
  return GPZB_OK;
}

int gpzb_scan_sizes(const uint64_t* sizes, uint64_t nblocks, uint64_t* offsets, void* ws, uint64_t ws_bytes,
                    void* stream) {
  const EncLayout L = enc_layout(nblocks, 1, 0);
  if (ws_bytes < L.bounds) return GPZB_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(ws, 0, L.bounds, s);
  unsigned long long* sz = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + L.status);
  if (e == cudaSuccess && nblocks) e = cudaMemcpyAsync(sz, sizes, 8 * nblocks, cudaMemcpyDeviceToDevice, s);
  if (e != cudaSuccess) return cuda_status(e);
  if (nblocks == 0) return cuda_status(cudaMemsetAsync(offsets, 0, 8, s));
  CompactParams C;
  memset(&C, 0, sizeof(C));
  C.sizes = sz;
  C.tstat = reinterpret_cast<unsigned long long*>(static_cast<uint8_t*>(ws) + L.tstat);
  C.nblocks = nblocks;
  C.res = reinterpret_cast<DevResult*>(ws);
  GPZB_COUNT_LAUNCH();
  k_scan_sizes<<<(unsigned)((nblocks + kScanTile - 1) / kScanTile), kScanThreads, 0, s>>>(C);
  e = cudaGetLastError();
  // exclusive offsets (in place in the workspace), then the total
  if (e == cudaSuccess) e = cudaMemcpyAsync(offsets, sz, 8 * nblocks, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(offsets + nblocks, &C.res->total_payload, 8, cudaMemcpyDeviceToDevice, s);
  return cuda_status(e);
}

int gpzb_encode_payloads(const void* const* axes, int dims, int prec, uint64_t count, uint32_t bs, uint32_t target,
                         int pres, double eb_abs, uint8_t* payloads, uint64_t payload_cap, uint64_t* offsets, void* ws,
                         uint64_t ws_bytes, void* stream, gpzb_result* res) {
  clear_result(res);
  int st = check_args(dims, prec, bs);
  if (st) return res->status = st;
  if (target == 0 || (target & (target - 1)) || !offsets) return res->status = GPZB_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t nb = nblocks_of(count, bs);
  if (nb == 0) {
    cudaError_t e = cudaMemsetAsync(offsets, 0, 8, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return res->status = cuda_status(e);
  }
  // the compress sequence in ABS mode with the given bound (pipeline.py:38-70
  // takes eb_abs directly), then K3b with the table pointed at `offsets` and
  // no global header
  void* side = nullptr;
  uint64_t side_cap = 0;
  for (int pass = 0; pass < 2; ++pass) {
    st = gpzb_workspace_reset_async(ws, ws_bytes, count, bs, stream);
    if (!st) st = gpzb_range_async(axes, dims, prec, count, bs, ws, ws_bytes, stream);
    if (!st) st = gpzb_encode_plan_async(axes, dims, prec, count, eb_abs, GPZB_ABSOLUTE, bs, target, pres, ws, ws_bytes,
                                         stream);
    if (!st)
      st = gpzb_encode_async(axes, dims, prec, count, eb_abs, GPZB_ABSOLUTE, bs, target, pres, ws, ws_bytes,
                             static_cast<uint8_t*>(side), side_cap, nullptr, 0, 0, count, nb, 0, stream);
    if (!st) st = gpzb_compress_result(ws, ws_bytes, count, bs, stream, res);
    if (st != GPZB_NEED_SIDE || pass == 1) break;
    side_cap = res->side_bytes;
    cudaError_t e = cudaMallocAsync(&side, side_cap, s);
    if (e != cudaSuccess) { st = cuda_status(e); side = nullptr; break; }
  }
  if (!st) {
    const uint64_t total = res->out_len - GPZB_GLOBAL_HEADER_SIZE - 8 * (nb + 1);
    res->out_len = total;
    if (total > payload_cap || (total && !payloads)) {
      st = GPZB_INVALID_ARGUMENT;  // res->out_len: the bytes needed
    } else {
      EncParams P = make_enc(axes, dims, prec, count, bs, ws);
      P.side = static_cast<uint8_t*>(side);
      CompactParams C = make_compact(P, dims, prec == GPZB_F64);
      C.table0 = reinterpret_cast<uint8_t*>(offsets);
      C.table = reinterpret_cast<uint8_t*>(offsets + 1);
      C.table_base = 0;
      C.header = nullptr;
      C.payload = payloads;
      launch_emit(C, s);
      cudaError_t e = cudaGetLastError();
      if (e == cudaSuccess) e = cudaStreamSynchronize(s);
      st = cuda_status(e);
    }
  }
  if (side) cudaFreeAsync(side, s);
  if (st == GPZB_NEED_SIDE) st = GPZB_INVALID_ARGUMENT;
  if (st && !res->status) res->status = st;
  return st;
}

const char* gpzb_version(void) { return "gpzb 0.1 sm_100a"; }

uint64_t gpzb_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }



const char* gpzb_reason_message(int r) {
  switch (r) {
    case R_NONE: return "ok";
    case R_NONFINITE: return "contains non-finite coordinates";
    case R_EB_NOT_POSITIVE: return "absolute bound must be positive";
    case R_AXIS_RANGE: return "axis range over the bound exceeds 64-bit bin indices";
    case R_GEOMETRY: return "geometry needs segments x offsets beyond the 64-bit linearization range";
    case R_SHORT: return "container shorter than the 46-byte global header";
    case R_MAGIC: return "bad magic at byte 0";
    case R_VERSION: return "unsupported container version";
    case R_DIMS: return "dims outside 1..3";
    case R_ENUM: return "invalid precision or eb_mode code";
    case R_EB_ABS: return "absolute bound is not a positive real";
    case R_FLAGS: return "unknown flag bits";
    case R_TABLE_TRUNC: return "container truncated inside the offset table";
    case R_TABLE_START: return "offset table must start at 0";
    case R_TABLE_ORDER: return "offset table is not nondecreasing";
    case R_TABLE_END: return "offset table end does not match the payload length";
    case R_BLK_SHORT: return "block payload shorter than its header";
    case R_BLK_UNIQUE: return "more unique ids than particles";
    case R_BLK_WIDTH: return "stream width exceeds 64 bits";
    case R_BLK_NOSEG: return "axis has no segments";
    case R_BLK_OFFBITS: return "axis offset width exceeds 63 bits";
    case R_BLK_BOUNDS: return "axis bounds are invalid";
    case R_BLK_TRUNC: return "block truncated";
    case R_BLK_TRAILING: return "trailing bytes after block streams";
    case R_BLK_PAD_DELTA: case R_BLK_PAD_COUNT: case R_BLK_PAD_OFF: case R_BLK_PAD_RANK:
      return "nonzero padding bits in packed stream";
    case R_BLK_IDS: return "decoded unique ids are not strictly increasing";
    case R_BLK_ZERO_RUN: return "decoded run length of zero";
    case R_BLK_RUN_SUM: return "run lengths do not cover the block's particles";
    case R_BLK_RUN_MAX: return "run length beyond any block size";
    case R_BLK_AXIS_RANGE: return "axis range over the bound exceeds 64-bit bin indices";
    case R_BLK_SEGCOUNT: return "segment count inconsistent with the stored bounds";
    case R_BLK_SEG_RANGE: return "segment id outside the block geometry";
    case R_BLK_OFF_RANGE: return "segment offset outside the block geometry";
    case R_BLK_RANKS: return "rank stream is not a permutation";
    case R_BLK_COUNT: return "particle count differs from the block boundary math";
    case R_BLK_TOO_BIG: return "particle count beyond the block size";
    case R_BLK_WINDOW: return "block payload exceeds the CUDA decoder's 24 KB window (oversized stream widths)";
    case R_NONFINITE_OUT: return "contains non-finite coordinates";
    case R_TOTAL: return "blocks decode to a different particle count than the header";
    case R_UNSUPPORTED_BS: return "block_size above the CUDA kernels' limit (2^24 particles)";
    default: return "unknown";
  }
}

int gpzb_compress_bound(uint64_t count, int dims, int prec, uint32_t bs, uint32_t target, int pres,
                        uint64_t* out_bytes) {
  int st = check_args(dims, prec, bs);
  if (st) return st;
  if (target == 0 || (target & (target - 1))) return GPZB_INVALID_ARGUMENT;
  const uint64_t nb = nblocks_of(count, bs);
  const int S = prec ? 8 : 4;
  const uint64_t H = 8 + dims * (2 * S + 5) + (pres ? 4 : 3);
  // widths: deltas <= 64, counts <= bitlen(bs), offsets <= 64, ranks <= bitlen(bs-1)
  auto bl = [](uint64_t v) { int b = 0; while (v) { ++b; v >>= 1; } return (uint64_t)b; };
  const uint64_t per = H + (bs * 64ull + 7) / 8 + (bs * bl(bs) + 7) / 8 + (bs * 64ull + 7) / 8 +
                       (pres ? (bs * bl(bs - 1) + 7) / 8 : 0);
  *out_bytes = GPZB_GLOBAL_HEADER_SIZE + 8 * (nb + 1) + nb * per + 16;
  return GPZB_OK;
}

int gpzb_compress_workspace(uint64_t count, int dims, int prec, uint32_t bs, uint64_t* ws_bytes) {
  int st = check_args(dims, prec, bs);
  if (st) return st;
  *ws_bytes = enc_layout(nblocks_of(count, bs), dims, prec, bs).total;
  return GPZB_OK;
}

// Decompress workspace: result record, one DecRec per block, K4a's list and,
// for blocks of more than 1024 particles, K4b's slices.
uint64_t dec_big_bytes(const gpzb_header* h) {
  if (h->block_size <= (uint32_t)kMaxBs || h->block_count == 0) return 0;
  return big_grid(h->block_count, big_dec_slice(h->block_size)) * big_dec_slice(h->block_size);
}

int gpzb_decompress_workspace(const gpzb_header* h, uint64_t* ws_bytes) {
  *ws_bytes = align_up(sizeof(DevResult)) + align_up(h->block_count * sizeof(DecRec)) + align_up(4 * h->block_count) +
              dec_big_bytes(h);
  return GPZB_OK;
}

int gpzb_workspace_reset_async(void* ws, uint64_t ws_bytes, uint64_t count, uint32_t bs, void* stream) {
  const uint64_t nb = bs ? nblocks_of(count, bs) : 0;
  const uint64_t need = enc_layout(nb, 1, 0).bounds;  // result record, sizes, scan tile words
  if (ws_bytes < std::min<uint64_t>(need, ws_bytes) || ws_bytes < align_up(sizeof(DevResult)))
    return GPZB_INVALID_ARGUMENT;
  return cuda_status(cudaMemsetAsync(ws, 0, std::min(need, ws_bytes), (cudaStream_t)stream));
}

int gpzb_range_words(void* ws, uint64_t ws_bytes, int64_t** words) {
  if (ws_bytes < sizeof(DevResult)) return GPZB_INVALID_ARGUMENT;
  *words = reinterpret_cast<int64_t*>(&reinterpret_cast<DevResult*>(ws)->range_w[0]);
  return GPZB_OK;
}

int gpzb_range_async(const void* const* axes, int dims, int prec, uint64_t count, uint32_t bs, void* ws,
                     uint64_t ws_bytes, void* stream) {
  int st = check_args(dims, prec, bs);
  if (st) return st;
  const uint64_t nb = nblocks_of(count, bs);
  if (ws_bytes < enc_layout(nb, dims, prec, bs).total) return GPZB_INVALID_ARGUMENT;
  if (nb == 0) return GPZB_OK;
  EncParams P = make_enc(axes, dims, prec, count, bs, ws);
  DISPATCH_DP(dims, prec, launch_range, P, (cudaStream_t)stream);
  return cuda_status(cudaGetLastError());
}

int gpzb_encode_plan_async(const void* const* axes, int dims, int prec, uint64_t count, double eb, int eb_mode,
                           uint32_t bs, uint32_t target, int pres, void* ws, uint64_t ws_bytes, void* stream) {
  int st = check_args(dims, prec, bs);
  if (st) return st;
  if (target == 0 || (target & (target - 1))) return GPZB_INVALID_ARGUMENT;
  const uint64_t nb = nblocks_of(count, bs);
  if (ws_bytes < enc_layout(nb, dims, prec, bs).total) return GPZB_INVALID_ARGUMENT;
  if (nb == 0) return GPZB_OK;
  EncParams P = make_enc(axes, dims, prec, count, bs, ws);
  P.target = target;
  P.eb = eb;
  P.rel = eb_mode == GPZB_RANGE_RELATIVE;
  P.preserve = pres != 0;
  DISPATCH_DP(dims, prec, launch_geometry, P, (cudaStream_t)stream);
  return cuda_status(cudaGetLastError());
}

int gpzb_encode_async(const void* const* axes, int dims, int prec, uint64_t count, double eb, int eb_mode,
                      uint32_t bs, uint32_t target, int pres, void* ws, uint64_t ws_bytes, uint8_t* side,
                      uint64_t side_cap, uint8_t* out, uint64_t out_cap, uint64_t table_base,
                      uint64_t header_count, uint64_t header_blocks, int write_header, void* stream) {
  int st = check_args(dims, prec, bs);
  if (st) return st;
  if (target == 0 || (target & (target - 1))) return GPZB_INVALID_ARGUMENT;
  const uint64_t nb = nblocks_of(count, bs);
  if (ws_bytes < enc_layout(nb, dims, prec, bs).total) return GPZB_INVALID_ARGUMENT;
  uint64_t bound = 0;
  gpzb_compress_bound(count, dims, prec, bs, target, pres, &bound);
  if (out && out_cap < bound) return GPZB_INVALID_ARGUMENT;
  if (nb == 0) return GPZB_OK;
  EncParams P = make_enc(axes, dims, prec, count, bs, ws);
  P.target = target;
  P.eb = eb;
  P.rel = eb_mode == GPZB_RANGE_RELATIVE;
  P.eb_mode_code = eb_mode;
  P.preserve = pres != 0;
  P.side = side;
  P.side_cap = side ? side_cap : 0;
  set_out(P, out, nb, table_base, header_count, header_blocks, write_header);
  DISPATCH_DP(dims, prec, launch_encode, P, (cudaStream_t)stream);
  return cuda_status(cudaGetLastError());
}

int gpzb_emit_async(const void* const* axes, int dims, int prec, uint64_t count, double eb, int eb_mode,
                    uint32_t bs, int pres, void* ws, uint64_t ws_bytes, const uint8_t* side, uint8_t* out,
                    uint64_t out_cap, uint64_t table_base, uint64_t header_count, uint64_t header_blocks,
                    int write_header, void* stream) {
  int st = check_args(dims, prec, bs);
  if (st) return st;
  const uint64_t nb = nblocks_of(count, bs);
  if (ws_bytes < enc_layout(nb, dims, prec, bs).total) return GPZB_INVALID_ARGUMENT;
  if (!out || out_cap < GPZB_GLOBAL_HEADER_SIZE + 8 * (nb + 1)) return GPZB_INVALID_ARGUMENT;
  if (nb == 0) return GPZB_OK;
  EncParams P = make_enc(axes, dims, prec, count, bs, ws);
  P.eb = eb;
  P.eb_mode_code = eb_mode;
  P.preserve = pres != 0;
  P.side = const_cast<uint8_t*>(side);
  set_out(P, out, nb, table_base, header_count, header_blocks, write_header);
  // out_cap is the exact container (or this shard's part of it) when the caller sized it from the scan
  const uint64_t fixed = (write_header ? GPZB_GLOBAL_HEADER_SIZE : 0) + 8 * (nb + 1);
  launch_emit(make_compact(P, dims, prec == GPZB_F64), (cudaStream_t)stream, out_cap > fixed ? (out_cap - fixed) / nb : 0);
  return cuda_status(cudaGetLastError());
}

int gpzb_compress_result(void* ws, uint64_t ws_bytes, uint64_t count, uint32_t bs, void* stream,
                         gpzb_result* res) {
  clear_result(res);
  if (ws_bytes < sizeof(DevResult)) return GPZB_INVALID_ARGUMENT;
  DevResult R;
  cudaError_t e = cudaMemcpyAsync(&R, ws, sizeof(R), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) return res->status = cuda_status(e);
  const uint64_t nb = nblocks_of(count, bs);
  res->nonfinite_mask = R.nonfinite_mask;
  res->eb_abs = R.eb_abs;
  res->side_bytes = R.side_bytes;
  if (R.nonfinite_mask) {  // Dataset construction fails before any block (model.py:75-77)
    res->status = GPZB_DOMAIN_ERROR;
    res->reason = R_NONFINITE;
    res->axis = __builtin_ctz(R.nonfinite_mask);
    return res->status;
  }
  if (R.err_block) {
    decode_err(R.err_block, &res->block, &res->axis, &res->reason);
    res->status = status_of_reason(res->reason);
    return res->status;
  }
  if (R.side_need) {  // general-encoder blocks did not fit the caller's side buffer
    res->status = GPZB_NEED_SIDE;
    return res->status;
  }
  res->out_len = GPZB_GLOBAL_HEADER_SIZE + 8 * (nb + 1) + R.total_payload;
  return GPZB_OK;
}

int gpzb_encode_path_counts(void* ws, uint64_t ws_bytes, uint64_t count, uint32_t bs, int dims, int prec,
                            void* stream, uint64_t* counts) {
  if (check_args(dims, prec, bs)) return GPZB_INVALID_ARGUMENT;
  const uint64_t nb = nblocks_of(count, bs);
  const EncLayout L = enc_layout(nb, dims, prec, bs);
  if (ws_bytes < L.total) return GPZB_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* dev = &reinterpret_cast<DevResult*>(ws)->path_blocks[0];
  cudaError_t e = cudaMemsetAsync(dev, 0, 8 * sizeof(unsigned long long), s);
  if (e == cudaSuccess && nb) {
    GPZB_COUNT_LAUNCH();
    k_path_counts<<<(unsigned)std::min<uint64_t>((nb + 255) / 256, 1024), 256, 0, s>>>(
        reinterpret_cast<const BlkRec*>(static_cast<uint8_t*>(ws) + L.rec), nb, dev);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(counts, dev, 8 * sizeof(uint64_t), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return cuda_status(e);
}

int gpzb_compress(const void* const* axes, int dims, int prec, uint64_t count, double eb, int eb_mode,
                  uint32_t bs, uint32_t target, int pres, void* ws, uint64_t ws_bytes, uint8_t* out,
                  uint64_t out_cap, void* stream, gpzb_result* res) {
  clear_result(res);
  int st = check_args(dims, prec, bs);
  if (st) return res->status = st;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t nb = nblocks_of(count, bs);
  if (nb == 0) {  // empty dataset: header + one table entry (pipeline.py:75, REL uses raw eb)
    uint8_t h[GPZB_GLOBAL_HEADER_SIZE + 8];
    memset(h, 0, sizeof(h));
    memcpy(h, "GPZ1", 4);
    put_le_host(h + 4, 1, 2);
    h[6] = (uint8_t)dims;
    h[7] = (uint8_t)prec;
    h[8] = pres ? 1 : 0;
    h[9] = (uint8_t)eb_mode;
    uint64_t bits;
    memcpy(&bits, &eb, 8);
    put_le_host(h + 10, bits, 8);
    put_le_host(h + 18, bits, 8);
    put_le_host(h + 26, bs, 4);
    if (out_cap < sizeof(h)) return res->status = GPZB_INVALID_ARGUMENT;
    cudaError_t e = cudaMemcpyAsync(out, h, sizeof(h), cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) return res->status = cuda_status(e);
    res->out_len = sizeof(h);
    res->eb_abs = eb;
    return GPZB_OK;
  }
  // one pass without a side buffer; general-encoder blocks (rare) report the
  // bytes they need and the pass is repeated once with a buffer that size
  void* side = nullptr;
  uint64_t side_cap = 0;
  for (int pass = 0; pass < 2; ++pass) {
    st = gpzb_workspace_reset_async(ws, ws_bytes, count, bs, stream);
    if (!st) st = gpzb_range_async(axes, dims, prec, count, bs, ws, ws_bytes, stream);
    if (!st) st = gpzb_encode_plan_async(axes, dims, prec, count, eb, eb_mode, bs, target, pres, ws, ws_bytes, stream);
    if (!st)
      st = gpzb_encode_async(axes, dims, prec, count, eb, eb_mode, bs, target, pres, ws, ws_bytes,
                             static_cast<uint8_t*>(side), side_cap, out, out_cap, 0, count, nb, 1, stream);
    if (!st) st = gpzb_compress_result(ws, ws_bytes, count, bs, stream, res);
    if (st != GPZB_NEED_SIDE || pass == 1) break;
    side_cap = res->side_bytes;
    cudaError_t e = cudaMallocAsync(&side, side_cap, s);  // the wrapper's one allocation (stream-ordered pool)
    if (e != cudaSuccess) { st = cuda_status(e); side = nullptr; break; }
  }
  if (side) cudaFreeAsync(side, s);
  if (st == GPZB_NEED_SIDE) st = GPZB_INVALID_ARGUMENT;  // cannot happen: the second pass had the exact size
  if (st && !res->status) res->status = st;
  return st;
}

int gpzb_parse_header(const uint8_t* hb, uint64_t avail, uint64_t len, gpzb_header* h, gpzb_result* res) {
  clear_result(res);
  memset(h, 0, sizeof(*h));
  auto fail = [&](int r) { res->status = GPZB_CORRUPT_DATA; res->reason = r; return res->status; };
  if (len < GPZB_GLOBAL_HEADER_SIZE || avail < GPZB_GLOBAL_HEADER_SIZE) return fail(R_SHORT);
  if (memcmp(hb, "GPZ1", 4) != 0) return fail(R_MAGIC);
  h->version = (uint32_t)get_le_host(hb + 4, 2);
  if (h->version != 1) return fail(R_VERSION);
  h->dims = hb[6];
  if (h->dims < 1 || h->dims > 3) return fail(R_DIMS);
  h->precision = hb[7];
  const uint32_t flags = hb[8];
  h->eb_mode = hb[9];
  if (h->precision > 1 || h->eb_mode > 1) return fail(R_ENUM);
  uint64_t b = get_le_host(hb + 10, 8);
  memcpy(&h->eb, &b, 8);
  b = get_le_host(hb + 18, 8);
  memcpy(&h->eb_abs, &b, 8);
  if (!(std::isfinite(h->eb_abs) && h->eb_abs > 0)) return fail(R_EB_ABS);
  if (flags & ~1u) return fail(R_FLAGS);
  h->preserve_order = flags & 1;
  h->block_size = (uint32_t)get_le_host(hb + 26, 4);
  h->particle_count = get_le_host(hb + 30, 8);
  h->block_count = get_le_host(hb + 38, 8);
  const unsigned __int128 te = (unsigned __int128)GPZB_GLOBAL_HEADER_SIZE + ((unsigned __int128)h->block_count + 1) * 8;
  if ((unsigned __int128)len < te) return fail(R_TABLE_TRUNC);
  h->table_end = (uint64_t)te;
  h->payload_len = len - h->table_end;
  return GPZB_OK;
}

int gpzb_block_counts_async(const uint8_t* c, uint64_t len, const gpzb_header* h, uint64_t* counts, void* stream) {
  if (h->block_count == 0) return GPZB_OK;
  const unsigned grid = (unsigned)((h->block_count + 255) / 256);
  GPZB_COUNT_LAUNCH();
  k_block_counts<<<grid, 256, 0, (cudaStream_t)stream>>>(c, len, h->table_end, h->payload_len, h->block_count, h->block_size,
                                                          counts);
  return cuda_status(cudaGetLastError());
}

int gpzb_decompress_range_async(const uint8_t* c, uint64_t len, const gpzb_header* h, void* const* axes_out,
                                uint64_t out_cap, const uint64_t* out_offsets, void* ws, uint64_t ws_bytes,
                                uint64_t first_block, uint64_t last_block, int reset, void* stream) {
  if (ws_bytes < sizeof(DevResult)) return GPZB_INVALID_ARGUMENT;
  if (first_block > last_block || last_block > h->block_count) return GPZB_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  DevResult* R = reinterpret_cast<DevResult*>(ws);
  // a new decode clears the whole outcome; a further range only the list count
  cudaError_t e = reset ? cudaMemsetAsync(R, 0, sizeof(DevResult), s)
                        : cudaMemsetAsync(&R->wide_count, 0, sizeof(R->wide_count), s);
  if (e != cudaSuccess) return cuda_status(e);
  if (first_block == last_block) return GPZB_OK;
  if (h->block_count > 0x7fffffffull) return GPZB_UNSUPPORTED;
  DecParams P;
  memset(&P, 0, sizeof(P));
  P.c = c;
  P.len = len;
  P.table_end = h->table_end;
  P.payload_len = h->payload_len;
  P.nblocks = h->block_count;
  P.count = h->particle_count;
  P.bs = h->block_size;
  P.eb_abs = h->eb_abs;
  for (uint32_t a = 0; a < h->dims; ++a) P.out[a] = axes_out[a];
  P.out_cap = out_cap;
  P.out_offsets = out_offsets;
  P.res = R;
  const uint64_t list_off = align_up(sizeof(DevResult)) + align_up(h->block_count * sizeof(DecRec));
  if (ws_bytes < list_off + 4 * h->block_count) return GPZB_INVALID_ARGUMENT;
  P.rec = reinterpret_cast<DecRec*>(static_cast<uint8_t*>(ws) + align_up(sizeof(DevResult)));
  P.list = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(ws) + list_off);
  P.big = static_cast<uint8_t*>(ws) + list_off + align_up(4 * h->block_count);
  if (ws_bytes < list_off + align_up(4 * h->block_count) + dec_big_bytes(h)) return GPZB_INVALID_ARGUMENT;
  P.blk_lo = first_block;
  P.blk_hi = last_block;
  DISPATCH_DP(h->dims, h->precision, launch_decode, P, h->preserve_order != 0, s);
  return cuda_status(cudaGetLastError());
}

int gpzb_decompress_async(const uint8_t* c, uint64_t len, const gpzb_header* h, void* const* axes_out,
                          uint64_t out_cap, const uint64_t* out_offsets, void* ws, uint64_t ws_bytes,
                          void* stream) {
  return gpzb_decompress_range_async(c, len, h, axes_out, out_cap, out_offsets, ws, ws_bytes, 0,
                                     h->block_count, 1, stream);
}

int gpzb_decompress_result(void* ws, uint64_t ws_bytes, const gpzb_header* h, void* stream, gpzb_result* res) {
  clear_result(res);
  if (ws_bytes < sizeof(DevResult)) return res->status = GPZB_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  DevResult R;
  cudaError_t e = cudaMemcpyAsync(&R, ws, sizeof(R), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return res->status = cuda_status(e);
  res->table_flags = R.table_flags;
  res->nonfinite_mask = R.nonfinite_mask;
  if (R.err_block) decode_err(R.err_block, &res->decode_block, &res->decode_axis, &res->decode_reason);
  if (R.err_count) {
    int32_t ax, rs;
    decode_err(R.err_count, &res->count_block, &ax, &rs);
  }
  // precedence: read_container table checks, then the first failing block,
  // then Dataset finiteness, then the total count (pipeline.py:160-205)
  if (R.table_flags) {
    res->status = GPZB_CORRUPT_DATA;
    res->reason = (R.table_flags & 1) ? R_TABLE_START : (R.table_flags & 2) ? R_TABLE_ORDER : R_TABLE_END;
    return res->status;
  }
  int64_t fb = -1;
  if (res->decode_block >= 0) fb = res->decode_block;
  if (res->count_block >= 0 && (fb < 0 || res->count_block < fb)) fb = res->count_block;
  if (fb >= 0) {
    res->block = fb;
    if (fb == res->decode_block) {
      res->reason = res->decode_reason;
      res->axis = res->decode_axis;
    } else {
      res->reason = R_BLK_COUNT;
    }
    res->status = status_of_reason(res->reason);
    return res->status;
  }
  if (R.nonfinite_mask) {
    res->status = GPZB_DOMAIN_ERROR;
    res->reason = R_NONFINITE_OUT;
    res->axis = __builtin_ctz(R.nonfinite_mask);
    return res->status;
  }
  if (h->block_count == 0 && h->particle_count != 0) {
    res->status = GPZB_CORRUPT_DATA;
    res->reason = R_TOTAL;
    return res->status;
  }
  res->out_len = h->particle_count;
  return GPZB_OK;
}

int gpzb_decompress(const uint8_t* c, uint64_t len, const gpzb_header* h, void* const* axes_out,
                    uint64_t out_cap, const uint64_t* out_offsets, void* ws, uint64_t ws_bytes, void* stream,
                    gpzb_result* res) {
  clear_result(res);
  int st = gpzb_decompress_async(c, len, h, axes_out, out_cap, out_offsets, ws, ws_bytes, stream);
  if (st) return res->status = st;
  return gpzb_decompress_result(ws, ws_bytes, h, stream, res);
}


/* ---- K5: pairing and error-bound statistics (metrics.py:49-152) ---- */

int gpzb_pair_workspace(uint64_t count, int dims, uint64_t* ws_bytes) {
  if (dims < 1 || dims > 3) return GPZB_INVALID_ARGUMENT;
  const uint64_t ns = 1 + 3 * (uint64_t)dims;
  *ws_bytes = align_up(sizeof(DevResult)) + align_up(8 + 8 * ns) + align_up(8 * ns * pair_stats_grid(count));
  return GPZB_OK;
}

int gpzb_pair_blocks(const void* const* orig, const void* const* rec, int dims, int prec, int rprec,
                     uint64_t count, double eb_abs, uint32_t bs, uint32_t target, int64_t* orig_idx,
                     int64_t* rec_idx, void* ws, uint64_t ws_bytes, void* stream, gpzb_result* res) {
  clear_result(res);
  int st = check_args(dims, prec, bs);
  if (st) return res->status = st;
  if ((rprec != GPZB_F32 && rprec != GPZB_F64) || target == 0 || (target & (target - 1)))
    return res->status = GPZB_INVALID_ARGUMENT;
  if (ws_bytes < sizeof(DevResult)) return res->status = GPZB_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  if (count == 0) return GPZB_OK;
  PairParams P;
  memset(&P, 0, sizeof(P));
  for (int a = 0; a < dims; ++a) { P.orig[a] = orig[a]; P.rec[a] = rec[a]; }
  P.count = count;
  P.nblocks = nblocks_of(count, bs);
  P.bs = bs;
  P.target = target;
  P.eb_abs = eb_abs;
  P.orig_idx = orig_idx;
  P.rec_idx = rec_idx;
  P.res = reinterpret_cast<DevResult*>(ws);
  cudaError_t e = cudaMemsetAsync(ws, 0, sizeof(DevResult), s);
  if (e != cudaSuccess) return res->status = cuda_status(e);
  void* big = nullptr;
  if (bs > (uint32_t)kMaxBs) {
    // blocks above 1024 particles: per-CTA key slices, the call's one
    // allocation (stream-ordered pool), freed behind the kernel
    const uint64_t slice = big_enc_slice(bs), grid = big_grid(P.nblocks, slice);
    e = cudaMallocAsync(&big, grid * slice, s);
    if (e != cudaSuccess) return res->status = cuda_status(e);
    P.big = static_cast<uint8_t*>(big);
    P.big_grid = (uint32_t)grid;
  }
  DISPATCH_DPR(dims, prec, rprec, launch_pair_blocks, P, s);
  e = cudaGetLastError();
  if (big) cudaFreeAsync(big, s);
  DevResult R;
  if (e == cudaSuccess) e = cudaMemcpyAsync(&R, ws, sizeof(R), cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return res->status = cuda_status(e);
  res->nonfinite_mask = R.nonfinite_mask;
  if (R.nonfinite_mask) {  // the Dataset invariant (model.py:75-77): original axes first
    res->status = GPZB_DOMAIN_ERROR;
    res->reason = R_NONFINITE;
    const uint32_t m = (R.nonfinite_mask & 7) ? (R.nonfinite_mask & 7) : (R.nonfinite_mask >> 4);
    res->axis = __builtin_ctz(m);
    return res->status;
  }
  if (R.err_block) {
    decode_err(R.err_block, &res->block, &res->axis, &res->reason);
    res->status = status_of_reason(res->reason);
    return res->status;
  }
  return GPZB_OK;
}

int gpzb_pair_stats(const void* const* orig, const void* const* rec, int dims, int prec, int rprec,
                    uint64_t count, const int64_t* orig_idx, const int64_t* rec_idx, double eb_abs,
                    uint64_t* viol, uint64_t viol_cap, void* ws, uint64_t ws_bytes, void* stream,
                    double* stats, uint64_t* viol_count) {
  uint64_t need = 0;
  if (gpzb_pair_workspace(count, dims, &need) || ws_bytes < need) return GPZB_INVALID_ARGUMENT;
  if ((prec != GPZB_F32 && prec != GPZB_F64) || (rprec != GPZB_F32 && rprec != GPZB_F64))
    return GPZB_INVALID_ARGUMENT;
  cudaStream_t s = (cudaStream_t)stream;
  const uint64_t ns = 1 + 3 * (uint64_t)dims;
  uint8_t* base = static_cast<uint8_t*>(ws);
  PairParams P;
  memset(&P, 0, sizeof(P));
  for (int a = 0; a < dims; ++a) { P.orig[a] = orig[a]; P.rec[a] = rec[a]; }
  P.count = count;
  P.eb_abs = eb_abs;
  P.orig_idx = const_cast<int64_t*>(orig_idx);
  P.rec_idx = const_cast<int64_t*>(rec_idx);
  P.viol_count = reinterpret_cast<unsigned long long*>(base + align_up(sizeof(DevResult)));
  P.out = reinterpret_cast<double*>(base + align_up(sizeof(DevResult)) + 8);
  P.partial = reinterpret_cast<double*>(base + align_up(sizeof(DevResult)) + align_up(8 + 8 * ns));
  P.viol = reinterpret_cast<unsigned long long*>(viol);
  P.viol_cap = viol ? viol_cap : 0;
  const unsigned grid = pair_stats_grid(count);
  cudaError_t e = cudaMemsetAsync(P.viol_count, 0, 8, s);
  if (e != cudaSuccess) return cuda_status(e);
  DISPATCH_DPR(dims, prec, rprec, launch_pair_stats, P, grid, s);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(stats, P.out, 8 * ns, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaMemcpyAsync(viol_count, P.viol_count, 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  return cuda_status(e);
}

}  // extern "C"
