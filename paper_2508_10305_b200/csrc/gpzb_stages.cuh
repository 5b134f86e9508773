// Stage-level kernels behind the per-stage C entry points (include/gpzb.h
// "stage-level entry points"): the block geometry, the quantized codes in
// input order and the payload-length scan, each callable on its own so a
// caller can compare one stage at a time with the reference:
//
//   gpzb_block_geometry  <- quantizer.block_bounds + derive_geometry  quantizer.py:51-129
//   gpzb_quantize        <- quantizer.quantize_block (codes in input order,
//                           optionally with carried block bounds)      quantizer.py:223-247
//   gpzb_scan_sizes      <- container.compact's prefix sum             container.py:203-208
//
// The compress path itself never calls these: there the same functions are
// fused into K1.5 / K2* / K3a.
#pragma once

#include "gpzb_compact.cuh"

namespace gpzb {

// One thread per block: geometry from per-block bounds (input precision TB)
// in derive_geometry's order of checks (quantizer.py:98-129).
template <int D, typename TB>
__global__ void k_stage_geometry(const TB* bounds, uint64_t nblocks, double eb_abs, uint32_t target, bool f64,
                                 AxisGeo* geo, double* lohi, uint64_t* Q, uint64_t* N, uint8_t* bits,
                                 DevResult* R) {
  const uint64_t blk = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (blk >= nblocks) return;
  int err = R_NONE, eax = 0;
  AxisGeo g[D];
  if (!(eb_abs > 0.0)) {
    err = R_EB_NOT_POSITIVE;
  } else {
#pragma unroll
    for (int a = 0; a < D; ++a) {
      if (!err && axis_geometry((double)bounds[(blk * D + a) * 2], (double)bounds[(blk * D + a) * 2 + 1], eb_abs, f64,
                                target, g[a])) {
        err = R_AXIS_RANGE;
        eax = a;
      }
    }
  }
  if (!err) {
    unsigned __int128 PN = 1;
    uint32_t sumb = 0;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      PN *= g[a].N;
      if (PN > ((unsigned __int128)1 << 64)) break;
      sumb += g[a].b;
    }
    if (PN > ((unsigned __int128)1 << 64) || sumb > 64) err = R_GEOMETRY;
  }
  if (err) {
    atomicMax(&R->err_block, err_code(blk, eax, err));
    return;
  }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const uint64_t i = blk * D + a;
    if (geo) geo[i] = g[a];
    if (lohi) { lohi[2 * i] = g[a].lo; lohi[2 * i + 1] = g[a].hi; }
    if (Q) Q[i] = g[a].Q;
    if (N) N[i] = g[a].N;
    if (bits) bits[i] = (uint8_t)g[a].b;
  }
}

// One thread per particle: bin index per axis with the reference's exact
// rule (certified reciprocal / exact division / edge snap, quantizer.py:142-173)
// and the (segment, offset) linearisation (quantizer.py:176-191), u64 each.
template <int D, typename T>
__global__ void k_stage_quantize(const EncParams P, const AxisGeo* geo, double eb_abs, uint64_t* seg,
                                 uint64_t* off) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= P.count) return;
  const uint64_t blk = i / P.bs;
  uint64_t s = 0, o = 0, stride = 1;
  uint32_t shift = 0, nf = 0;
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const AxisGeo& g = geo[blk * D + a];
    const double x = (double)reinterpret_cast<const T*>(P.axes[a])[i];
    if (!isfinite(x)) nf |= 1u << a;
    const uint64_t q = quantize_coord(x, g, eb_abs, sizeof(T) == 8);
    s += shr64(q, g.b) * stride;
    o |= shl64(q & mask64(g.b), shift);
    stride *= g.N;
    shift += g.b;
  }
  if (nf) atomicOr(&P.res->nonfinite_mask, nf);
  seg[i] = s;
  off[i] = o;
}

}  // namespace gpzb
