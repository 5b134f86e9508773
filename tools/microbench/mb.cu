// Microbenchmarks that decide the encode-kernel design on B200 (sm_100a).
// Each kernel runs one full wave and reports lane-ops per SM-cycle, measured
// with clock64 inside each CTA (so DVFS does not enter the ratio).
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cub/block/block_radix_sort.cuh>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1);} } while (0)

__device__ unsigned long long g_cycles[4096];
__device__ unsigned g_sink[4096];

// ---- quantize variants: 1024 particles x 3 axes per CTA-iteration -------
__device__ __forceinline__ double f2d_int(float f) {
  uint32_t u = __float_as_uint(f);
  uint32_t e = (u >> 23) & 0xff;
  uint32_t hi = (u & 0x80000000u) | ((e + 896u) << 20) | ((u >> 3) & 0xfffffu);
  uint32_t lo = u << 29;
  hi = e ? hi : (u & 0x80000000u);   // zero (denormals not handled here)
  return __hiloint2double(hi, lo);
}

template <int MODE>
__global__ void k_quant(int iters, float lo_f, double rinv) {
  __shared__ float xs[3072];
  for (int i = threadIdx.x; i < 3072; i += blockDim.x) xs[i] = lo_f + 0.001f * (i % 977);
  __syncthreads();
  const double lo = (double)lo_f;
  const double magic = 4503599627370496.0;  // 2^52
  unsigned acc = 0, bad = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 4
    for (int j = threadIdx.x; j < 3072; j += 256) {
      float f = xs[j];
      double x = MODE == 0 ? (double)f : f2d_int(f);
      double t = __dsub_rn(x, lo);
      double r = __dmul_rn(t, rinv);
      double y = __dadd_rz(r, magic);
      unsigned q = (unsigned)__double2loint(y);
      unsigned rl = (unsigned)__double2loint(r);
      bad += (rl + 1u) <= 1u;
      acc ^= q + it;
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[(blockIdx.x * 256 + threadIdx.x) & 4095] = acc + bad;
}

// ---- shared-memory atomics -------------------------------------------------
template <int OP>
__global__ void k_atoms(int iters) {
  __shared__ unsigned c[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) c[i] = 0;
  __syncthreads();
  unsigned h = threadIdx.x * 2654435761u;
  unsigned long long t0 = clock64();
  unsigned acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int k = 0; k < 8; ++k) {
      unsigned a = (h + (it * 8 + k) * 40503u) >> 21;  // 0..2047, spread
      if (OP == 0) acc += atomicAdd(&c[a], 1u);
      else if (OP == 1) atomicOr(&c[a], 1u << (k & 31));
      else acc += atomicAdd(&c[(threadIdx.x & 31) * 64 + k], 1u);  // distinct banks? no: stride 64
    }
  }
  unsigned long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[(blockIdx.x * 256 + threadIdx.x) & 4095] = acc + c[threadIdx.x];
}

// ---- match.any ---------------------------------------------------------------
__global__ void k_match(int iters) {
  unsigned h = threadIdx.x * 2654435761u;
  unsigned acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int k = 0; k < 8; ++k) {
      unsigned key = (h + (it * 8 + k) * 40503u) >> 24;
      acc += __match_any_sync(0xffffffffu, key);
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[(blockIdx.x * 256 + threadIdx.x) & 4095] = acc;
}

// ---- FP64 add throughput -----------------------------------------------------
__global__ void k_dadd(int iters) {
  double a0 = threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const double s = 1e-9;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    a0 = __dadd_rn(a0, s); a1 = __dadd_rn(a1, s); a2 = __dadd_rn(a2, s); a3 = __dadd_rn(a3, s);
    a4 = __dadd_rn(a4, s); a5 = __dadd_rn(a5, s); a6 = __dadd_rn(a6, s); a7 = __dadd_rn(a7, s);
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[(blockIdx.x * 256 + threadIdx.x) & 4095] = (unsigned)(a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7);
}

// ---- F2F.F64.F32 throughput ---------------------------------------------------
__global__ void k_f2f(int iters) {
  float f[8];
  for (int k = 0; k < 8; ++k) f[k] = threadIdx.x + k;
  unsigned acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      double d = (double)f[k];
      acc ^= __double2hiint(d);
      f[k] = __int_as_float(__float_as_int(f[k]) + 1);
    }
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[(blockIdx.x * 256 + threadIdx.x) & 4095] = acc;
}

// ---- CUB block radix sort of 1024 keys --------------------------------------
template <int BITS>
__global__ void k_cubsort(int iters) {
  using Sort = cub::BlockRadixSort<uint32_t, 256, 4>;
  __shared__ typename Sort::TempStorage tmp;
  uint32_t keys[4];
  unsigned h = (blockIdx.x * 256 + threadIdx.x) * 2654435761u;
  unsigned acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < 4; ++k) { h = h * 1664525u + 1013904223u; keys[k] = h >> (32 - BITS); }
    Sort(tmp).Sort(keys, 0, BITS);
    acc += keys[0] ^ keys[3];
    __syncthreads();
  }
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) g_cycles[blockIdx.x] = t1 - t0;
  g_sink[(blockIdx.x * 256 + threadIdx.x) & 4095] = acc;
}


template <typename L>
static void run(const char* name, L launch, int ctas_per_sm, int iters, double lane_ops_per_iter_per_cta) {
  int grid = 148 * ctas_per_sm;
  launch(grid, iters);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  launch(grid, iters);
  cudaEventRecord(b);
  CK(cudaDeviceSynchronize());
  float ms; cudaEventElapsedTime(&ms, a, b);
  static unsigned long long cyc[4096];
  CK(cudaMemcpyFromSymbol(cyc, g_cycles, sizeof(unsigned long long) * grid));
  double mean = 0; for (int i = 0; i < grid; ++i) mean += cyc[i]; mean /= grid;
  double per_sm_cycle = ctas_per_sm * lane_ops_per_iter_per_cta * iters / mean;
  printf("%-30s ctas/sm=%d cyc/cta-iter=%9.1f  ops/SM/cyc=%7.2f  (%.3f ms, clk~%.0f MHz)\n", name,
         ctas_per_sm, mean / iters, per_sm_cycle, ms, mean / (ms * 1e3));
}

int main() {
  int dev; cudaGetDevice(&dev);
  cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  printf("%s  SMs=%d  cc=%d.%d\n", p.name, p.multiProcessorCount, p.major, p.minor);
  const double rinv = 1.0 / 0.00213;
  for (int occ : {2, 4, 8}) {
    run("quant F2F (coords)", [&](int g, int it) { k_quant<0><<<g, 256>>>(it, 0.5f, rinv); }, occ, 200, 3072);
    run("quant int-cvt (coords)", [&](int g, int it) { k_quant<1><<<g, 256>>>(it, 0.5f, rinv); }, occ, 200, 3072);
  }
  for (int occ : {4, 8}) {
    run("atoms add spread", [&](int g, int it) { k_atoms<0><<<g, 256>>>(it); }, occ, 200, 256 * 8);
    run("atoms or spread", [&](int g, int it) { k_atoms<1><<<g, 256>>>(it); }, occ, 200, 256 * 8);
    run("atoms add stride64(conflict)", [&](int g, int it) { k_atoms<2><<<g, 256>>>(it); }, occ, 200, 256 * 8);
    run("match.any 8-bit", [&](int g, int it) { k_match<<<g, 256>>>(it); }, occ, 200, 256 * 8);
    run("dadd", [&](int g, int it) { k_dadd<<<g, 256>>>(it); }, occ, 2000, 256 * 8);
    run("f2f.f64.f32", [&](int g, int it) { k_f2f<<<g, 256>>>(it); }, occ, 2000, 256 * 8);
  }
  for (int occ : {2, 4}) {
    run("cub sort 1024x u32 8 bits (keys)", [&](int g, int it) { k_cubsort<8><<<g, 256>>>(it); }, occ, 50, 1024);
    run("cub sort 1024x u32 16 bits (keys)", [&](int g, int it) { k_cubsort<16><<<g, 256>>>(it); }, occ, 50, 1024);
    run("cub sort 1024x u32 24 bits (keys)", [&](int g, int it) { k_cubsort<24><<<g, 256>>>(it); }, occ, 50, 1024);
    run("cub sort 1024x u32 32 bits (keys)", [&](int g, int it) { k_cubsort<32><<<g, 256>>>(it); }, occ, 50, 1024);
  }
  return 0;
}
