// Which pipe runs fp16x2 min/max (HMNMX2) on sm_100a, and is it exact as an ordered
// max of non-negative int16 bit patterns?  (the align kernel is
// ALU-pipe bound; a pure max/min moved to another pipe frees ALU issue.)
//
// Rates: warp-instructions per SM per cycle over 8 independent chains per thread, for
// VIMNMX.S16x2 alone, HMNMX2 alone, 1:1 mixes with VIMNMX.S16x2 / VIADDMNMX.S16x2 / IMAD.
// A 1:1 mix that issues ~2x the rate of either alone means separate pipes.
// Exactness: max.f16x2 vs integer max on all pairs of a grid of patterns in [0, 0x7BFF].
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmnmx hmnmx.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define NCH 8
#define ITERS 4096

__device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t hmin2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("min.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t vmax2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm volatile("max.s16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t vaddmax2(uint32_t a, uint32_t b, uint32_t c) {
  return __viaddmax_s16x2(a, b, c);
}
__device__ __forceinline__ uint32_t imad(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t d;
  asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
  return d;
}

enum { OP_VMAX2, OP_HMAX2, OP_HMIN2, OP_MIX_V_H, OP_MIX_VADD_H, OP_MIX_IMAD_H, OP_MIX_VADD_IMAD, OP_N };
static const char* kName[] = {"VIMNMX.S16x2 (max.s16x2)", "HMNMX2 (max.f16x2)", "HMNMX2 (min.f16x2)",
                              "mix max.s16x2 : max.f16x2 1:1", "mix VIADDMNMX.S16x2 : max.f16x2 1:1",
                              "mix IMAD : max.f16x2 1:1", "mix VIADDMNMX.S16x2 : IMAD 1:1"};

template <int OP>
__global__ void __launch_bounds__(256) bench(const uint32_t* __restrict__ in, uint32_t* __restrict__ out,
                                             unsigned long long* __restrict__ span) {
  uint32_t a[NCH];
  const uint32_t b = in[0], c = in[1];
#pragma unroll
  for (int k = 0; k < NCH; ++k) a[k] = in[2 + k] + threadIdx.x;
  __syncthreads();
  const unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      if (OP == OP_VMAX2) a[k] = vmax2(a[k], b + k);
      else if (OP == OP_HMAX2) a[k] = hmax2(a[k], b + k);
      else if (OP == OP_HMIN2) a[k] = hmin2(a[k], b + k);
      else if (OP == OP_MIX_V_H) a[k] = (k & 1) ? hmax2(a[k], b + k) : vmax2(a[k], b + k);
      else if (OP == OP_MIX_VADD_H) a[k] = (k & 1) ? hmax2(a[k], b + k) : vaddmax2(a[k], b, c + k);
      else if (OP == OP_MIX_IMAD_H) a[k] = (k & 1) ? hmax2(a[k], b + k) : imad(a[k], b, c + k);
      else a[k] = (k & 1) ? imad(a[k], b, c + k) : vaddmax2(a[k], b, c + k);
    }
  }
  const unsigned long long t1 = clock64();
  uint32_t s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s ^= a[k];
  if (s == 0x7fffffffu) out[threadIdx.x] = s;
  if (threadIdx.x == 0) span[blockIdx.x] = t1 - t0;
}

// exactness: for patterns x, y in [lo, hi] (both halves), max.f16x2 == integer max?
__global__ void exact(uint32_t lo, uint32_t hi, uint32_t step, unsigned long long* bad, unsigned long long* tot) {
  unsigned long long nb = 0, nt = 0;
  for (uint32_t x = lo + (blockIdx.x * blockDim.x + threadIdx.x) * step; x <= hi;
       x += gridDim.x * blockDim.x * step) {
    for (uint32_t y = lo; y <= hi; y += 7) {
      const uint32_t a = x | (y << 16), b = y | (x << 16);
      const uint32_t m = hmax2(a, b), n = hmin2(a, b);
      const uint32_t mx = x > y ? x : y, mn = x < y ? x : y;
      nb += (m != (mx | (mx << 16))) + (n != (mn | (mn << 16)));
      nt += 2;
    }
  }
  atomicAdd(bad, nb);
  atomicAdd(tot, nt);
}

template <int OP>
static void run(int nsm, const uint32_t* din, uint32_t* dout, unsigned long long* dspan) {
  const int bps = 4, threads = 256, grid = nsm * bps;
  bench<OP><<<grid, threads>>>(din, dout, dspan);
  bench<OP><<<grid, threads>>>(din, dout, dspan);
  cudaDeviceSynchronize();
  unsigned long long h[4096];
  cudaMemcpy(h, dspan, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
  const double wi = (double)grid * (threads / 32) * ITERS * NCH;
  printf("{\"op\": \"%s\", \"warp_instr_per_sm_per_clk\": %.3f, \"lanes_per_sm_per_clk\": %.1f}\n",
         kName[OP], wi / nsm / mx, 32.0 * wi / nsm / mx);
}

int main() {
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  uint32_t hin[16];
  for (int i = 0; i < 16; ++i) hin[i] = 0x12340000u + 0x01010101u * i;
  uint32_t *din, *dout;
  unsigned long long* dspan;
  cudaMalloc(&din, sizeof(hin));
  cudaMalloc(&dout, 4096);
  cudaMalloc(&dspan, 8 * 4096);
  cudaMemcpy(din, hin, sizeof(hin), cudaMemcpyHostToDevice);
  run<OP_VMAX2>(nsm, din, dout, dspan);
  run<OP_HMAX2>(nsm, din, dout, dspan);
  run<OP_HMIN2>(nsm, din, dout, dspan);
  run<OP_MIX_V_H>(nsm, din, dout, dspan);
  run<OP_MIX_VADD_H>(nsm, din, dout, dspan);
  run<OP_MIX_IMAD_H>(nsm, din, dout, dspan);
  run<OP_MIX_VADD_IMAD>(nsm, din, dout, dspan);
  unsigned long long *dbad, *dtot, hb, ht;
  cudaMalloc(&dbad, 8);
  cudaMalloc(&dtot, 8);
  const uint32_t ranges[3][2] = {{0x0000, 0x7BFF}, {0x0400, 0x7BFF}, {0x0000, 0x03FF}};
  for (auto& r : ranges) {
    cudaMemset(dbad, 0, 8);
    cudaMemset(dtot, 0, 8);
    exact<<<1184, 256>>>(r[0], r[1], 3, dbad, dtot);
    cudaMemcpy(&hb, dbad, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&ht, dtot, 8, cudaMemcpyDeviceToHost);
    printf("{\"exactness\": \"max/min.f16x2 vs int max/min\", \"range\": [%u, %u], \"checked\": %llu, \"wrong\": %llu}\n",
           r[0], r[1], ht, hb);
  }
  return 0;
}
