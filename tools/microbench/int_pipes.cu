// INT32 pipe-rate microbenchmark for sm_100a (B200).
//
// Measures the issue rate (warp-instructions per SM per SM-cycle) of the integer
// instructions the alignment kernel is built from, so that the roofline in
// DESIGN.md rests on measured numbers rather than guesses.  Each thread runs NCH
// independent dependency chains so that latency is hidden; every block records
// its SM-cycle span with clock64(), and the rate is total warp-instructions /
// (num_SMs x max block span).
//
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o int_pipes int_pipes.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>

#define NCH 8
#define ITERS 4096

enum Op {
  OP_IADD, OP_IMNMX, OP_VIADDMAX, OP_VIADDMIN, OP_VIMAX3, OP_IMAD, OP_IMADHI, OP_PRMT, OP_LOP3,
  OP_SHF, OP_MIX_MAX_IMAD, OP_MIX_VIADD_IMADHI, OP_MIX3_VIADD_VIMAX3_IMAD, OP_SHFL, OP_REDUX, OP_MIX_CELL, OP_NOPS
};
static const char* kOpName[] = {
  "IADD3(add.s32)", "IMNMX(max.s32)", "VIADDMNMX(__viaddmax_s32)", "VIADDMNMX(__viaddmin_s32)",
  "VIMNMX3(__vimax3_s32)", "IMAD(mad.lo)", "IMAD.HI(mad.hi)", "PRMT", "LOP3", "SHF(funnel)",
  "mix: IMNMX+IMAD 1:1", "mix: VIADDMNMX+IMAD.HI 1:1", "mix: VIADDMNMX+VIMNMX3+IMAD 1:1:1",
  "SHFL.IDX", "REDUX.MAX", "mix cell: 2xVIADDMNMX+2xVIMNMX3+VIADDMIN (ALU) : 2xIMAD+IMAD.HI (FMA)"};

template <int OP>
__global__ void __launch_bounds__(256) bench(const int* __restrict__ in, int* __restrict__ out,
                                             unsigned long long* __restrict__ span) {
  int a[NCH];
  const int b = in[0], c = in[1], d = in[2];
#pragma unroll
  for (int k = 0; k < NCH; ++k) a[k] = in[3 + k] + threadIdx.x;
  __syncthreads();
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int k = 0; k < NCH; ++k) {
      if (OP == OP_IADD) {
        asm volatile("add.s32 %0, %0, %1;" : "+r"(a[k]) : "r"(b));
      } else if (OP == OP_IMNMX) {
        asm volatile("max.s32 %0, %0, %1;" : "+r"(a[k]) : "r"(b + k));
      } else if (OP == OP_VIADDMAX) {
        a[k] = __viaddmax_s32(a[k], b, c + k);
      } else if (OP == OP_VIADDMIN) {
        a[k] = __viaddmin_s32(a[k], b, c + k);
      } else if (OP == OP_VIMAX3) {
        a[k] = __vimax3_s32(a[k], b + k, c);
      } else if (OP == OP_IMAD) {
        asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
      } else if (OP == OP_IMADHI) {
        asm volatile("mad.hi.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
      } else if (OP == OP_PRMT) {
        asm volatile("prmt.b32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
      } else if (OP == OP_LOP3) {
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[k]) : "r"(b), "r"(c));
      } else if (OP == OP_SHF) {
        asm volatile("shf.r.wrap.b32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
      } else if (OP == OP_MIX_MAX_IMAD) {
        if (k & 1) asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
        else asm volatile("max.s32 %0, %0, %1;" : "+r"(a[k]) : "r"(b + k));
      } else if (OP == OP_MIX_VIADD_IMADHI) {
        if (k & 1) asm volatile("mad.hi.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
        else a[k] = __viaddmax_s32(a[k], b, c + k);
      } else if (OP == OP_MIX3_VIADD_VIMAX3_IMAD) {
        if (k % 3 == 0) a[k] = __viaddmax_s32(a[k], b, c + k);
        else if (k % 3 == 1) a[k] = __vimax3_s32(a[k], b + k, c);
        else asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
      } else if (OP == OP_SHFL) {
        a[k] = __shfl_sync(0xffffffffu, a[k], (threadIdx.x + 1) & 31);
      } else if (OP == OP_MIX_CELL) {
        const int r = k & 7;
        if (r == 0 || r == 1) a[k] = __viaddmax_s32(a[k], b, c + k);
        else if (r == 2 || r == 7) a[k] = __vimax3_s32(a[k], b + k, c);
        else if (r == 3) a[k] = __viaddmin_s32(a[k], b, c + k);
        else if (r == 5) asm volatile("mad.hi.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
        else asm volatile("mad.lo.s32 %0, %0, %1, %2;" : "+r"(a[k]) : "r"(b), "r"(c));
      } else if (OP == OP_REDUX) {
        a[k] = __reduce_max_sync(0xffffffffu, a[k] + d);
      }
    }
  }
  unsigned long long t1 = clock64();
  int s = 0;
#pragma unroll
  for (int k = 0; k < NCH; ++k) s ^= a[k];
  if (s == 0x7fffffff) out[threadIdx.x] = s;  // keep results live
  if (threadIdx.x == 0) span[blockIdx.x] = t1 - t0;
}

template <int OP>
static void run(int nsm, int blocks_per_sm, int threads, const int* din, int* dout,
                unsigned long long* dspan) {
  int grid = nsm * blocks_per_sm;
  bench<OP><<<grid, threads>>>(din, dout, dspan);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  bench<OP><<<grid, threads>>>(din, dout, dspan);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long* hspan = new unsigned long long[grid];
  cudaMemcpy(hspan, dspan, sizeof(unsigned long long) * grid, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0;
  double mean = 0;
  for (int i = 0; i < grid; ++i) {
    if (hspan[i] > mx) mx = hspan[i];
    mean += hspan[i];
  }
  mean /= grid;
  delete[] hspan;
  double warp_instr = (double)grid * (threads / 32) * (double)ITERS * NCH;
  double per_sm_per_clk = warp_instr / nsm / (double)mx;  // warp-instr / SM / cycle
  double clk_ghz = (double)mx / (ms * 1e6);
  printf("{\"op\": \"%s\", \"warps_per_sm\": %d, \"warp_instr_per_sm_per_clk\": %.3f, "
         "\"lane_ops_per_sm_per_clk\": %.1f, \"ms\": %.3f, \"sm_clk_ghz_est\": %.3f, "
         "\"span_mean_over_max\": %.3f}\n",
         kOpName[OP], blocks_per_sm * threads / 32, per_sm_per_clk, per_sm_per_clk * 32, ms, clk_ghz,
         mean / mx);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("CUDA error %s\n", cudaGetErrorString(err));
}

int main() {
  int dev = 0, nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  int hin[16];
  for (int i = 0; i < 16; ++i) hin[i] = 3 + 7 * i;
  hin[0] = 0x01234567;
  hin[1] = 0x00003210;
  hin[2] = 1;
  int *din, *dout;
  unsigned long long* dspan;
  cudaMalloc(&din, sizeof(hin));
  cudaMalloc(&dout, 1024 * sizeof(int));
  cudaMalloc(&dspan, sizeof(unsigned long long) * nsm * 64);
  cudaMemcpy(din, hin, sizeof(hin), cudaMemcpyHostToDevice);
  for (int occ : {4, 8}) {  // blocks of 256 threads per SM -> 32 / 64 warps per SM
    run<OP_IADD>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_IMNMX>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_VIADDMAX>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_VIADDMIN>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_VIMAX3>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_IMAD>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_IMADHI>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_PRMT>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_LOP3>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_SHF>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_MIX_MAX_IMAD>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_MIX_VIADD_IMADHI>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_MIX3_VIADD_VIMAX3_IMAD>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_SHFL>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_REDUX>(nsm, occ / 2, 256, din, dout, dspan);
    run<OP_MIX_CELL>(nsm, occ / 2, 256, din, dout, dspan);
  }
  printf("{\"num_sms\": %d}\n", nsm);
  return 0;
}
