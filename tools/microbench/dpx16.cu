// DPX 16x2 semantics (wrap vs saturate) and throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void sem(unsigned* o) {
  // lane values: a = 0x7FFF (32767) in lo, 0x8000 (-32768) in hi; b = +1 lo, -1 hi
  unsigned a = 0x80007FFFu, b = 0xFFFF0001u, c = 0x80008000u;  // c = (-32768, -32768)
  o[0] = __viaddmax_s16x2(a, b, c);   // wrap: lo 32767+1=-32768, hi -32768-1=32767
  o[1] = __viaddmin_s16x2(a, b, 0x7FFF7FFFu);
  o[2] = __vmaxs2(a, 0u);
  o[3] = __vimax3_s16x2(a, b, c);
}
template <int OP>
__global__ void thr(const unsigned* in, unsigned* out, unsigned long long* span) {
  unsigned a[8]; const unsigned b = in[0], c = in[1];
  for (int k = 0; k < 8; ++k) a[k] = in[2 + k] + threadIdx.x;
  unsigned long long t0 = clock64();
#pragma unroll 1
  for (int it = 0; it < 4096; ++it) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (OP == 0) a[k] = __viaddmax_s16x2(a[k], b, c + k);
      else if (OP == 1) a[k] = __vimax3_s16x2(a[k], b + k, c);
      else if (OP == 2) a[k] = __vmaxs2(a[k], b + k);
      else a[k] = __viaddmin_s16x2(a[k], b, c + k);
    }
  }
  unsigned long long t1 = clock64();
  unsigned s = 0; for (int k = 0; k < 8; ++k) s ^= a[k];
  if (s == 0x12345678u) out[threadIdx.x] = s;
  if (threadIdx.x == 0) span[blockIdx.x] = t1 - t0;
}
template <int OP> void run(const char* name, int nsm, unsigned* din, unsigned* dout, unsigned long long* dspan) {
  int grid = nsm * 4;
  thr<OP><<<grid, 256>>>(din, dout, dspan);
  thr<OP><<<grid, 256>>>(din, dout, dspan);
  cudaDeviceSynchronize();
  unsigned long long* h = new unsigned long long[grid];
  cudaMemcpy(h, dspan, 8 * grid, cudaMemcpyDeviceToHost);
  unsigned long long mx = 0; for (int i = 0; i < grid; ++i) if (h[i] > mx) mx = h[i];
  double wi = (double)grid * 8 * 4096 * 8;
  printf("{\"op\": \"%s\", \"lane_ops_per_sm_per_clk\": %.1f}\n", name, wi / nsm / mx * 32);
  delete[] h;
}
int main() {
  unsigned* o; cudaMalloc(&o, 64); sem<<<1, 1>>>(o); unsigned h[4];
  cudaMemcpy(h, o, 16, cudaMemcpyDeviceToHost);
  printf("{\"viaddmax_s16x2(0x80007FFF, 0xFFFF0001, 0x80008000)\": \"0x%08x\", \"note\": \"0x7fff8000 = wrap, 0x80007fff = saturate\"}\n", h[0]);
  printf("{\"viaddmin_s16x2\": \"0x%08x\", \"vmaxs2\": \"0x%08x\", \"vimax3\": \"0x%08x\"}\n", h[1], h[2], h[3]);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  unsigned hin[16]; for (int i = 0; i < 16; ++i) hin[i] = 0x00010002u * (i + 1);
  unsigned *din, *dout; unsigned long long* dspan;
  cudaMalloc(&din, 64); cudaMalloc(&dout, 4096); cudaMalloc(&dspan, 8 * nsm * 8);
  cudaMemcpy(din, hin, 64, cudaMemcpyHostToDevice);
  run<0>("VIADDMNMX.S16x2", nsm, din, dout, dspan);
  run<1>("VIMNMX3.S16x2", nsm, din, dout, dspan);
  run<2>("VIMNMX.S16x2 (vmaxs2)", nsm, din, dout, dspan);
  run<3>("VIADDMNMX.S16x2 min", nsm, din, dout, dspan);
  return 0;
}
