// Throughput of mma.sync.m8n8k4.f64 (DMMA) per SM on this GPU: clk per instruction with
// 1..16 warps per CTA, 4 independent accumulator chains per warp.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, double a, double b) {
  double c[8][2];
  for (int i = 0; i < 8; ++i) c[i][0] = c[i][1] = a * threadIdx.x;
  __syncthreads();
  long long t0 = clock64();
#pragma unroll 4
  for (int i = 0; i < 512; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) dmma(c[j][0], c[j][1], a, b);
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) cyc[0] = t1 - t0;
  double s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024 * 1024); cudaMalloc(&c, 64);
  for (int warps = 1; warps <= 16; warps *= 2) {
    k<<<148, 32 * warps>>>(o, c, 1e-3, 0.999); cudaDeviceSynchronize();
    long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double per = (double)h / 4096.0;     // clk per DMMA per warp
    printf("warps/SM %2d: %.2f clk per DMMA per warp -> %.1f FMA/clk/SM\n", warps, per, 256.0 * warps / per);
  }
  return 0;
}
