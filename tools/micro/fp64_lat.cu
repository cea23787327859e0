// Dependent-chain latency and single-warp issue interval of DFMA / DADD / SHFL on this GPU.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, long long* cyc, double a, double b) {
  double x = a + threadIdx.x, y0 = a, y1 = b, y2 = a + 1, y3 = b + 1, y4 = a + 2, y5 = b + 2, y6 = a + 3, y7 = b + 3;
  long long t0 = clock64();
#pragma unroll 64
  for (int i = 0; i < 1024; ++i) x = fma(x, b, a);
  long long t1 = clock64();
#pragma unroll 8
  for (int i = 0; i < 1024; ++i) {
    y0 = fma(y0, b, a); y1 = fma(y1, b, a); y2 = fma(y2, b, a); y3 = fma(y3, b, a);
    y4 = fma(y4, b, a); y5 = fma(y5, b, a); y6 = fma(y6, b, a); y7 = fma(y7, b, a);
  }
  long long t2 = clock64();
  double z = x;
#pragma unroll 64
  for (int i = 0; i < 1024; ++i) z = __shfl_sync(0xffffffffu, z, (i + 1) & 31);
  long long t3 = clock64();
  float f = (float)a + threadIdx.x;
#pragma unroll 64
  for (int i = 0; i < 1024; ++i) f = fmaf(f, (float)b, (float)a);
  long long t4 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x + y0 + y1 + y2 + y3 + y4 + y5 + y6 + y7 + z + f;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024 * 256); cudaMalloc(&c, 64);
  for (int warps = 1; warps <= 8; warps *= 2) {
    k<<<1, 32 * warps>>>(o, c, 1e-3, 0.999); cudaDeviceSynchronize();
    long long h[4]; cudaMemcpy(h, c, 32, cudaMemcpyDeviceToHost);
    printf("warps/CTA %d: dependent DFMA %.1f clk; 8 independent DFMA chains %.1f clk per DFMA; dependent SHFL(64-bit) %.1f clk; dependent FFMA %.1f clk\n",
           warps, h[0] / 1024.0, h[1] / 8192.0, h[2] / 1024.0, h[3] / 1024.0);
  }
  return 0;
}
