// Dev micro-benchmark: polar_newton vs jacobi_svd + procrustes on random k x k matrices.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_19325_b200/csrc
//   -I include tools/polar_bench.cu paper_2605_19325_b200/csrc/kernels_small.cu -o /tmp/pb
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <vector>
#include "internal.h"
namespace enmf {
thread_local int64_t* g_launch_counter = nullptr;
void reduce_parts(const double*, int, int64_t, double*, cudaStream_t) {}
}
int main() {
  const int k = 128;
  std::vector<double> h(k * k);
  srand(1);
  for (auto& v : h) v = (double)rand() / RAND_MAX - 0.5;
  for (int i = 0; i < k; ++i) h[i * k + i] += 3.0 * (1.0 + i);   // cond ~ 100s
  double *M, *R, *R2, *Cs, *Ds, *sv, *jw;
  int* fail;
  int* iters;
  cudaMalloc(&iters, 4);
  cudaMalloc(&M, 8 * k * k); cudaMalloc(&R, 8 * k * k); cudaMalloc(&R2, 8 * k * k);
  cudaMalloc(&Cs, 8 * k * k); cudaMalloc(&Ds, 8 * k * k); cudaMalloc(&sv, 8 * k);
  cudaMalloc(&jw, 16 * k * k); cudaMalloc(&fail, 4);
  cudaMemcpy(M, h.data(), 8 * k * k, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  enmf::polar_newton(M, k, R, fail, 0);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) enmf::polar_newton(M, k, R, fail, 0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  enmf::polar_newton(M, k, R, fail, 0, iters);
  int fh, ih; cudaMemcpy(&fh, fail, 4, cudaMemcpyDeviceToHost); cudaMemcpy(&ih, iters, 4, cudaMemcpyDeviceToHost);
  printf("polar_newton: %.3f ms/call fail=%d iters=%d (%s)\n", ms / 10, fh, ih, cudaGetErrorString(cudaGetLastError()));
  {
    double* nsw; int* st2;
    cudaMalloc(&nsw, 8 * (3 * k * k + 256)); cudaMalloc(&st2, 8);
    double* R3; cudaMalloc(&R3, 8 * k * k);
    enmf::polar_ns(M, k, R3, st2, nsw, 48, 0);
    cudaEventRecord(a);
    for (int i = 0; i < 10; ++i) enmf::polar_ns(M, k, R3, st2, nsw, 48, 0);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    int sh[2]; cudaMemcpy(sh, st2, 8, cudaMemcpyDeviceToHost);
    std::vector<double> r3(k * k), r1(k * k);
    cudaMemcpy(r3.data(), R3, 8 * k * k, cudaMemcpyDeviceToHost);
    cudaMemcpy(r1.data(), R, 8 * k * k, cudaMemcpyDeviceToHost);
    double d = 0, n = 0;
    for (int i = 0; i < k * k; ++i) { d += (r1[i] - r3[i]) * (r1[i] - r3[i]); n += r1[i] * r1[i]; }
    printf("polar_ns: %.3f ms/call done=%d fail=%d |R_ns - R_newton|/|R| = %.3e (%s)\n", ms / 10,
           sh[0], sh[1], sqrt(d / n), cudaGetErrorString(cudaGetLastError()));
  }
  cudaEventRecord(a);
  for (int i = 0; i < 3; ++i) {
    enmf::jacobi_svd(M, k, Cs, sv, Ds, jw, 0);
    enmf::procrustes_from_svd(Cs, sv, Ds, k, R2, 0);
  }
  cudaEventRecord(b); cudaEventSynchronize(b);
  cudaEventElapsedTime(&ms, a, b);
  printf("jacobi+procrustes: %.3f ms/call\n", ms / 3);
  std::vector<double> r1(k * k), r2(k * k);
  cudaMemcpy(r1.data(), R, 8 * k * k, cudaMemcpyDeviceToHost);
  cudaMemcpy(r2.data(), R2, 8 * k * k, cudaMemcpyDeviceToHost);
  double d = 0, n = 0;
  for (int i = 0; i < k * k; ++i) { d += (r1[i] - r2[i]) * (r1[i] - r2[i]); n += r2[i] * r2[i]; }
  printf("|R_newton - R_jacobi| / |R| = %.3e\n", sqrt(d / n));
  return 0;
}
