// Microbenchmark: fp64 FMA / exp / div throughput and HBM stream bandwidth on B200.
// Informs the exp budget of the FINOM scan kernels.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

__global__ void k_fma(double* out, int iters, double a) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  for (int i = 0; i < iters; ++i) {
    x0 = fma(x0, a, 1e-9); x1 = fma(x1, a, 1e-9); x2 = fma(x2, a, 1e-9); x3 = fma(x3, a, 1e-9);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void k_exp(double* out, int iters, double step) {
  double s = 0, x0 = -(threadIdx.x & 63) * 0.37, x1 = x0 - 0.11;
  for (int i = 0; i < iters; ++i) { s += exp(x0) + exp(x1); x0 -= step; x1 -= step; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_expdiv(double* out, int iters, double step, double eps) {
  double s = 0, x0 = -(threadIdx.x & 63) * 0.37e-3, x1 = x0 - 0.11e-3;
  for (int i = 0; i < iters; ++i) { s += exp(x0 / eps) + exp(x1 / eps); x0 -= step; x1 -= step; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_div(double* out, int iters, double eps) {
  double s = 0, x0 = threadIdx.x * 0.37e-3 + 1, x1 = x0 + 0.11e-3;
  for (int i = 0; i < iters; ++i) { s += x0 / eps + x1 / eps; x0 += 1e-7; x1 += 1e-7; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_copy(const double2* __restrict__ a, double2* __restrict__ b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) b[i] = a[i];
}
int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("dev %s SMs %d clock %d kHz smem/block optin %zu\n", p.name, p.multiProcessorCount, p.clockRate, p.sharedMemPerBlockOptin);
  int sms = p.multiProcessorCount, blocks = sms * 8, threads = 256; int iters = 4096;
  double* out; CK(cudaMalloc(&out, blocks * threads * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1); float ms;
  double nthr = (double)blocks * threads;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0); k_fma<<<blocks, threads>>>(out, iters, 0.999999); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("DFMA: %.3f T/s\n", nthr * iters * 4 / (ms * 1e-3) / 1e12);
    cudaEventRecord(e0); k_exp<<<blocks, threads>>>(out, iters, 1e-4); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("exp: %.3f G/s\n", nthr * iters * 2 / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0); k_expdiv<<<blocks, threads>>>(out, iters, 1e-7, 1e-3); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("exp(x/eps): %.3f G/s\n", nthr * iters * 2 / (ms * 1e-3) / 1e9);
    cudaEventRecord(e0); k_div<<<blocks, threads>>>(out, iters, 1e-3); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("div: %.3f G/s\n", nthr * iters * 2 / (ms * 1e-3) / 1e9);
  }
  size_t n = (size_t)1 << 27; double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
  cudaMemset(a, 0, n * 16);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0); k_copy<<<sms * 16, 512>>>(a, b, n); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("copy: %.1f GB/s\n", 2.0 * n * 16 / (ms * 1e-3) / 1e9);
  }
  return 0;
}
