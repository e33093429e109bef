#include <cstdio>
__global__ void kd(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 + threadIdx.x * 1e-4;
  double c[8][2] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a0), "d"(b0));
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void kf(double* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 + threadIdx.x * 1e-4;
  double c[8] = {};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = fma(a0, b0, c[t]);
  }
  double s = 0; for (int t = 0; t < 8; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  double* o; cudaMalloc(&o, 148 * 8 * 1024 * 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int iters = 4096;
  for (int warps : {4, 8, 16}) {
    kd<<<148 * 4, warps * 32>>>(o, 10);
    cudaEventRecord(a); kd<<<148 * 4, warps * 32>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double fl = 2.0 * 256 * 8 * double(iters) * 148 * 4 * warps;
    printf("DMMA warps/CTA=%d (4 CTA/SM): %.1f TFLOP/s\n", warps, fl / ms / 1e9);
    cudaEventRecord(a); kf<<<148 * 4, warps * 32>>>(o, iters); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    fl = 2.0 * 32 * 8 * double(iters) * 148 * 4 * warps;
    printf("DFMA warps/CTA=%d: %.1f TFLOP/s\n", warps, fl / ms / 1e9);
  }
  return 0;
}
