// Measured compute peaks of this B200 for the roofline denominators the bench does not get from
// MEASURED_PEAKS.json (which holds HBM GB/s and bf16 tensor TF/s only): FP32 FFMA, packed FP32
// FFMA2, legacy-MMA TF32 (mma.sync m16n8k8), DMMA (FP64 mma.sync m8n8k4) and DFMA. Each kernel
// runs 8 independent accumulator chains per thread on every SM; prints one JSON line.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/peak_bench.cu -o /tmp/peak_bench
#include <cstdio>

__global__ void k_ffma(float* out, int iters) {
  float a = threadIdx.x * 1e-3f, b = 1.0f + threadIdx.x * 1e-4f, c[8] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = fmaf(a, b, c[t]);
  float s = 0;
  for (int t = 0; t < 8; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_ffma2(float* out, int iters) {
  float2 a = make_float2(threadIdx.x * 1e-3f, 2.f), b = make_float2(1.0f + threadIdx.x * 1e-4f, 3.f);
  float2 c[8] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = __ffma2_rn(a, b, c[t]);
  float s = 0;
  for (int t = 0; t < 8; ++t) s += c[t].x + c[t].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_tf32(float* out, int iters) {
  unsigned a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3}, b[2] = {threadIdx.x, 7u};
  float c[8][4] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  float s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_dmma(float* out, int iters) {
  double a0 = threadIdx.x * 1e-3, b0 = 1.0 + threadIdx.x * 1e-4, c[8][2] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[t][0]), "+d"(c[t][1])
                   : "d"(a0), "d"(b0));
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(s);
}
__global__ void k_dfma(float* out, int iters) {
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4, c[8] = {};
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t] = fma(a, b, c[t]);
  double s = 0;
  for (int t = 0; t < 8; ++t) s += c[t];
  out[blockIdx.x * blockDim.x + threadIdx.x] = float(s);
}

template <class K>
double run(K k, double flops_per_thread_iter, int warps) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float* o;
  cudaMalloc(&o, size_t(sms) * 4 * 1024 * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int iters = 8192, ctas = sms * 4;
  k<<<ctas, warps * 32>>>(o, 16);
  cudaEventRecord(a);
  k<<<ctas, warps * 32>>>(o, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(o);
  return flops_per_thread_iter * iters * double(ctas) * warps * 32 / (ms * 1e-3) / 1e12;
}

int main() {
  double best[5] = {0, 0, 0, 0, 0};
  for (int w : {4, 8}) {
    best[0] = fmax(best[0], run(k_ffma, 2.0 * 8, w));
    best[1] = fmax(best[1], run(k_ffma2, 4.0 * 8, w));
    best[2] = fmax(best[2], run(k_tf32, 2.0 * 16 * 8 * 8 * 8 / 32, w));
    best[3] = fmax(best[3], run(k_dmma, 2.0 * 8 * 8 * 4 * 8 / 32, w));
    best[4] = fmax(best[4], run(k_dfma, 2.0 * 8, w));
  }
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("{\"fp32_ffma_tflops\": %.1f, \"fp32_ffma2_tflops\": %.1f, \"tf32_mma_sync_tflops\": %.1f, "
         "\"fp64_dmma_tflops\": %.1f, \"fp64_dfma_tflops\": %.1f, \"sm_clock_mhz_attr\": %d}\n",
         best[0], best[1], best[2], best[3], best[4], clk / 1000);
  return 0;
}
