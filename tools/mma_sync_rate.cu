// Throughput probe: legacy warp MMA (mma.sync) vs FP32 FFMA on sm_100a.
#include <cstdio>
#include <cuda_fp16.h>
__global__ void mma_f16(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void mma_tf32(float* out, int iters) {
  unsigned a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  float c[8][4] = {};
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void ffma(float* out, int iters) {
  float x[16];
  for (int j = 0; j < 16; ++j) x[j] = threadIdx.x + j;
  const float a = 1.0001f, b = 0.999f;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = fmaf(x[j], a, b);
  }
  float s = 0;
  for (int j = 0; j < 16; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out;
  cudaMalloc(&out, 148 * 16 * 1024 * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 148;
  for (int warps : {4, 8, 16}) {
    int threads = 32 * warps, iters = 4096;
    for (int kind = 0; kind < 3; ++kind) {
      auto run = [&]() {
        if (kind == 0) mma_f16<<<sms * 2, threads>>>(out, iters);
        if (kind == 1) mma_tf32<<<sms * 2, threads>>>(out, iters);
        if (kind == 2) ffma<<<sms * 2, threads>>>(out, iters);
      };
      run();
      cudaEventRecord(e0);
      run();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double warps_total = 2.0 * sms * warps;
      double flops = kind == 0 ? warps_total * iters * 8 * 4096.0
                   : kind == 1 ? warps_total * iters * 8 * 2048.0
                               : warps_total * 32 * iters * 8 * 16 * 2.0;
      printf("%s warps/CTA=%d: %.1f TFLOP/s (%.3f ms)\n", kind == 0 ? "mma.sync f16 m16n8k16" : kind == 1 ? "mma.sync tf32 m16n8k8" : "FFMA fp32", warps, flops / ms / 1e9, ms);
    }
  }
  return 0;
}
