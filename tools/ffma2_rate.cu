// Throughput probe: FP32 FFMA (3 register operands) vs packed FFMA2
// (fma.rn.f32x2) on sm_100a, with a resident-warp sweep and the SM clock
// read from clock64 so the result is FMA lanes per clock per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/ffma2_rate tools/ffma2_rate.cu
// Modes of the FFMA2 kernel:
//   active  = warps that run the FFMA2 loop; the other resident warps of the
//             CTA either exit at once (park = 0), wait at a named barrier
//             until the math warps finish (park = 1), or run a shared-memory
//             load/store loop (park = 2)
//   ctas    = CTAs per SM (grid = 148 * ctas)
#include <cmath>
#include <cstdio>
typedef unsigned long long u64;
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}
__global__ void k_ffma(float* out, int iters, long long* clk) {
  float x[32];
  for (int j = 0; j < 32; ++j) x[j] = threadIdx.x + j;
  float a = 1.0001f + threadIdx.x * 1e-9f, b = 0.999f + threadIdx.x * 1e-9f;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int j = 0; j < 32; ++j) x[j] = fmaf(x[j], a, b);
  }
  long long t1 = clock64();
  float s = 0;
  for (int j = 0; j < 32; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}
// NCH independent chains per thread (ILP), 3 distinct 64-bit source operands
template <int NCH>
__global__ void k_ffma2(float* out, int iters, long long* clk, int active, int park) {
  __shared__ u64 sm[1024];
  const int warp = threadIdx.x >> 5;
  if (warp >= active) {
    if (park == 1) {
      asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
    } else if (park == 2) {
      u64 v = threadIdx.x;
      for (int i = 0; i < iters * 16; ++i) {
        sm[(threadIdx.x + i) & 1023] = v;
        v += sm[(threadIdx.x * 7 + i) & 1023];
      }
      out[blockIdx.x * blockDim.x + threadIdx.x] = (float)v;
    }
    return;
  }
  u64 x[NCH];
  for (int j = 0; j < NCH; ++j) x[j] = threadIdx.x + j;
  u64 a = 0x3f8000013f800001ull + threadIdx.x, b = 0x3f7fbe773f7fbe77ull + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 128 / NCH; ++r)
#pragma unroll
      for (int j = 0; j < NCH; ++j) x[j] = ffma2(x[j], a, b);
  }
  long long t1 = clock64();
  u64 s = 0;
  for (int j = 0; j < NCH; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    clk[3 * blockIdx.x] = t0;
    clk[3 * blockIdx.x + 1] = t1;
    clk[3 * blockIdx.x + 2] = smid;
  }
  if (park == 1) asm volatile("bar.sync 1, %0;" ::"r"(blockDim.x) : "memory");
}
// busiest-SM span: total FFMA2 warp instructions issued on an SM / (last end - first start)
static double sm_rate(const long long* clk, int blocks, double insts_per_block) {
  double worst = 1e30;
  for (int sm = 0; sm < 256; ++sm) {
    long long lo = 0, hi = 0;
    int n = 0;
    for (int b = 0; b < blocks; ++b)
      if (clk[3 * b + 2] == sm) {
        if (!n || clk[3 * b] < lo) lo = clk[3 * b];
        if (!n || clk[3 * b + 1] > hi) hi = clk[3 * b + 1];
        ++n;
      }
    if (n) worst = fmin(worst, n * insts_per_block / (double)(hi - lo));
  }
  return worst;
}
int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 4 * 1024 * 4);
  cudaMallocManaged(&clk, 148 * 4 * 8 * 3);
  const int iters = 2048;
  for (int warps : {4, 8, 16, 32}) {
    for (int rep = 0; rep < 2; ++rep) {
      k_ffma<<<148, 32 * warps>>>(out, iters, clk);
      cudaDeviceSynchronize();
    }
    double insts = (double)warps * iters * 128, c = (double)clk[0];
    printf("FFMA  warps/SM=%d: %.3f warp-inst/clk/SM, %.1f FMA lanes/clk/SM\n", warps, insts / c, insts * 32 / c);
  }
  struct Cfg { int resident, active, park, ctas, nch; };
  const Cfg cfgs[] = {
      {4, 4, 0, 1, 16},  {8, 8, 0, 1, 16},  {16, 16, 0, 1, 16}, {24, 24, 0, 1, 16}, {32, 32, 0, 1, 8},
      {8, 8, 0, 2, 16},  {8, 8, 0, 3, 16},  {4, 4, 0, 4, 16},   {16, 8, 1, 1, 16},  {16, 8, 2, 1, 16},
      {8, 8, 0, 1, 32},  {16, 16, 0, 1, 32}, {8, 8, 0, 2, 32},
  };
  for (const Cfg& c : cfgs) {
    for (int rep = 0; rep < 2; ++rep) {
      if (c.nch == 8) k_ffma2<8><<<148 * c.ctas, 32 * c.resident>>>(out, iters, clk, c.active, c.park);
      else if (c.nch == 16) k_ffma2<16><<<148 * c.ctas, 32 * c.resident>>>(out, iters, clk, c.active, c.park);
      else if (c.nch == 64) k_ffma2<64><<<148 * c.ctas, 32 * c.resident>>>(out, iters, clk, c.active, c.park);
      else k_ffma2<32><<<148 * c.ctas, 32 * c.resident>>>(out, iters, clk, c.active, c.park);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) {
        printf("FFMA2 resident=%d ctas=%d chains=%d: launch failed: %s\n", c.resident, c.ctas, c.nch, cudaGetErrorString(e));
        break;
      }
    }
    double r = sm_rate(clk, 148 * c.ctas, (double)c.active * iters * 128);
    printf("FFMA2 resident=%d active=%d park=%d ctas/SM=%d chains=%d: %.3f warp-inst/clk/SM, %.1f FMA lanes/clk/SM (slowest SM)\n",
           c.resident, c.active, c.park, c.ctas, c.nch, r, r * 64);
  }
  return 0;
}
