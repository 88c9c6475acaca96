// CUDA-core complex GEMM for small / awkward contraction steps, plus the
// element-wise helpers (axpy, 3xTF32 plane split, fixed-order tree reduce).
//
// Reference op: the np.matmul of contract_pair (contract.py:131-165).  Used
// where a step is too small to feed tensor cores (most of the ~800 steps of
// a circuit slice) or for complex128 ("double" precision) tensors.
#include <algorithm>

#include "tnc_common.cuh"

namespace tnc {

namespace {

template <typename R>
struct cpx {
  R re, im;
};

template <typename T>
__device__ __forceinline__ cpx<typename real_of<T>::type> load_c(const T* p) {
  T v = *p;
  return {v.re, v.im};
}

// C[m*ldcm + n*ldcn] (+)= sum_k X[m*ldx + k] * Y[n*ldy + k]
// 64x64 output tile per 256-thread block, 4x4 complex outputs per thread.
template <typename T>
__global__ void __launch_bounds__(256) simt_cgemm_kernel(int64_t M, int64_t N, int64_t K,
                                                         const T* __restrict__ X, int64_t ldx,
                                                         const T* __restrict__ Y, int64_t ldy,
                                                         T* __restrict__ C, int64_t ldcm,
                                                         int64_t ldcn, int accumulate) {
  using R = typename real_of<T>::type;
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ R xs_re[BK][BM + 1], xs_im[BK][BM + 1];
  __shared__ R ys_re[BK][BN + 1], ys_im[BK][BN + 1];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * BM;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x) * BN;
  R acc_re[4][4], acc_im[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc_re[i][j] = acc_im[i][j] = R(0);

  for (int64_t k0 = 0; k0 < K; k0 += BK) {
    // each thread loads 4 elements of X and 4 of Y (k fastest for coalescing)
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      int idx = tid + r * 256;  // 0..1023
      int kk = idx & (BK - 1);
      int mm = idx >> 4;
      int64_t gm = m0 + mm, gk = k0 + kk;
      R vr = R(0), vi = R(0);
      if (gm < M && gk < K) {
        T v = X[gm * ldx + gk];
        vr = v.re;
        vi = v.im;
      }
      xs_re[kk][mm] = vr;
      xs_im[kk][mm] = vi;
      int64_t gn = n0 + mm;
      vr = R(0);
      vi = R(0);
      if (gn < N && gk < K) {
        T v = Y[gn * ldy + gk];
        vr = v.re;
        vi = v.im;
      }
      ys_re[kk][mm] = vr;
      ys_im[kk][mm] = vi;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      R ar[4], ai[4], br[4], bi[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        ar[i] = xs_re[kk][ty + 16 * i];
        ai[i] = xs_im[kk][ty + 16 * i];
        br[i] = ys_re[kk][tx + 16 * i];
        bi[i] = ys_im[kk][tx + 16 * i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc_re[i][j] = fma(ar[i], br[j], acc_re[i][j]);
          acc_re[i][j] = fma(-ai[i], bi[j], acc_re[i][j]);
          acc_im[i][j] = fma(ar[i], bi[j], acc_im[i][j]);
          acc_im[i][j] = fma(ai[i], br[j], acc_im[i][j]);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int64_t gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int64_t gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      T* p = C + gm * ldcm + gn * ldcn;
      T v;
      v.re = acc_re[i][j];
      v.im = acc_im[i][j];
      if (accumulate) {
        T o = *p;
        v.re += o.re;
        v.im += o.im;
      }
      *p = v;
    }
  }
}

// Tiny-K / tiny-N path: one thread per output element, full K loop.
template <typename T>
__global__ void __launch_bounds__(256) simt_dot_kernel(int64_t M, int64_t N, int64_t K,
                                                       const T* __restrict__ X, int64_t ldx,
                                                       const T* __restrict__ Y, int64_t ldy,
                                                       T* __restrict__ C, int64_t ldcm,
                                                       int64_t ldcn, int accumulate) {
  using R = typename real_of<T>::type;
  const int64_t total = M * N;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t m, n;
    if (ldcn == 1) {  // walk the output contiguously
      m = e / N;
      n = e - m * N;
    } else {
      n = e / M;
      m = e - n * M;
    }
    const T* xr = X + m * ldx;
    const T* yr = Y + n * ldy;
    R re = R(0), im = R(0);
    for (int64_t k = 0; k < K; ++k) {
      T a = xr[k], b = yr[k];
      re = fma(a.re, b.re, re);
      re = fma(-a.im, b.im, re);
      im = fma(a.re, b.im, im);
      im = fma(a.im, b.re, im);
    }
    T* p = C + m * ldcm + n * ldcn;
    if (accumulate) {
      T o = *p;
      re += o.re;
      im += o.im;
    }
    T v;
    v.re = re;
    v.im = im;
    *p = v;
  }
}

// Split-K for tiny M*N with huge K (e.g. the (2,21,4) closing step of a
// circuit slice): block (chunk, tile) folds K range [chunk*kc, ...) for a
// TM x TN output tile; each thread strides over k (coalesced across the warp),
// keeps TM*TN complex partials in registers, then a fixed-order warp-shuffle +
// shared-memory reduction produces the block partial [chunk][M][N].
template <typename T, int TM, int TN>
__global__ void __launch_bounds__(256) simt_splitk_kernel(int64_t M, int64_t N, int64_t K, int64_t kc,
                                                          const T* __restrict__ X, int64_t ldx,
                                                          const T* __restrict__ Y, int64_t ldy,
                                                          T* __restrict__ parts) {
  using R = typename real_of<T>::type;
  const int64_t chunk = blockIdx.x;
  const int64_t n_tiles_n = (N + TN - 1) / TN;
  const int64_t m0 = (blockIdx.y / n_tiles_n) * TM;
  const int64_t n0 = (blockIdx.y % n_tiles_n) * TN;
  const int64_t k_lo = chunk * kc;
  const int64_t k_hi = min(K, k_lo + kc);
  R acc_re[TM][TN], acc_im[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc_re[i][j] = acc_im[i][j] = R(0);
  for (int64_t k = k_lo + threadIdx.x; k < k_hi; k += blockDim.x) {
    T x[TM], y[TN];
#pragma unroll
    for (int i = 0; i < TM; ++i) {
      if (m0 + i < M) x[i] = X[(m0 + i) * ldx + k];
      else x[i].re = x[i].im = R(0);
    }
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      if (n0 + j < N) y[j] = Y[(n0 + j) * ldy + k];
      else y[j].re = y[j].im = R(0);
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        acc_re[i][j] = fma(x[i].re, y[j].re, acc_re[i][j]);
        acc_re[i][j] = fma(-x[i].im, y[j].im, acc_re[i][j]);
        acc_im[i][j] = fma(x[i].re, y[j].im, acc_im[i][j]);
        acc_im[i][j] = fma(x[i].im, y[j].re, acc_im[i][j]);
      }
  }
  __shared__ R red[8][TM * TN * 2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      R re = acc_re[i][j], im = acc_im[i][j];
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        re += __shfl_xor_sync(0xffffffffu, re, s);
        im += __shfl_xor_sync(0xffffffffu, im, s);
      }
      if (lane == 0) {
        red[warp][2 * (i * TN + j)] = re;
        red[warp][2 * (i * TN + j) + 1] = im;
      }
    }
  __syncthreads();
  for (int o = threadIdx.x; o < TM * TN; o += blockDim.x) {
    R re = R(0), im = R(0);
    for (int w = 0; w < 8; ++w) {
      re += red[w][2 * o];
      im += red[w][2 * o + 1];
    }
    const int i = o / TN, j = o % TN;
    if (m0 + i < M && n0 + j < N) {
      T v;
      v.re = re;
      v.im = im;
      parts[chunk * M * N + (m0 + i) * N + (n0 + j)] = v;
    }
  }
}

// Split-K with in-kernel gathers (K3 for the tiny-output, huge-K steps such as
// C4's (6,26,4) closing contraction): no operand permutation pass.  Block b
// folds K range [b*kc, ...) in chunks of 64: the X rows (<= 64) and Y rows
// (<= 64) of the chunk are gathered straight from the strided operands into
// shared memory -- walking K contiguously when the operand's innermost leg is
// a common leg, rows contiguously otherwise -- and every thread accumulates
// up to 16 of the M*N outputs.  Partials [block][M][N] go to the fixed-order
// tree reduction.
template <typename T>
__global__ void __launch_bounds__(256) splitk_gather_kernel(
    int64_t M, int64_t N, int64_t K, int64_t kc, const T* __restrict__ X, const T* __restrict__ Y,
    const int64_t* __restrict__ tabs, int64_t s0, int64_t s1, int64_t s2, int x_kfast, int y_kfast,
    T* __restrict__ parts) {
  using R = typename real_of<T>::type;
  constexpr int CK = 64;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* xs = reinterpret_cast<T*>(smem_raw);      // [M][CK + 1]
  T* ys = xs + M * (CK + 1);                    // [N][CK + 1]
  const int64_t* rowx = tabs;
  const int64_t* rowy = rowx + M;
  const int64_t* tx0 = rowy + N;
  const int64_t* tx1 = tx0 + s0;
  const int64_t* tx2 = tx1 + s1;
  const int64_t* ty0 = tx2 + s2;
  const int64_t* ty1 = ty0 + s0;
  const int64_t* ty2 = ty1 + s1;
  const int64_t k_lo = static_cast<int64_t>(blockIdx.x) * kc;
  const int64_t k_hi = min(K, k_lo + kc);
  const int tid = threadIdx.x;
  const int n_out = static_cast<int>(M * N);
  // qubit legs make the level sizes powers of two: decode with shifts, not
  // 64-bit divisions (which dominated the gather cost)
  const bool pow2 = ((s0 & (s0 - 1)) == 0) && ((s1 & (s1 - 1)) == 0);
  const int sh0 = __ffsll(s0) - 1, sh1 = __ffsll(s1) - 1;
  auto decode = [&](int64_t k, int64_t& a, int64_t& b, int64_t& c) {
    if (pow2) {
      a = k & (s0 - 1);
      b = (k >> sh0) & (s1 - 1);
      c = k >> (sh0 + sh1);
    } else {
      a = k % s0;
      const int64_t q = k / s0;
      b = q % s1;
      c = q / s1;
    }
  };
  // compute mapping: 4x4 output blocks, `ksplit` threads per block taking
  // interleaved k (consecutive threads -> consecutive k: conflict-free smem)
  const int nbm = static_cast<int>((M + 3) / 4), nbn = static_cast<int>((N + 3) / 4);
  const int nblk = nbm * nbn;
  int ksplit = 1;
  while (ksplit * 2 * nblk <= 256) ksplit *= 2;
  const int g = tid % ksplit, blk = tid / ksplit;
  const bool active = blk < nblk;
  const int m0 = active ? (blk / nbn) * 4 : 0, n0 = active ? (blk % nbn) * 4 : 0;
  R acc_re[16], acc_im[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) acc_re[j] = acc_im[j] = R(0);
  for (int64_t k0 = k_lo; k0 < k_hi; k0 += CK) {
    for (int e = tid; e < M * CK; e += 256) {
      int m, kk;
      if (x_kfast) { m = e / CK; kk = e % CK; } else { m = e % static_cast<int>(M); kk = e / static_cast<int>(M); }
      const int64_t k = k0 + kk;
      T v;
      if (k < k_hi) {
        int64_t a, b, c;
        decode(k, a, b, c);
        v = X[rowx[m] + tx0[a] + tx1[b] + tx2[c]];
      } else {
        v.re = v.im = R(0);
      }
      xs[m * (CK + 1) + kk] = v;
    }
    for (int e = tid; e < N * CK; e += 256) {
      int n, kk;
      if (y_kfast) { n = e / CK; kk = e % CK; } else { n = e % static_cast<int>(N); kk = e / static_cast<int>(N); }
      const int64_t k = k0 + kk;
      T v;
      if (k < k_hi) {
        int64_t a, b, c;
        decode(k, a, b, c);
        v = Y[rowy[n] + ty0[a] + ty1[b] + ty2[c]];
      } else {
        v.re = v.im = R(0);
      }
      ys[n * (CK + 1) + kk] = v;
    }
    __syncthreads();
    if (active) {
      for (int kk = g; kk < CK; kk += ksplit) {
        T a[4], b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int m = min(m0 + i, static_cast<int>(M) - 1);
          const int n = min(n0 + i, static_cast<int>(N) - 1);
          a[i] = xs[m * (CK + 1) + kk];
          b[i] = ys[n * (CK + 1) + kk];
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            R re = acc_re[4 * i + j], im = acc_im[4 * i + j];
            re = fma(a[i].re, b[j].re, re);
            re = fma(-a[i].im, b[j].im, re);
            im = fma(a[i].re, b[j].im, im);
            im = fma(a[i].im, b[j].re, im);
            acc_re[4 * i + j] = re;
            acc_im[4 * i + j] = im;
          }
      }
    }
    __syncthreads();
  }
  // fixed-order reduction over the k-groups of each output block
  R* red = reinterpret_cast<R*>(smem_raw);  // [256 threads][32]
  if (active) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      red[tid * 32 + 2 * j] = acc_re[j];
      red[tid * 32 + 2 * j + 1] = acc_im[j];
    }
  }
  __syncthreads();
  for (int o = tid; o < n_out; o += 256) {
    const int m = o / static_cast<int>(N), n = o % static_cast<int>(N);
    const int b = (m / 4) * nbn + n / 4;
    const int j = (m % 4) * 4 + (n % 4);
    R re = R(0), im = R(0);
    for (int gg = 0; gg < ksplit; ++gg) {
      re += red[(b * ksplit + gg) * 32 + 2 * j];
      im += red[(b * ksplit + gg) * 32 + 2 * j + 1];
    }
    T v;
    v.re = re;
    v.im = im;
    parts[static_cast<int64_t>(blockIdx.x) * n_out + o] = v;
  }
}

template <typename T>
__global__ void axpy_kernel(int64_t n, const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    T a = x[i], b = y[i];
    b.re += a.re;
    b.im += a.im;
    y[i] = b;
  }
}

// Round to the nearest TF32 (ties away from zero) with the 13 low mantissa
// bits explicitly zeroed, so `big` is exact in TF32 and x - big is exact in
// fp32 (|small| <= 2^-12 |x|).
__device__ __forceinline__ float tf32_round(float x) {
  uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) return x;  // inf / nan unchanged
  u = (u + 0x1000u) & 0xffffe000u;
  return __uint_as_float(u);
}

// 3xTF32 operand planes.  mode 0: big/small of the interleaved row [2*Kp];
// mode 1: expanded rows 2r = (re, -im), 2r+1 = (im, re) per complex k.
__global__ void tf32_split_kernel(int mode, int64_t R, int64_t K, int64_t Kp,
                                  const c64* __restrict__ X, int64_t ldx, float* __restrict__ big,
                                  float* __restrict__ small) {
  const int64_t total = R * Kp;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t r = e / Kp;
    int64_t k = e - r * Kp;
    float re = 0.f, im = 0.f;
    if (k < K) {
      c64 v = X[r * ldx + k];
      re = v.re;
      im = v.im;
    }
    float bre = tf32_round(re), bim = tf32_round(im);
    float sre = re - bre, sim = im - bim;
    if (mode == 0) {
      float2* b2 = reinterpret_cast<float2*>(big) + r * Kp + k;
      float2* s2 = reinterpret_cast<float2*>(small) + r * Kp + k;
      *b2 = make_float2(bre, bim);
      *s2 = make_float2(sre, sim);
    } else {
      float2* b0 = reinterpret_cast<float2*>(big) + (2 * r) * Kp + k;
      float2* s0 = reinterpret_cast<float2*>(small) + (2 * r) * Kp + k;
      float2* b1 = b0 + Kp;
      float2* s1 = s0 + Kp;
      *b0 = make_float2(bre, -bim);
      *s0 = make_float2(sre, -sim);
      *b1 = make_float2(bim, bre);
      *s1 = make_float2(sim, sre);
    }
  }
}

// 2-piece FP16 operand planes with a power-of-two scale per row ("3xFP16"):
//   row r is scaled by 2^-e[r] so its largest |component| lies in
//   [2^14, 2^15) (f16_row_exponent), hi = fp16(x), lo = fp16(x - hi); then
//   x = 2^e (hi + lo) to ~2^-22 relative down to 2^-16 of the row maximum and
//   to ~2^-38 of the row maximum below that (fp16 subnormals), and
//   x*y ~= hi*hi' + hi*lo' + lo*hi' keeps fp32-class accuracy relative to the
//   row/column norms with half the operand bytes of 3xTF32 and the 2x-rate
//   kind::f16 tensor-core path.  One warp per row.
// mode 0: planes [R, 2*Kp] (interleaved re, im);  mode 1: expanded [2R, 2*Kp]
// with rows 2r = (re, -im), 2r+1 = (im, re).  e[r] is written to `exps`.
__global__ void __launch_bounds__(256) f16_split_kernel(int mode, int64_t R, int64_t K, int64_t Kp,
                                                        const c64* __restrict__ X, int64_t ldx,
                                                        __half* __restrict__ hi, __half* __restrict__ lo,
                                                        int* __restrict__ exps) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < R; r += warps) {
    const c64* row = X + r * ldx;
    float mx = 0.f;
    for (int64_t k = lane; k < K; k += 32) {
      c64 v = row[k];
      mx = fmaxf(mx, fmaxf(fabsf(v.re), fabsf(v.im)));
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
    const int e = f16_row_exponent(mx);
    if (lane == 0) exps[r] = e;
    const float sc = ldexpf(1.f, -e);
    for (int64_t k = lane; k < Kp; k += 32) {
      float re = 0.f, im = 0.f;
      if (k < K) {
        c64 v = row[k];
        re = v.re * sc;
        im = v.im * sc;
      }
      const __half hre = __float2half_rn(re), him = __float2half_rn(im);
      const __half lre = __float2half_rn(re - __half2float(hre));
      const __half lim = __float2half_rn(im - __half2float(him));
      if (mode == 0) {
        reinterpret_cast<__half2*>(hi)[r * Kp + k] = __halves2half2(hre, him);
        reinterpret_cast<__half2*>(lo)[r * Kp + k] = __halves2half2(lre, lim);
      } else {
        __half2* h0 = reinterpret_cast<__half2*>(hi) + (2 * r) * Kp + k;
        __half2* l0 = reinterpret_cast<__half2*>(lo) + (2 * r) * Kp + k;
        h0[0] = __halves2half2(hre, __hneg(him));
        l0[0] = __halves2half2(lre, __hneg(lim));
        h0[Kp] = __halves2half2(him, hre);
        l0[Kp] = __halves2half2(lim, lre);
      }
    }
  }
}

// Few, very long rows (e.g. the (7,20,7) split-K step): phase 1 reduces each
// row's max |component| across many blocks (non-negative floats order like
// their bit patterns, so atomicMax on the bits is exact), phase 2 splits
// element-parallel.
__global__ void row_absmax_kernel(int64_t R, int64_t K, const c64* __restrict__ X, int64_t ldx,
                                  unsigned* __restrict__ rowmax) {
  const int64_t r = blockIdx.y;
  float mx = 0.f;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < K;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    c64 v = X[r * ldx + k];
    mx = fmaxf(mx, fmaxf(fabsf(v.re), fabsf(v.im)));
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, s));
  if ((threadIdx.x & 31) == 0) atomicMax(rowmax + r, __float_as_uint(mx));
}

__global__ void f16_split_elem_kernel(int mode, int64_t R, int64_t K, int64_t Kp,
                                      const c64* __restrict__ X, int64_t ldx, __half* __restrict__ hi,
                                      __half* __restrict__ lo, const unsigned* __restrict__ rowmax,
                                      int* __restrict__ exps) {
  const int64_t total = R * Kp;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / Kp;
    const int64_t k = e - r * Kp;
    const float mx = __uint_as_float(rowmax[r]);
    const int ex = f16_row_exponent(mx);
    if (k == 0) exps[r] = ex;
    const float sc = ldexpf(1.f, -ex);
    float re = 0.f, im = 0.f;
    if (k < K) {
      c64 v = X[r * ldx + k];
      re = v.re * sc;
      im = v.im * sc;
    }
    const __half hre = __float2half_rn(re), him = __float2half_rn(im);
    const __half lre = __float2half_rn(re - __half2float(hre));
    const __half lim = __float2half_rn(im - __half2float(him));
    if (mode == 0) {
      reinterpret_cast<__half2*>(hi)[r * Kp + k] = __halves2half2(hre, him);
      reinterpret_cast<__half2*>(lo)[r * Kp + k] = __halves2half2(lre, lim);
    } else {
      __half2* h0 = reinterpret_cast<__half2*>(hi) + (2 * r) * Kp + k;
      __half2* l0 = reinterpret_cast<__half2*>(lo) + (2 * r) * Kp + k;
      h0[0] = __halves2half2(hre, __hneg(him));
      l0[0] = __halves2half2(lre, __hneg(lim));
      h0[Kp] = __halves2half2(him, hre);
      l0[Kp] = __halves2half2(lim, lre);
    }
  }
}

// Fixed-order pairwise tree over P partial tiles [P][MN] (complex, fp32 or
// fp64): level by level, partial i += partial i+stride, exactly the
// left-complete combine of contract.py:200-207.  The root is written to
// out (strided) if given.
template <typename T>
__global__ void tree_level_kernel(int64_t P, int64_t MN, int64_t stride, T* __restrict__ parts) {
  // pairs (i, i+stride) for i multiple of 2*stride
  const int64_t n_pairs = (P + 2 * stride - 1) / (2 * stride);
  const int64_t total = n_pairs * MN;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t pair = e / MN;
    int64_t off = e - pair * MN;
    int64_t i = pair * 2 * stride;
    int64_t j = i + stride;
    if (j >= P) continue;
    T a = parts[i * MN + off], b = parts[j * MN + off];
    a.re += b.re;
    a.im += b.im;
    parts[i * MN + off] = a;
  }
}

template <typename T>
__global__ void scatter_mn_kernel(int64_t M, int64_t N, const T* __restrict__ src,
                                  T* __restrict__ dst, int64_t ldcm, int64_t ldcn) {
  const int64_t total = M * N;
  for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t m = e / N, n = e - (e / N) * N;
    dst[m * ldcm + n * ldcn] = src[e];
  }
}

inline unsigned grid_for(int64_t work, int threads = 256) {
  int64_t blocks = ceil_div(work, threads);
  blocks = std::min<int64_t>(blocks, static_cast<int64_t>(num_sms()) * 32);
  return static_cast<unsigned>(std::max<int64_t>(blocks, 1));
}

}  // namespace

int simt_cgemm_launch(int dtype, int64_t M, int64_t N, int64_t K, const void* X, int64_t ldx,
                      const void* Y, int64_t ldy, void* C, int64_t ldcm, int64_t ldcn,
                      int accumulate, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return TNC_OK;
  const double eb = static_cast<double>(elem_bytes(dtype));
  ProfScope prof(PROF_SIMT_GEMM, 8.0 * M * N * K, eb * (double(M) * K + double(N) * K + double(M) * N), stream);
  const bool tiled = (M >= 32 && N >= 32 && K >= 8);
  if (tiled) {
    dim3 grid(static_cast<unsigned>(ceil_div(N, 64)), static_cast<unsigned>(ceil_div(M, 64)));
    if (grid.y > 65535) {
      // fall back to the dot kernel for enormous M (grid.y limit)
    } else {
      if (dtype == TNC_C128)
        simt_cgemm_kernel<c128><<<grid, 256, 0, stream>>>(
            M, N, K, static_cast<const c128*>(X), ldx, static_cast<const c128*>(Y), ldy,
            static_cast<c128*>(C), ldcm, ldcn, accumulate);
      else
        simt_cgemm_kernel<c64><<<grid, 256, 0, stream>>>(
            M, N, K, static_cast<const c64*>(X), ldx, static_cast<const c64*>(Y), ldy,
            static_cast<c64*>(C), ldcm, ldcn, accumulate);
      TNC_CHECK_LAUNCH();
      return TNC_OK;
    }
  }
  unsigned g = grid_for(M * N);
  if (dtype == TNC_C128)
    simt_dot_kernel<c128><<<g, 256, 0, stream>>>(M, N, K, static_cast<const c128*>(X), ldx,
                                                  static_cast<const c128*>(Y), ldy,
                                                  static_cast<c128*>(C), ldcm, ldcn, accumulate);
  else
    simt_dot_kernel<c64><<<g, 256, 0, stream>>>(M, N, K, static_cast<const c64*>(X), ldx,
                                                static_cast<const c64*>(Y), ldy,
                                                static_cast<c64*>(C), ldcm, ldcn, accumulate);
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

int64_t splitk_chunks(int64_t M, int64_t N, int64_t K) {
  const int64_t tiles = ceil_div(M, 4) * ceil_div(N, 8);
  int64_t chunks = std::max<int64_t>(1, static_cast<int64_t>(num_sms()) * 4 / std::max<int64_t>(tiles, 1));
  chunks = std::min<int64_t>(chunks, ceil_div(K, 1024));  // >= 4 k per thread
  return std::max<int64_t>(chunks, 1);
}

int simt_splitk_launch(int dtype, int64_t M, int64_t N, int64_t K, const void* X, int64_t ldx,
                       const void* Y, int64_t ldy, void* C, int64_t ldcm, int64_t ldcn, void* parts,
                       cudaStream_t stream) {
  if (M <= 0 || N <= 0) return TNC_OK;
  const int64_t chunks = splitk_chunks(M, N, K);
  const int64_t kc = ceil_div(K, chunks);
  const int64_t tiles = ceil_div(M, 4) * ceil_div(N, 8);
  if (tiles > 65535) TNC_RET(TNC_ERR_UNSUPPORTED, "split-K: output too large");
  {
    const double eb = static_cast<double>(elem_bytes(dtype));
    ProfScope prof(PROF_SIMT_GEMM, 8.0 * M * N * K, eb * (double(M) * K + double(N) * K + double(M) * N),
                   stream);
    dim3 grid(static_cast<unsigned>(chunks), static_cast<unsigned>(tiles));
    if (dtype == TNC_C128)
      simt_splitk_kernel<c128, 4, 8><<<grid, 256, 0, stream>>>(M, N, K, kc, static_cast<const c128*>(X), ldx,
                                                               static_cast<const c128*>(Y), ldy,
                                                               static_cast<c128*>(parts));
    else
      simt_splitk_kernel<c64, 4, 8><<<grid, 256, 0, stream>>>(M, N, K, kc, static_cast<const c64*>(X), ldx,
                                                              static_cast<const c64*>(Y), ldy,
                                                              static_cast<c64*>(parts));
    TNC_CHECK_LAUNCH();
  }
  return tree_reduce_launch(dtype, chunks, M * N, parts, C, M, N, ldcm, ldcn, stream);
}

int splitk_gather_launch(int dtype, int64_t M, int64_t N, int64_t K, const void* X, const void* Y,
                         const int64_t* tabs, const int64_t* lvl, int x_kfast, int y_kfast,
                         int64_t chunks, void* C, int64_t ldcm, int64_t ldcn, void* parts,
                         cudaStream_t stream) {
  if (M <= 0 || N <= 0) return TNC_OK;
  if (M > 64 || N > 64 || M * N > 4096) TNC_RET(TNC_ERR_UNSUPPORTED, "gather split-K: output too large");
  const int64_t kc = ceil_div(K, chunks);
  const size_t eb = elem_bytes(dtype);
  // operand tiles, reused afterwards for the k-group reduction (256 x 16 complex)
  const size_t smem = std::max(static_cast<size_t>(M + N) * 65 * eb, static_cast<size_t>(256) * 16 * eb);
  {
    ProfScope prof(PROF_SIMT_GEMM, 8.0 * M * N * K, double(eb) * (double(M) * K + double(N) * K + double(M) * N),
                   stream);
    if (dtype == TNC_C128) {
      auto k = splitk_gather_kernel<c128>;
      TNC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      k<<<static_cast<unsigned>(chunks), 256, smem, stream>>>(M, N, K, kc, static_cast<const c128*>(X),
                                                              static_cast<const c128*>(Y), tabs, lvl[0], lvl[1],
                                                              lvl[2], x_kfast, y_kfast, static_cast<c128*>(parts));
    } else {
      auto k = splitk_gather_kernel<c64>;
      TNC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      k<<<static_cast<unsigned>(chunks), 256, smem, stream>>>(M, N, K, kc, static_cast<const c64*>(X),
                                                              static_cast<const c64*>(Y), tabs, lvl[0], lvl[1],
                                                              lvl[2], x_kfast, y_kfast, static_cast<c64*>(parts));
    }
    TNC_CHECK_LAUNCH();
  }
  return tree_reduce_launch(dtype, chunks, M * N, parts, C, M, N, ldcm, ldcn, stream);
}

int axpy_launch(int dtype, int64_t n, const void* x, void* y, cudaStream_t stream) {
  if (n <= 0) return TNC_OK;
  ProfScope prof(PROF_AXPY, 2.0 * n, 3.0 * n * elem_bytes(dtype), stream);
  unsigned g = grid_for(n);
  if (dtype == TNC_C128)
    axpy_kernel<c128><<<g, 256, 0, stream>>>(n, static_cast<const c128*>(x), static_cast<c128*>(y));
  else
    axpy_kernel<c64><<<g, 256, 0, stream>>>(n, static_cast<const c64*>(x), static_cast<c64*>(y));
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

int tf32_split_launch(int mode, int64_t R, int64_t K, int64_t Kp, const void* X, int64_t ldx,
                      void* big, void* small, cudaStream_t stream) {
  if (R <= 0 || Kp <= 0) return TNC_OK;
  ProfScope prof(PROF_SPLIT_PREP, 0.0, 8.0 * R * K + (mode ? 32.0 : 16.0) * R * Kp, stream);
  tf32_split_kernel<<<grid_for(R * Kp), 256, 0, stream>>>(
      mode, R, K, Kp, static_cast<const c64*>(X), ldx, static_cast<float*>(big),
      static_cast<float*>(small));
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

int f16_split_launch(int mode, int64_t R, int64_t K, int64_t Kp, const void* X, int64_t ldx,
                     void* hi, void* lo, int* exps, void* scratch, cudaStream_t stream) {
  if (R <= 0 || Kp <= 0) return TNC_OK;
  ProfScope prof(PROF_SPLIT_PREP, 0.0, 8.0 * R * K + (mode ? 16.0 : 8.0) * R * Kp, stream);
  if (R < static_cast<int64_t>(num_sms()) * 32 && K >= 4096 && R <= 65535) {
    // few long rows: cross-block row max (into `scratch`), then an
    // element-parallel split that derives the scale exponents
    unsigned* rowmax = static_cast<unsigned*>(scratch);
    TNC_CUDA_TRY(cudaMemsetAsync(rowmax, 0, static_cast<size_t>(R) * sizeof(unsigned), stream));
    const int64_t per_row = std::max<int64_t>(1, std::min<int64_t>(ceil_div(K, 256 * 8),
                                                                   num_sms() * 8 / std::max<int64_t>(R, 1) + 1));
    row_absmax_kernel<<<dim3(static_cast<unsigned>(per_row), static_cast<unsigned>(R)), 256, 0, stream>>>(
        R, K, static_cast<const c64*>(X), ldx, rowmax);
    TNC_CHECK_LAUNCH();
    f16_split_elem_kernel<<<grid_for(R * Kp), 256, 0, stream>>>(mode, R, K, Kp, static_cast<const c64*>(X), ldx,
                                                               static_cast<__half*>(hi), static_cast<__half*>(lo),
                                                               rowmax, exps);
    TNC_CHECK_LAUNCH();
    return TNC_OK;
  }
  const int64_t blocks = std::min<int64_t>(ceil_div(R, 8), static_cast<int64_t>(num_sms()) * 16);
  f16_split_kernel<<<static_cast<unsigned>(std::max<int64_t>(blocks, 1)), 256, 0, stream>>>(
      mode, R, K, Kp, static_cast<const c64*>(X), ldx, static_cast<__half*>(hi), static_cast<__half*>(lo),
      exps);
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

int tree_reduce_launch(int dtype, int64_t P, int64_t MN, void* partials, void* out, int64_t M,
                       int64_t N, int64_t ldcm, int64_t ldcn, cudaStream_t stream) {
  ProfScope prof(PROF_REDUCE, 2.0 * P * MN, 2.0 * P * MN * elem_bytes(dtype), stream);
  for (int64_t stride = 1; stride < P; stride *= 2) {
    int64_t pairs = (P + 2 * stride - 1) / (2 * stride);
    unsigned g = grid_for(pairs * MN);
    if (dtype == TNC_C128)
      tree_level_kernel<c128><<<g, 256, 0, stream>>>(P, MN, stride, static_cast<c128*>(partials));
    else
      tree_level_kernel<c64><<<g, 256, 0, stream>>>(P, MN, stride, static_cast<c64*>(partials));
    TNC_CHECK_LAUNCH();
  }
  if (out) {
    unsigned g = grid_for(M * N);
    if (dtype == TNC_C128)
      scatter_mn_kernel<c128><<<g, 256, 0, stream>>>(M, N, static_cast<const c128*>(partials),
                                                     static_cast<c128*>(out), ldcm, ldcn);
    else
      scatter_mn_kernel<c64><<<g, 256, 0, stream>>>(M, N, static_cast<const c64*>(partials),
                                                    static_cast<c64*>(out), ldcm, ldcn);
    TNC_CHECK_LAUNCH();
  }
  return TNC_OK;
}

}  // namespace tnc
