// Shared helpers of the B200 TNC kernels: status handling, complex types,
// small device utilities.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/tnc_b200.h"

namespace tnc {

// thread-local last error message (tnc_last_error)
void set_error(const std::string& msg);
const char* last_error();

#define TNC_RET(code, msg)               \
  do {                                   \
    ::tnc::set_error(msg);               \
    return (code);                       \
  } while (0)

#define TNC_CUDA_TRY(expr)                                                       \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::tnc::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e));     \
      return TNC_ERR_CUDA;                                                       \
    }                                                                            \
  } while (0)

// every kernel launch site ends with TNC_CHECK_LAUNCH(): it also counts the
// launch (tnc_launch_count) so benchmarks can report how many of OUR kernels ran
void count_launch();

#define TNC_CHECK_LAUNCH()                                                       \
  do {                                                                           \
    ::tnc::count_launch();                                                       \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      ::tnc::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return TNC_ERR_CUDA;                                                       \
    }                                                                            \
  } while (0)

#define TNC_TRY(expr)          \
  do {                         \
    int _s = (expr);           \
    if (_s != TNC_OK) return _s; \
  } while (0)

// 3xFP16 per-row scale exponent: the row is multiplied by 2^-e so that its
// largest |component| lands in [2^14, 2^15).  Scaling to the top of the fp16
// range (rather than to [0.5, 1)) keeps the lo = fp16(x - hi) plane normal
// down to 2^-16 of the row maximum and its subnormal step at 2^-38 of it, so
// rows with a large max/rms ratio keep fp32-class accuracy.  e is clamped so
// that 2^-e stays a normal float.
constexpr int kF16ScaleBits = 15;
__host__ __device__ __forceinline__ int f16_row_exponent(float mx) {
  int e = 0;
  if (mx > 0.f && isfinite(mx)) {
    frexpf(mx, &e);  // mx = f * 2^e, f in [0.5, 1)
    e -= kF16ScaleBits;
    if (e < -126) e = -126;
  }
  return e;
}

// complex element types (interleaved re, im), 8 and 16 bytes
struct __align__(8) c64 {
  float re, im;
};
struct __align__(16) c128 {
  double re, im;
};

template <typename T> struct real_of;
template <> struct real_of<c64> { using type = float; };
template <> struct real_of<c128> { using type = double; };

inline int num_sms() {
  static int n = -1;
  if (n < 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

inline size_t elem_bytes(int dtype) { return dtype == TNC_C128 ? 16 : 8; }

// Plan-time upload of a host index table to a device buffer owned by the plan
// (freed with the plan).  Plan creation may allocate and synchronise; the
// per-call launch paths (tnc_contract) never do.  The pageable copy is
// completed (legacy-stream sync) before returning, so kernels on any stream
// see the table.
// Host-only processes (no CUDA device) still plan: the table stays pending
// and a launch of such a plan reports an error.
inline int upload_table(const int64_t* host, size_t n, int64_t** dev) {
  *dev = nullptr;
  if (n == 0) return TNC_OK;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
    cudaGetLastError();
    return TNC_OK;
  }
  TNC_CUDA_TRY(cudaMalloc(dev, n * sizeof(int64_t)));
  TNC_CUDA_TRY(cudaMemcpy(*dev, host, n * sizeof(int64_t), cudaMemcpyHostToDevice));
  TNC_CUDA_TRY(cudaStreamSynchronize(cudaStreamLegacy));
  return TNC_OK;
}

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// Compact description of a strided n-d view used by the gather kernels.
struct Axis {
  int64_t dim;
  int64_t in_stride;
  int64_t out_stride;
};

// ---- optional per-kernel device timing (tnc_profile_*) ----
enum ProfKind { PROF_TC_GEMM = 0, PROF_SIMT_GEMM = 1, PROF_PERMUTE = 2, PROF_SPLIT_PREP = 3,
                PROF_REDUCE = 4, PROF_ABSORB = 5, PROF_AXPY = 6, PROF_STREAM = 7,
                PROF_TC_GATHER = 8, PROF_AUX = 9, PROF_KINDS = 10 };
// RAII: when profiling is enabled, records CUDA events around the launches
// issued in its scope on `stream` and books `flops` / `bytes` of algorithmic
// work to `kind`.
class ProfScope {
 public:
  ProfScope(int kind, double flops, double bytes, cudaStream_t stream);
  ~ProfScope();

 private:
  int kind_;
  double flops_, bytes_;
  cudaStream_t stream_;
  cudaEvent_t start_ = nullptr;
};

// ---- entry points implemented in the kernel translation units ----
// permute: general strided -> contiguous (target order)
int permute_launch(int dtype, int rank, const int64_t* dims, const int64_t* in_strides,
                   const int32_t* perm, const void* in, void* out, cudaStream_t stream);
// strided 2-d -> contiguous row-major gather, rows/cols each a group of legs
// (used by the contraction prep).  Equivalent to permute with the given axes.
// SIMT complex GEMM: C[m*ldcm + n*ldcn] = sum_k X[m*ldx + k] * Y[n*ldy + k]
int simt_cgemm_launch(int dtype, int64_t M, int64_t N, int64_t K, const void* X, int64_t ldx,
                      const void* Y, int64_t ldy, void* C, int64_t ldcm, int64_t ldcn,
                      int accumulate, cudaStream_t stream);
// split-K for tiny M*N, huge K: chunk partials in `parts` ([chunks][M][N]),
// then the fixed-order tree reduction into C
int64_t splitk_chunks(int64_t M, int64_t N, int64_t K);
int simt_splitk_launch(int dtype, int64_t M, int64_t N, int64_t K, const void* X, int64_t ldx,
                       const void* Y, int64_t ldy, void* C, int64_t ldcm, int64_t ldcn, void* parts,
                       cudaStream_t stream);
// split-K with in-kernel operand gathers: `tabs` = device [rowx(M) | rowy(N) |
// tx0 tx1 tx2 | ty0 ty1 ty2] (level sizes `lvl`), K index k = k0 + s0*(k1 + s1*k2)
int splitk_gather_launch(int dtype, int64_t M, int64_t N, int64_t K, const void* X, const void* Y,
                         const int64_t* tabs, const int64_t* lvl, int x_kfast, int y_kfast,
                         int64_t chunks, void* C, int64_t ldcm, int64_t ldcn, void* parts,
                         cudaStream_t stream);
// axpy y += x
int axpy_launch(int dtype, int64_t n, const void* x, void* y, cudaStream_t stream);
// 3xTF32 prep: split complex X[R, K] (row-major, K contiguous, leading dim ldx)
// into tf32 big / small planes.  mode 0: "A" planes (interleaved copy) of shape
// [R, 2*Kp]; mode 1: "B" expanded planes of shape [2R, 2*Kp] (rows 2r: (re,-im),
// 2r+1: (im, re)).  Columns >= 2K are zero.
int tf32_split_launch(int mode, int64_t R, int64_t K, int64_t Kp, const void* X, int64_t ldx,
                      void* big, void* small, cudaStream_t stream);
// 3xFP16 prep: per-row power-of-two scaled hi/lo fp16 planes (same shapes as
// tf32_split_launch, 2-byte elements) + per-row scale exponents
int f16_split_launch(int mode, int64_t R, int64_t K, int64_t Kp, const void* X, int64_t ldx,
                     void* hi, void* lo, int* exps, void* scratch /* 4*R bytes */,
                     cudaStream_t stream);
// tcgen05 complex GEMM on prepared planes (see tnc_gemm_tc.cu).  f16 = 0:
// 3xTF32 fp32 planes; f16 = 1: 3xFP16 half planes with row/column scale
// exponents ex (rows of A) / ey (complex columns of C).
int tc_cgemm_launch(int f16, int64_t M, int64_t N, int64_t K, int64_t Kp, const void* Abig,
                    const void* Asmall, const void* Bbig, const void* Bsmall, const int* ex,
                    const int* ey, void* C, int64_t ldcm, int64_t ldcn, int k_splits,
                    float* partials, cudaStream_t stream,
                    const int64_t* row_off = nullptr, const int64_t* col_off = nullptr);
// fixed-order pairwise tree reduction of P partial [M,N] fp32-complex buffers
int tree_reduce_launch(int dtype, int64_t P, int64_t MN, void* partials, void* out_or_null,
                       int64_t M, int64_t N, int64_t ldcm, int64_t ldcn, cudaStream_t stream);

// K5 narrow-step streaming contraction (tnc_stream.cu).  Leg kinds: 0 =
// X-free, 1 = common, 2 = Y-free; extents are all 2.
struct StreamLeg {
  int kind;
  int64_t x_stride, y_stride, out_stride;
};
struct StreamPlan;
int stream_prepare(int n_legs, const StreamLeg* legs, StreamPlan** out);
void stream_destroy(StreamPlan* sp);
int stream_launch(const StreamPlan* sp, const void* x, const void* y, void* c, cudaStream_t stream);

// K4 step fusion (tnc_absorb.cu)
int absorb_chain_workspace(int t_rank, int n_gates, const int32_t* axes, size_t* bytes);
int absorb_chain_launch(int t_rank, const void* t_in, void* t_out, int n_gates, const void* const* gates,
                        const int64_t* gate_strides, const int32_t* axes, void* workspace,
                        size_t workspace_bytes, cudaStream_t stream);
void absorb_shutdown();
int absorb_chain_passes(int t_rank, int n_gates, const int32_t* axes, int* passes, int* groups);

}  // namespace tnc
