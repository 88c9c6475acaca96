// K2: complex GEMM on 5th-gen tensor cores, 3xTF32 split, TMEM accumulate.
//
// Reference op: the np.matmul inside contract_pair (contract.py:131-165),
// which the reference runs in complex128 for "single" tensors
// (execute.py:154-158).  fp32 accuracy is kept with the 3xTF32 scheme
//     x*y ~= big(x)*big(y) + big(x)*small(y) + small(x)*big(y)
// (big = rna-rounded TF32, small = x - big), all three products issued as
// tcgen05.mma kind::tf32 into one fp32 TMEM accumulator.
//
// Complex arithmetic is folded into ONE real GEMM:
//     A  (complex [M, K], interleaved)      == real [M, 2K]
//     B^ (real [2N, 2K], K-major): row 2n = (Br, -Bi) pairs, row 2n+1 = (Bi, Br)
//     D = A . B^T  (real [M, 2N]) == complex C [M, N] interleaved.
// The operand planes (big/small, zero-padded to Kp) are produced by
// tf32_split_kernel; this kernel streams them with TMA (128B swizzle) into a
// multi-stage smem ring and one elected thread issues the MMAs.
//
// Roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM owner + MMA
// issuer, warps 2..5 = epilogue (TMEM -> registers -> global, any strides).
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "tnc_common.cuh"

namespace tnc {

namespace {

constexpr int kBM = 128;        // rows of A per CTA (TMEM lanes)
constexpr int kBK = 32;         // real K per stage = 128 B rows (SWIZZLE_128B atom)
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity), "r"(0x989680)
      : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand, 128B swizzle: 8-row atoms of 1024 B, SBO = 1024 B.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;             // LBO (unused for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;     // SBO
  d |= static_cast<uint64_t>(1) << 46;             // sm100 descriptor version
  d |= static_cast<uint64_t>(2) << 61;             // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
        "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
        "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
        "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

template <int BN, int STAGES>
struct TcCfg {
  static constexpr int kABytes = kBM * kBK * 4;     // one A plane tile
  static constexpr int kBBytes = BN * kBK * 4;      // one B plane tile
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kSmem = STAGES * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  // instruction descriptor: D=f32, A=B=tf32, both K-major, N, M=128
  static constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) |
                                     (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(kBM >> 4) << 24);
};

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc_cgemm_kernel(const __grid_constant__ CUtensorMap mapAb,
                    const __grid_constant__ CUtensorMap mapAs,
                    const __grid_constant__ CUtensorMap mapBb,
                    const __grid_constant__ CUtensorMap mapBs, int64_t M, int64_t N,
                    int num_kb_total, int kb_per_split, float2* __restrict__ C, int64_t ldcm,
                    int64_t ldcn, float2* __restrict__ partials) {
  using Cfg = TcCfg<BN, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t m0 = static_cast<int64_t>(blockIdx.y) * kBM;
  const int n0r = blockIdx.x * BN;  // real column (= 2 * complex column)
  const int split = blockIdx.z;
  const int kb_lo = split * kb_per_split;
  const int kb_hi = min(num_kb_total, kb_lo + kb_per_split);
  const int nkb = kb_hi - kb_lo;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(static_cast<uint32_t>(BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapAb)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBb)) : "memory");
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        uint8_t* st = smem + s * Cfg::kStageBytes;
        mbar_expect_tx(&full[s], Cfg::kStageBytes);
        const int kc = (kb_lo + i) * kBK;
        tma_load_2d(&mapAb, &full[s], st, kc, static_cast<int32_t>(m0));
        tma_load_2d(&mapAs, &full[s], st + Cfg::kABytes, kc, static_cast<int32_t>(m0));
        tma_load_2d(&mapBb, &full[s], st + 2 * Cfg::kABytes, kc, n0r);
        tma_load_2d(&mapBs, &full[s], st + 2 * Cfg::kABytes + Cfg::kBBytes, kc, n0r);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      for (int i = 0; i < nkb; ++i) {
        const int s = i % STAGES;
        const uint32_t ph = (i / STAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = smem_u32(smem + s * Cfg::kStageBytes);
        const uint32_t a_big = st, a_small = st + Cfg::kABytes;
        const uint32_t b_big = st + 2 * Cfg::kABytes, b_small = b_big + Cfg::kBBytes;
#pragma unroll
        for (int kk = 0; kk < kBK / 8; ++kk) {
          const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
          const uint32_t acc0 = (i > 0 || kk > 0) ? 1u : 0u;
          mma_tf32(tmem_base, sw128_desc(a_small + off), sw128_desc(b_big + off), Cfg::kIdesc,
                   acc0);
          mma_tf32(tmem_base, sw128_desc(a_big + off), sw128_desc(b_small + off), Cfg::kIdesc, 1u);
          mma_tf32(tmem_base, sw128_desc(a_big + off), sw128_desc(b_big + off), Cfg::kIdesc, 1u);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // epilogue warps 2..5 -> TMEM lane quadrant (warp % 4)
    const int quad = warp & 3;
    const int64_t row = m0 + quad * 32 + lane;
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16);
    const int64_t ncplx0 = n0r / 2;
    float2* dst_base;
    int64_t sm, sn;
    if (partials != nullptr) {
      dst_base = partials + static_cast<int64_t>(split) * M * N;
      sm = N;
      sn = 1;
    } else {
      dst_base = C;
      sm = ldcm;
      sn = ldcn;
    }
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t v[32];
      tmem_ld32(t_row + c, v);
      if (row < M && nkb > 0) {
        float2* drow = dst_base + row * sm;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int64_t n = ncplx0 + c / 2 + j;
          if (n < N) drow[n * sn] = make_float2(__uint_as_float(v[2 * j]), __uint_as_float(v[2 * j + 1]));
        }
      } else if (row < M) {
        float2* drow = dst_base + row * sm;
        for (int j = 0; j < 16; ++j) {
          const int64_t n = ncplx0 + c / 2 + j;
          if (n < N) drow[n * sn] = make_float2(0.f, 0.f);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(static_cast<uint32_t>(BN)));
  }
}

// ---- host: tensor-map encoding through the driver entry point ----
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

int make_map(CUtensorMap* map, const float* base, int64_t rows, int64_t cols_real, int box_rows) {
  EncodeFn enc = get_encode();
  if (!enc) TNC_RET(TNC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols_real), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols_real) * 4};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) TNC_RET(TNC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return TNC_OK;
}

template <int BN, int STAGES>
int launch_cfg(int64_t M, int64_t N, int64_t Kp, const float* Ab, const float* As, const float* Bb,
               const float* Bs, void* C, int64_t ldcm, int64_t ldcn, int k_splits,
               float* partials, cudaStream_t stream) {
  using Cfg = TcCfg<BN, STAGES>;
  const int64_t Kr = 2 * Kp;
  CUtensorMap mAb, mAs, mBb, mBs;
  TNC_TRY(make_map(&mAb, Ab, M, Kr, kBM));
  TNC_TRY(make_map(&mAs, As, M, Kr, kBM));
  TNC_TRY(make_map(&mBb, Bb, 2 * N, Kr, BN));
  TNC_TRY(make_map(&mBs, Bs, 2 * N, Kr, BN));
  const int num_kb = static_cast<int>(Kr / kBK);
  const int splits = std::max(1, std::min(k_splits, num_kb));
  const int kb_per = static_cast<int>(ceil_div(num_kb, splits));
  const int real_splits = static_cast<int>(ceil_div(num_kb, kb_per));
  auto kern = tc_cgemm_kernel<BN, STAGES>;
  TNC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
  dim3 grid(static_cast<unsigned>(ceil_div(2 * N, BN)), static_cast<unsigned>(ceil_div(M, kBM)),
            static_cast<unsigned>(real_splits));
  if (grid.y > 65535) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_cgemm: M too large for grid");
  kern<<<grid, kThreads, Cfg::kSmem, stream>>>(mAb, mAs, mBb, mBs, M, N, num_kb, kb_per,
                                               static_cast<float2*>(C), ldcm, ldcn,
                                               real_splits > 1 ? reinterpret_cast<float2*>(partials)
                                                               : nullptr);
  TNC_CHECK_LAUNCH();
  if (real_splits > 1)
    return tree_reduce_launch(TNC_C64, real_splits, M * N, partials, C, M, N, ldcm, ldcn, stream);
  return TNC_OK;
}

}  // namespace

int tc_cgemm_launch(int64_t M, int64_t N, int64_t Kp, const float* Abig, const float* Asmall,
                    const float* Bbig, const float* Bsmall, void* C, int64_t ldcm, int64_t ldcn,
                    int k_splits, float* partials, cudaStream_t stream) {
  if (M <= 0 || N <= 0) return TNC_OK;
  if (Kp % 16 != 0) TNC_RET(TNC_ERR_INVALID, "tc_cgemm: Kp must be a multiple of 16");
  if (2 * N >= 256)
    return launch_cfg<256, 2>(M, N, Kp, Abig, Asmall, Bbig, Bsmall, C, ldcm, ldcn, k_splits,
                              partials, stream);
  return launch_cfg<128, 3>(M, N, Kp, Abig, Asmall, Bbig, Bsmall, C, ldcm, ldcn, k_splits,
                            partials, stream);
}

}  // namespace tnc
