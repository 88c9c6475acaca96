// K2: complex GEMM on 5th-gen tensor cores, 3-product split, TMEM accumulate.
//
// Reference op: the np.matmul inside contract_pair (contract.py:131-165),
// which the reference runs in complex128 for "single" tensors
// (execute.py:154-158).  fp32 accuracy is kept with a 3-product split
//     x*y ~= hi(x)*hi(y) + hi(x)*lo(y) + lo(x)*hi(y)
// issued as three tcgen05.mma into one fp32 TMEM accumulator.  Two operand
// formats (template flag F16):
//   * 3xFP16 (AUTO default): hi = fp16(x * 2^-e), lo = fp16(x * 2^-e - hi)
//     with a per-row power-of-two scale (f16_row_exponent), kind::f16;
//     the epilogue multiplies by 2^(e_row + e_col);
//   * 3xTF32 (TNC_TC_TF32=1, and K <= 16): big = nearest TF32, small =
//     x - big, kind::tf32.
//
// Complex arithmetic is folded into ONE real GEMM:
//     A  (complex [M, K], interleaved)      == real [M, 2K]
//     B^ (real [2N, 2K], K-major): row 2n = (Br, -Bi) pairs, row 2n+1 = (Bi, Br)
//     D = A . B^T  (real [M, 2N]) == complex C [M, N] interleaved.
// The operand planes (big/small, zero-padded to Kp) come from
// tf32_split_kernel; this kernel streams them with TMA (swizzled) into a
// multi-stage smem ring and one elected thread issues the MMAs.
//
// Accuracy: measured on B200, the tensor-core fp32 accumulation error grows
// LINEARLY with the accumulation chain (rel-L2 ~1.4e-8 per complex K), so a
// K = 2^15 contraction accumulated in TMEM alone would miss the 1e-5 contract.
// The MMA warp therefore accumulates short K-chunks (kb_per_chunk k-blocks)
// into alternating TMEM buffers and the epilogue warps fold each finished
// chunk into fp32 registers with round-to-nearest adds (error independent of
// K: ~4e-7 per GEMM with 32-complex-K chunks, ~1e-6 with the 128-K chunks
// the 3xFP16 path uses by default).
//
// Roles (320 threads, persistent over (split, m, n) work units):
//   warp 0     TMA producer (one elected lane)
//   warp 1     TMEM owner + MMA issuer (one elected lane)
//   warps 2..9 chunk reducers / epilogue: warp w reads TMEM lane quadrant
//              w % 4 and column half (w - 2) / 4, keeps BN/2 fp32 running sums
//              per thread, writes C (any strides) or split-K partials.
#include <cuda.h>

#include <algorithm>
#include <mutex>

#include "tnc_common.cuh"
#include "tnc_tcgen05.cuh"

namespace tnc {

namespace {

constexpr int kBM = 128;  // rows of A per CTA (TMEM lanes)
constexpr int kThreads = 320;
constexpr int kEpiWarps = 8;

using namespace tc5;  // mbarrier / commit / TMEM-load wrappers shared with the gather-fed kernel

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst,
                                            int32_t c0, int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

// K-major operand in the canonical swizzled layout: 8-row atoms of 8*SWZ
// bytes (SBO), rows SWZ bytes long.  SWZ = 128 -> layout 2, SWZ = 64 -> 4.
template <int SWZ>
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;                  // LBO (ignored when swizzled)
  d |= static_cast<uint64_t>((8 * SWZ) >> 4) << 32;     // SBO: one 8-row atom
  d |= static_cast<uint64_t>(1) << 46;                  // sm100 descriptor version
  d |= static_cast<uint64_t>(SWZ == 128 ? 2 : 4) << 61; // swizzle mode
  return d;
}

// Whole-warp variants: every lane runs the (warp-uniform) issue loop and
// elect.sync picks the issuing lane inside the asm, so the compiler keeps the
// operands in uniform registers instead of wrapping each MMA in a
// single-lane waterfall loop (ncu: ~15 dependent instructions per MMA).
template <int CG, bool F16>
__device__ __forceinline__ void mma_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
  if constexpr (CG == 1 && F16) {
    asm volatile(
        "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else if constexpr (CG == 1) {
    asm volatile(
        "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else if constexpr (F16) {
    asm volatile(
        "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  } else {
    asm volatile(
        "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
        "@e tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
  }
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

struct TcParams {
  int64_t M, N;          // complex rows of A / complex columns of C
  int num_kb;            // k-blocks over the padded real K
  int kb_per_split;      // k-blocks per split-K unit
  int splits;
  int m_blocks, n_blocks;
  int group_m;           // raster group height (m-blocks)
  int kb_per_chunk;      // k-blocks accumulated in TMEM before a register fold
  float2* C;
  int64_t ldcm, ldcn;    // complex strides of C[m, n]
  float2* partials;      // [splits][M][N] when splits > 1
  const int* ex;         // 3xFP16: per-row scale exponent of A (nullptr for TF32)
  const int* ey;         // 3xFP16: per-complex-column scale exponent of B
  // fused output permutation (one split): C[row_off[m] + col_off[n]] -- the
  // caller's leg order is a permutation of the row legs and the column legs,
  // so the offset of C[m, n] separates into a row part and a column part
  const int64_t* row_off;
  const int64_t* col_off;
};

// Undo the 3xFP16 per-row / per-column power-of-two operand scaling of one
// thread's row segment (HALF fp32 = HALF/2 complex columns from ncol0).  The
// column exponents come in as 16-byte vectors (ncol0 is a multiple of 4 and
// the exponent array is 256-byte aligned); columns past N get exponent 0.
template <int HALF>
__device__ __forceinline__ void unscale(float (&acc)[HALF], const TcParams& p, int64_t row, int64_t ncol0) {
  const int er = p.ex[row];
  const int4* ey4 = reinterpret_cast<const int4*>(p.ey + ncol0);
#pragma unroll
  for (int q = 0; q < HALF / 8; ++q) {
    int4 e = make_int4(0, 0, 0, 0);
    if (ncol0 + 4 * q + 4 <= p.N) {
      e = __ldg(ey4 + q);
    } else {
      if (ncol0 + 4 * q + 0 < p.N) e.x = p.ey[ncol0 + 4 * q + 0];
      if (ncol0 + 4 * q + 1 < p.N) e.y = p.ey[ncol0 + 4 * q + 1];
      if (ncol0 + 4 * q + 2 < p.N) e.z = p.ey[ncol0 + 4 * q + 2];
    }
    const int es[4] = {er + e.x, er + e.y, er + e.z, er + e.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (es[j] >= -126 && es[j] <= 127) {
        const float sc = __int_as_float((es[j] + 127) << 23);
        acc[8 * q + 2 * j] *= sc;
        acc[8 * q + 2 * j + 1] *= sc;
      } else {  // combined scale outside the normal range: exact ldexp on the value
        acc[8 * q + 2 * j] = ldexpf(acc[8 * q + 2 * j], es[j]);
        acc[8 * q + 2 * j + 1] = ldexpf(acc[8 * q + 2 * j + 1], es[j]);
      }
    }
  }
}

template <int BN, int SWZ, int STAGES, bool F16>
struct TcCfg {
  static constexpr int kElem = F16 ? 2 : 4;         // bytes per plane element
  static constexpr int kBK = SWZ / kElem;           // real K per k-block
  static constexpr int kABytes = kBM * SWZ;         // one A plane tile
  static constexpr int kBBytes = BN * SWZ;          // one B plane tile
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kSmem = STAGES * kStageBytes + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr int kHalf = BN / 2;              // columns per epilogue warp
  static constexpr int kMmaPerKb = SWZ / 32;        // one MMA consumes 32 bytes of K
  // instruction descriptor: D=f32, A=B=tf32 (2) or f16 (0), K-major, N=BN, M=128
  static constexpr uint32_t kFmt = F16 ? 0u : 2u;
  static constexpr uint32_t kIdesc = (1u << 4) | (kFmt << 7) | (kFmt << 10) |
                                     (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(kBM >> 4) << 24);
};

__device__ __forceinline__ void decode_unit(const TcParams& p, int u, int& split, int& mb, int& nb) {
  const int tiles = p.m_blocks * p.n_blocks;
  split = u / tiles;
  const int t = u - split * tiles;
  const int span = p.group_m * p.n_blocks;
  const int g = t / span;
  const int first_m = g * p.group_m;
  const int gsize = min(p.group_m, p.m_blocks - first_m);
  const int r = t - g * span;
  mb = first_m + r % gsize;
  nb = r / gsize;
}

template <int BN, int SWZ, int STAGES, bool F16>
__global__ void __launch_bounds__(kThreads, 1)
    tc_cgemm_kernel(const __grid_constant__ CUtensorMap mapAb,
                    const __grid_constant__ CUtensorMap mapAs,
                    const __grid_constant__ CUtensorMap mapBb,
                    const __grid_constant__ CUtensorMap mapBs, const TcParams p) {
  using Cfg = TcCfg<BN, SWZ, STAGES, F16>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;   // [2] chunk ready in TMEM buffer b
  uint64_t* tempty = tfull + 2;       // [2] TMEM buffer b drained
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int units = p.m_blocks * p.n_blocks * p.splits;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(static_cast<uint32_t>(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapAb)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapAs)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBb)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mapBs)) : "memory");
      uint32_t it = 0;
      for (int u = blockIdx.x; u < units; u += gridDim.x) {
        int split, mb, nb;
        decode_unit(p, u, split, mb, nb);
        const int kb_lo = split * p.kb_per_split;
        const int kb_hi = min(p.num_kb, kb_lo + p.kb_per_split);
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * Cfg::kStageBytes;
          mbar_expect_tx(&full[s], Cfg::kStageBytes);
          const int kc = kb * Cfg::kBK;
          tma_load_2d(&mapAb, &full[s], st, kc, mb * kBM);
          tma_load_2d(&mapAs, &full[s], st + Cfg::kABytes, kc, mb * kBM);
          tma_load_2d(&mapBb, &full[s], st + 2 * Cfg::kABytes, kc, nb * BN);
          tma_load_2d(&mapBs, &full[s], st + 2 * Cfg::kABytes + Cfg::kBBytes, kc, nb * BN);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // whole warp, warp-uniform control flow; one elected lane issues
    const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
    const uint64_t dhi = umma_desc<SWZ>(0);  // descriptor without the address field
    const uint32_t smem0 = smem_u32(smem);
    uint32_t it = 0, ch = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int split, mb, nb;
      decode_unit(p, u, split, mb, nb);
      const int kb_lo = split * p.kb_per_split;
      const int kb_hi = min(p.num_kb, kb_lo + p.kb_per_split);
      int in_chunk = 0;
      uint32_t dcol = 0;
      for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
        if (in_chunk == 0) {
          const uint32_t b = ch & 1;
          mbar_wait(&tempty[b], ((ch >> 1) & 1) ^ 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          dcol = tbase + b * BN;
        }
        const int s = it % STAGES;
        const uint32_t ph = (it / STAGES) & 1;
        mbar_wait(&full[s], ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t st = smem0 + s * Cfg::kStageBytes;
        // address field = bits [0,14) of (addr >> 4); 32 bytes of K = +2
        const uint64_t a_big = dhi | ((st >> 4) & 0x3FFF);
        const uint64_t a_small = dhi | (((st + Cfg::kABytes) >> 4) & 0x3FFF);
        const uint64_t b_big = dhi | (((st + 2 * Cfg::kABytes) >> 4) & 0x3FFF);
        const uint64_t b_small = dhi | (((st + 2 * Cfg::kABytes + Cfg::kBBytes) >> 4) & 0x3FFF);
#pragma unroll
        for (int kk = 0; kk < Cfg::kMmaPerKb; ++kk) {
          const uint64_t o = 2 * kk;
          const uint32_t acc0 = (in_chunk > 0 || kk > 0) ? 1u : 0u;
          mma_elect<1, F16>(dcol, a_small + o, b_big + o, Cfg::kIdesc, acc0);
          mma_elect<1, F16>(dcol, a_big + o, b_small + o, Cfg::kIdesc, 1u);
          mma_elect<1, F16>(dcol, a_big + o, b_big + o, Cfg::kIdesc, 1u);
        }
        mma_commit_elect(&empty[s]);
        ++in_chunk;
        if (in_chunk == p.kb_per_chunk || kb + 1 == kb_hi) {
          mma_commit_elect(&tfull[ch & 1]);
          ++ch;
          in_chunk = 0;
        }
      }
    }
    __syncwarp();
  } else {
    // chunk reducers + epilogue
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    float acc[Cfg::kHalf];
    uint32_t ch = 0;
    for (int u = blockIdx.x; u < units; u += gridDim.x) {
      int split, mb, nb;
      decode_unit(p, u, split, mb, nb);
      const int kb_lo = split * p.kb_per_split;
      const int kb_hi = min(p.num_kb, kb_lo + p.kb_per_split);
      const int nchunks = (kb_hi - kb_lo + p.kb_per_chunk - 1) / p.kb_per_chunk;
      for (int c = 0; c < nchunks; ++c, ++ch) {
        const uint32_t b = ch & 1;
        mbar_wait(&tfull[b], (ch >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t taddr = tmem_base + lane_base + b * BN + half * Cfg::kHalf;
#pragma unroll
        for (int g = 0; g < Cfg::kHalf / 32; ++g) {
          uint32_t v[32];
          tmem_ld32(taddr + g * 32, v);
          if (c == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[g * 32 + j] = __uint_as_float(v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[g * 32 + j] += __uint_as_float(v[j]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[b]);
      }
      if (nchunks == 0) {
#pragma unroll
        for (int j = 0; j < Cfg::kHalf; ++j) acc[j] = 0.f;
      }
      // store this thread's row: complex columns [ncol0, ncol0 + kHalf/2)
      const int64_t row = static_cast<int64_t>(mb) * kBM + quad * 32 + lane;
      if (row < p.M) {
        const int64_t ncol0 = (static_cast<int64_t>(nb) * BN + half * Cfg::kHalf) / 2;
        float2* dst;
        int64_t sm, sn;
        if (p.splits > 1) {
          dst = p.partials + static_cast<int64_t>(split) * p.M * p.N;
          sm = p.N;
          sn = 1;
        } else {
          dst = p.C;
          sm = p.ldcm;
          sn = p.ldcn;
        }
        float2* drow = dst + row * sm;
        if constexpr (F16) unscale<Cfg::kHalf>(acc, p, row, ncol0);
        if (p.col_off != nullptr && p.splits == 1) {
          float2* prow = p.C + p.row_off[row];
#pragma unroll
          for (int j = 0; j < Cfg::kHalf / 2; ++j) {
            const int64_t n = ncol0 + j;
            if (n < p.N) prow[__ldg(p.col_off + n)] = make_float2(acc[2 * j], acc[2 * j + 1]);
          }
        } else if (sn == 1 && (sm % 2) == 0 && ncol0 + Cfg::kHalf / 2 <= p.N) {
          float4* d4 = reinterpret_cast<float4*>(drow + ncol0);
#pragma unroll
          for (int j = 0; j < Cfg::kHalf / 4; ++j)
            d4[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < Cfg::kHalf / 2; ++j) {
            const int64_t n = ncol0 + j;
            if (n < p.N) drow[n * sn] = make_float2(acc[2 * j], acc[2 * j + 1]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(static_cast<uint32_t>(2 * BN)));
  }
}

// ============================================================================
// 2-CTA variant (cta_group::2): a CTA pair computes a 256 x BN tile; each CTA
// stages its own 128 A rows and HALF of the B tile (BN/2 rows), so per-SM
// operand traffic (smem writes, L2 reads) drops by a third and the leader's
// single-thread MMA issue drives both SMs' tensor cores.
//   leader (rank 0): TMA producer, MMA issuer, epilogue of rows 0..127
//   peer   (rank 1): TMA producer (signals the leader's barrier), epilogue of
//                    rows 128..255 (its own TMEM half)
// ============================================================================

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__device__ __forceinline__ uint32_t map_to_rank(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}

__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}

__device__ __forceinline__ bool mbar_try_cluster(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2, %3;\n"
      "selp.u32 %0, 1, 0, P1;\n"
      "}\n"
      : "=r"(ok)
      : "r"(addr), "r"(parity), "r"(0x989680)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (uint32_t spin = 0; !mbar_try_cluster(addr, parity); ++spin) {
    if (spin > (1u << 24)) __trap();
  }
}

// TMA load into this CTA's smem whose completion is counted on the LEADER's
// barrier (peer bit cleared), as the 2-SM MMA consumes both CTAs' tiles.
__device__ __forceinline__ void tma_load_2d_2sm(const CUtensorMap* map, uint64_t* bar, void* dst,
                                                int32_t c0, int32_t c1) {
  const uint32_t mbar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(mbar), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void mma_commit_2sm_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

template <int BN, int SWZ, int STAGES, bool F16>
struct Tc2Cfg {
  static constexpr int kElem = F16 ? 2 : 4;
  static constexpr int kBK = SWZ / kElem;
  static constexpr int kABytes = kBM * SWZ;          // own 128 rows of one A plane
  static constexpr int kBBytes = (BN / 2) * SWZ;     // own half of one B plane
  static constexpr int kStageBytes = 2 * kABytes + 2 * kBBytes;
  static constexpr int kSmem = STAGES * kStageBytes + 1024 + 256;
  static constexpr int kHalf = BN / 2;
  static constexpr int kMmaPerKb = SWZ / 32;
  static constexpr uint32_t kFmt = F16 ? 0u : 2u;
  static constexpr uint32_t kIdesc = (1u << 4) | (kFmt << 7) | (kFmt << 10) |
                                     (static_cast<uint32_t>(BN >> 3) << 17) |
                                     (static_cast<uint32_t>(256 >> 4) << 24);
};

template <int BN, int SWZ, int STAGES, bool F16>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc_cgemm_2sm_kernel(const __grid_constant__ CUtensorMap mapAb,
                        const __grid_constant__ CUtensorMap mapAs,
                        const __grid_constant__ CUtensorMap mapBb,
                        const __grid_constant__ CUtensorMap mapBs, const TcParams p) {
  using Cfg = Tc2Cfg<BN, SWZ, STAGES, F16>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int units = p.m_blocks * p.n_blocks * p.splits;  // m_blocks of 256 rows
  const int pair = blockIdx.x >> 1;
  const int pairs = gridDim.x >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(static_cast<uint32_t>(2 * BN)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync_all();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int u = pair; u < units; u += pairs) {
        int split, mb, nb;
        decode_unit(p, u, split, mb, nb);
        const int kb_lo = split * p.kb_per_split;
        const int kb_hi = min(p.num_kb, kb_lo + p.kb_per_split);
        const int arow = mb * 256 + static_cast<int>(rank) * kBM;
        const int brow = nb * BN + static_cast<int>(rank) * (BN / 2);
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          uint8_t* st = smem + s * Cfg::kStageBytes;
          if (leader) mbar_expect_tx(&full[s], 2 * Cfg::kStageBytes);
          const int kc = kb * Cfg::kBK;
          tma_load_2d_2sm(&mapAb, &full[s], st, kc, arow);
          tma_load_2d_2sm(&mapAs, &full[s], st + Cfg::kABytes, kc, arow);
          tma_load_2d_2sm(&mapBb, &full[s], st + 2 * Cfg::kABytes, kc, brow);
          tma_load_2d_2sm(&mapBs, &full[s], st + 2 * Cfg::kABytes + Cfg::kBBytes, kc, brow);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (leader) {
      // whole warp, warp-uniform control flow; one elected lane issues
      const uint32_t tbase = __shfl_sync(0xffffffffu, tmem_base, 0);
      const uint64_t dhi = umma_desc<SWZ>(0);
      const uint32_t smem0 = smem_u32(smem);
      uint32_t it = 0, ch = 0;
      for (int u = pair; u < units; u += pairs) {
        int split, mb, nb;
        decode_unit(p, u, split, mb, nb);
        const int kb_lo = split * p.kb_per_split;
        const int kb_hi = min(p.num_kb, kb_lo + p.kb_per_split);
        int in_chunk = 0;
        uint32_t dcol = 0;
        for (int kb = kb_lo; kb < kb_hi; ++kb, ++it) {
          if (in_chunk == 0) {
            const uint32_t b = ch & 1;
            mbar_wait_cluster(&tempty[b], ((ch >> 1) & 1) ^ 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            dcol = tbase + b * BN;
          }
          const int s = it % STAGES;
          const uint32_t ph = (it / STAGES) & 1;
          mbar_wait(&full[s], ph);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint32_t st = smem0 + s * Cfg::kStageBytes;
          const uint64_t a_big = dhi | ((st >> 4) & 0x3FFF);
          const uint64_t a_small = dhi | (((st + Cfg::kABytes) >> 4) & 0x3FFF);
          const uint64_t b_big = dhi | (((st + 2 * Cfg::kABytes) >> 4) & 0x3FFF);
          const uint64_t b_small = dhi | (((st + 2 * Cfg::kABytes + Cfg::kBBytes) >> 4) & 0x3FFF);
#pragma unroll
          for (int kk = 0; kk < Cfg::kMmaPerKb; ++kk) {
            const uint64_t o = 2 * kk;
            const uint32_t acc0 = (in_chunk > 0 || kk > 0) ? 1u : 0u;
            mma_elect<2, F16>(dcol, a_small + o, b_big + o, Cfg::kIdesc, acc0);
            mma_elect<2, F16>(dcol, a_big + o, b_small + o, Cfg::kIdesc, 1u);
            mma_elect<2, F16>(dcol, a_big + o, b_big + o, Cfg::kIdesc, 1u);
          }
          mma_commit_2sm_elect(&empty[s]);
          ++in_chunk;
          if (in_chunk == p.kb_per_chunk || kb + 1 == kb_hi) {
            mma_commit_2sm_elect(&tfull[ch & 1]);
            ++ch;
            in_chunk = 0;
          }
        }
      }
    }
    __syncwarp();
  } else {
    const int quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const uint32_t lane_base = static_cast<uint32_t>(quad * 32) << 16;
    float acc[Cfg::kHalf];
    uint32_t ch = 0;
    for (int u = pair; u < units; u += pairs) {
      int split, mb, nb;
      decode_unit(p, u, split, mb, nb);
      const int kb_lo = split * p.kb_per_split;
      const int kb_hi = min(p.num_kb, kb_lo + p.kb_per_split);
      const int nchunks = (kb_hi - kb_lo + p.kb_per_chunk - 1) / p.kb_per_chunk;
      for (int c = 0; c < nchunks; ++c, ++ch) {
        const uint32_t b = ch & 1;
        mbar_wait(&tfull[b], (ch >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const uint32_t taddr = tmem_base + lane_base + b * BN + half * Cfg::kHalf;
#pragma unroll
        for (int g = 0; g < Cfg::kHalf / 32; ++g) {
          uint32_t v[32];
          tmem_ld32(taddr + g * 32, v);
          if (c == 0) {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[g * 32 + j] = __uint_as_float(v[j]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[g * 32 + j] += __uint_as_float(v[j]);
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(map_to_rank(smem_u32(&tempty[b]), 0));
      }
      if (nchunks == 0) {
#pragma unroll
        for (int j = 0; j < Cfg::kHalf; ++j) acc[j] = 0.f;
      }
      const int64_t row = static_cast<int64_t>(mb) * 256 + rank * kBM + quad * 32 + lane;
      if (row < p.M) {
        const int64_t ncol0 = (static_cast<int64_t>(nb) * BN + half * Cfg::kHalf) / 2;
        float2* dst;
        int64_t sm, sn;
        if (p.splits > 1) {
          dst = p.partials + static_cast<int64_t>(split) * p.M * p.N;
          sm = p.N;
          sn = 1;
        } else {
          dst = p.C;
          sm = p.ldcm;
          sn = p.ldcn;
        }
        float2* drow = dst + row * sm;
        if constexpr (F16) unscale<Cfg::kHalf>(acc, p, row, ncol0);
        if (sn == 1 && (sm % 2) == 0 && ncol0 + Cfg::kHalf / 2 <= p.N) {
          float4* d4 = reinterpret_cast<float4*>(drow + ncol0);
#pragma unroll
          for (int j = 0; j < Cfg::kHalf / 4; ++j)
            d4[j] = make_float4(acc[4 * j], acc[4 * j + 1], acc[4 * j + 2], acc[4 * j + 3]);
        } else {
#pragma unroll
          for (int j = 0; j < Cfg::kHalf / 2; ++j) {
            const int64_t n = ncol0 + j;
            if (n < p.N) drow[n * sn] = make_float2(acc[2 * j], acc[2 * j + 1]);
          }
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  cluster_sync_all();
  if (warp == 1) {
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(static_cast<uint32_t>(2 * BN)));
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
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  });
  return fn;
}

int make_map(CUtensorMap* map, const void* base, int64_t rows, int64_t cols_real, int box_rows,
             int swz, int elem) {
  EncodeFn enc = get_encode();
  if (!enc) TNC_RET(TNC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols_real), static_cast<cuuint64_t>(rows)};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(cols_real) * elem};
  cuuint32_t box[2] = {static_cast<cuuint32_t>(swz / elem), static_cast<cuuint32_t>(box_rows)};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, elem == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   2, const_cast<void*>(base), dims,
                   strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swz == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) TNC_RET(TNC_ERR_CUDA, "cuTensorMapEncodeTiled failed");
  return TNC_OK;
}

int env_int(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

template <int BN, int SWZ, int STAGES, bool F16>
int launch_cfg(int64_t M, int64_t N, int64_t K, int64_t Kp, const void* Ab, const void* As,
               const void* Bb, const void* Bs, const int* ex, const int* ey, void* C, int64_t ldcm,
               int64_t ldcn, int k_splits, float* partials, cudaStream_t stream,
               const int64_t* row_off = nullptr, const int64_t* col_off = nullptr) {
  using Cfg = TcCfg<BN, SWZ, STAGES, F16>;
  const int64_t Kr = 2 * Kp;
  CUtensorMap mAb, mAs, mBb, mBs;
  TNC_TRY(make_map(&mAb, Ab, M, Kr, kBM, SWZ, Cfg::kElem));
  TNC_TRY(make_map(&mAs, As, M, Kr, kBM, SWZ, Cfg::kElem));
  TNC_TRY(make_map(&mBb, Bb, 2 * N, Kr, BN, SWZ, Cfg::kElem));
  TNC_TRY(make_map(&mBs, Bs, 2 * N, Kr, BN, SWZ, Cfg::kElem));
  TcParams p{};
  p.M = M;
  p.N = N;
  p.num_kb = static_cast<int>(Kr / Cfg::kBK);
  const int splits = std::max(1, std::min(k_splits, p.num_kb));
  p.kb_per_split = static_cast<int>(ceil_div(p.num_kb, splits));
  p.splits = static_cast<int>(ceil_div(p.num_kb, p.kb_per_split));
  p.m_blocks = static_cast<int>(ceil_div(M, kBM));
  p.n_blocks = static_cast<int>(ceil_div(2 * N, BN));
  // raster group of 64 m-blocks: measured best on the C3/C4 GEMM shapes (+2-4% over 16;
  // >= 128 loses ~15%), ncu DRAM reads 818 -> 579 GB on the 2^(15,15,14) step
  p.group_m = std::max(1, env_int("TNC_GROUP_M", 64));
  // TMEM accumulation chain per register fold (see header comment): 128
  // complex K for 3xFP16 (measured rel-L2 ~1e-6 per GEMM; 32 K gives ~4e-7
  // but folds 4x as often, -2.5 % on C3 under the power cap), 32 for 3xTF32
  p.kb_per_chunk = std::max(1, env_int("TNC_CHUNK_KB", (F16 ? 256 : 64) / Cfg::kBK));
  p.C = static_cast<float2*>(C);
  p.ldcm = ldcm;
  p.ldcn = ldcn;
  p.partials = p.splits > 1 ? reinterpret_cast<float2*>(partials) : nullptr;
  p.ex = ex;
  p.ey = ey;
  if (row_off && p.splits != 1) TNC_RET(TNC_ERR_INVALID, "tc_cgemm: fused output order needs one split");
  p.row_off = row_off;
  p.col_off = col_off;
  const int64_t units = static_cast<int64_t>(p.m_blocks) * p.n_blocks * p.splits;
  if (units > INT32_MAX) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_cgemm: too many tiles");
  auto kern = tc_cgemm_kernel<BN, SWZ, STAGES, F16>;
  TNC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
  const int grid = static_cast<int>(std::min<int64_t>(units, num_sms()));
  {
    ProfScope prof(PROF_TC_GEMM, 8.0 * M * N * K,
                   8.0 * (double(M) * K + double(N) * K + double(M) * N), stream);
    kern<<<grid, kThreads, Cfg::kSmem, stream>>>(mAb, mAs, mBb, mBs, p);
    TNC_CHECK_LAUNCH();
  }
  if (p.splits > 1)
    return tree_reduce_launch(TNC_C64, p.splits, M * N, partials, C, M, N, ldcm, ldcn, stream);
  return TNC_OK;
}

template <int BN, int SWZ, int STAGES, bool F16>
int launch_cfg_2sm(int64_t M, int64_t N, int64_t K, int64_t Kp, const void* Ab, const void* As,
                   const void* Bb, const void* Bs, const int* ex, const int* ey, void* C, int64_t ldcm,
                   int64_t ldcn, int k_splits, float* partials, cudaStream_t stream) {
  using Cfg = Tc2Cfg<BN, SWZ, STAGES, F16>;
  const int64_t Kr = 2 * Kp;
  CUtensorMap mAb, mAs, mBb, mBs;
  TNC_TRY(make_map(&mAb, Ab, M, Kr, kBM, SWZ, Cfg::kElem));
  TNC_TRY(make_map(&mAs, As, M, Kr, kBM, SWZ, Cfg::kElem));
  TNC_TRY(make_map(&mBb, Bb, 2 * N, Kr, BN / 2, SWZ, Cfg::kElem));
  TNC_TRY(make_map(&mBs, Bs, 2 * N, Kr, BN / 2, SWZ, Cfg::kElem));
  TcParams p{};
  p.M = M;
  p.N = N;
  p.num_kb = static_cast<int>(Kr / Cfg::kBK);
  const int splits = std::max(1, std::min(k_splits, p.num_kb));
  p.kb_per_split = static_cast<int>(ceil_div(p.num_kb, splits));
  p.splits = static_cast<int>(ceil_div(p.num_kb, p.kb_per_split));
  p.m_blocks = static_cast<int>(ceil_div(M, 256));
  p.n_blocks = static_cast<int>(ceil_div(2 * N, BN));
  p.group_m = std::max(1, env_int("TNC_GROUP_M", 8));
  // 64 complex K per TMEM chain: the cross-CTA drain handshake needs >= 2
  // k-blocks per chunk to stay off the MMA critical path (~9e-7 rel-L2 / GEMM)
  p.kb_per_chunk = std::max(1, env_int("TNC_CHUNK_KB", 128 / Cfg::kBK));
  p.C = static_cast<float2*>(C);
  p.ldcm = ldcm;
  p.ldcn = ldcn;
  p.partials = p.splits > 1 ? reinterpret_cast<float2*>(partials) : nullptr;
  p.ex = ex;
  p.ey = ey;
  const int64_t units = static_cast<int64_t>(p.m_blocks) * p.n_blocks * p.splits;
  if (units > INT32_MAX) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_cgemm: too many tiles");
  auto kern = tc_cgemm_2sm_kernel<BN, SWZ, STAGES, F16>;
  TNC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
  const int pairs = static_cast<int>(std::min<int64_t>(units, num_sms() / 2));
  {
    ProfScope prof(PROF_TC_GEMM, 8.0 * M * N * K,
                   8.0 * (double(M) * K + double(N) * K + double(M) * N), stream);
    kern<<<2 * pairs, kThreads, Cfg::kSmem, stream>>>(mAb, mAs, mBb, mBs, p);
    TNC_CHECK_LAUNCH();
  }
  if (p.splits > 1)
    return tree_reduce_launch(TNC_C64, p.splits, M * N, partials, C, M, N, ldcm, ldcn, stream);
  return TNC_OK;
}

}  // namespace

int tc_cgemm_launch(int f16, int64_t M, int64_t N, int64_t K, int64_t Kp, const void* Abig,
                    const void* Asmall, const void* Bbig, const void* Bsmall, const int* ex,
                    const int* ey, void* C, int64_t ldcm, int64_t ldcn, int k_splits,
                    float* partials, cudaStream_t stream, const int64_t* row_off, const int64_t* col_off) {
  if (M <= 0 || N <= 0) return TNC_OK;
  if (Kp % (f16 ? 32 : 16) != 0)
    TNC_RET(TNC_ERR_INVALID, "tc_cgemm: Kp must be a multiple of 32 (f16) / 16 (tf32)");
  const int cfg = env_int("TNC_TC_CFG", 0);
#define TNC_TC_ARGS M, N, K, Kp, Abig, Asmall, Bbig, Bsmall, ex, ey, C, ldcm, ldcn, k_splits, partials, stream
#define TNC_TC_ARGS_OUT TNC_TC_ARGS, row_off, col_off
  if (f16) {
    if (2 * N >= 256) {
      if (cfg == 1) return launch_cfg<256, 64, 4, true>(TNC_TC_ARGS_OUT);
      // the 2-CTA kernel (cfg 2) wins on square 8192^3 but loses on the C3
      // step shapes; the 1-SM kernel is the default until that is understood
      if (cfg == 2 && M >= 256 && !row_off) return launch_cfg_2sm<256, 128, 3, true>(TNC_TC_ARGS);
      return launch_cfg<256, 128, 2, true>(TNC_TC_ARGS_OUT);
    }
    return launch_cfg<128, 128, 3, true>(TNC_TC_ARGS_OUT);
  }
  if (2 * N >= 256) {
    if (cfg == 1) return launch_cfg<256, 128, 2, false>(TNC_TC_ARGS_OUT);
    return launch_cfg<256, 64, 4, false>(TNC_TC_ARGS_OUT);
  }
  return launch_cfg<128, 64, 6, false>(TNC_TC_ARGS_OUT);
#undef TNC_TC_ARGS_OUT
#undef TNC_TC_ARGS
}

}  // namespace tnc
