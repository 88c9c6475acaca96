// K6: gather-fed tensor-core contraction (3xTF32 on tcgen05, split-K).
//
// Reference op: contract_pair (contract.py:131-165) = permute A and B into
// TTGT order (tensor.py:252-274), np.matmul, transpose -- and, for the
// small-M/N huge-K steps, split_common_contract's panel sum
// (contract.py:168-208).  Here the permutations never touch HBM: the
// kernel's worker warps gather each operand tile straight from the
// operand's own strided layout, split it into 3xTF32 big/small planes in
// shared memory (the canonical 128-byte-swizzled K-major UMMA layout), and
// one elected thread issues tcgen05.mma kind::tf32 into TMEM.  Every leg has
// extent 2 (quantum-circuit networks), so every index map is a GF(2)-linear
// function of the index bits: global offsets are sums of per-bit strides and
// swizzled smem addresses are XORs of per-bit addresses.
//
//   tile     = 128 rows of X (7 X-free legs R) x all Y columns (<= 128
//              complex, every Y-free leg) x one k-block of KBC complex K
//              (kb common legs KL); R and KL are chosen on the host so that
//              X, Y and the output are read / written in runs (tile bits
//              cover each tensor's fastest legs)
//   unit     = (m-block, k-split); persistent CTAs stride over units
//   complex  = one real GEMM: X interleaved [M, 2K] times the expanded Y^
//              (rows 2n = (Yr, -Yi), 2n+1 = (Yi, Yr)) gives interleaved C
//   accuracy = chunks of 128 complex K accumulate in alternating TMEM buffers
//              and are folded into fp32 registers (same scheme as K2)
//   output   = one split: C written in its FINAL (caller's) leg order; more
//              splits: fp32 partials [split][row][col] (canonical order),
//              then the fixed-order tree reduction
//
// Pair stores: every X smem store moves a K-adjacent element pair, 16 bytes per
// plane.  The pair leg sits on k bit 0; when it is X's stride-1 leg the pair
// is also 16 contiguous bytes in HBM (memory pair: one 16-byte load, Y
// likewise when it is Y's stride-1 leg too), otherwise it is the thread's
// first iteration bit (register pair: two 8-byte loads, one 16-byte store).
//
// Roles.  256 worker threads (8 warps = 2 per SM sub-partition): every warp
// gathers + splits (loads run one k-block ahead of the smem stores), folds
// TMEM lane quadrant w % 4, column half w / 4, and stores.  MMA issue:
//   * <= 128-column tiles: warp 0 issues the MMAs of k-block g-1 right after
//     its loads of k-block g+1 (one elected lane); the narrowest tiles (<= 16
//     columns) run two such CTAs per SM (16-K k-blocks, 128 registers);
//   * 256-column tiles: a third warpgroup holds a dedicated MMA warp (384
//     threads; setmaxnreg gives the workers 240 registers, that warpgroup 24).
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <mutex>
#include <type_traits>
#include <vector>

#include "tnc_common.cuh"
#include "tnc_gather_tc.cuh"
#include "tnc_tcgen05.cuh"

namespace tnc {

namespace {

using namespace tc5;

constexpr int kGtWorkers = 256;
constexpr int kGtWorkerWarps = kGtWorkers / 32;
constexpr int kGtThreads = kGtWorkers;  // warp 0 also issues the MMAs (a dedicated ninth MMA warp measured 3 % slower:
                                        // 288 threads cap the kernel at 224 registers)
constexpr int kGtMaxBits = 12;          // tile bits per operand (7 row/col + 5 k)
constexpr int kGtTabs = 5;              // outer tables: xm, om, cm (m-block), xk, yk (k-block)

struct GtParams {
  const float2* X;
  const float2* Y;
  float2* C;            // final output (splits == 1)
  float2* parts;        // [splits][rows_x * rows_y] canonical order (splits > 1)
  const int64_t* tabs;  // [kGtTabs][4][256] outer-index offset tables
  int64_t m_blocks, kblocks, mn;
  int splits, chunk_kb;
  int rbits, fy;        // real row / column bits (phantom bits, stride 0, sit above)
  // tile bit j (thread bit j for j < 8, iteration bit j - 8 above): element
  // offset in the operand and XOR-linear smem byte address in the stage plane
  uint32_t xg[kGtMaxBits], xs[kGtMaxBits];
  uint32_t yg[kGtMaxBits], ys[kGtMaxBits];
  int64_t orow[7], crow[7];  // per tile-row bit: final / partial-layout stride
  int64_t ocol[7], ccol[7];  // per column bit
  // outer k-block index kb -> kb + 1 flips bit b = ctz(kb + 1) on and the bits
  // below it off: X / Y offsets move by these carry deltas
  int64_t dxk[32], dyk[32];
  // same for the m-block index mb -> mb + 1: X, final-output, partial offsets
  int64_t dxm[32], dom[32], dcm[32];
};

template <int NMMA, int KBC, int STAGES, bool PX, bool PY>
struct GtCfg {
  static constexpr int kLogK = KBC == 32 ? 5 : 4;
  static constexpr int kLogN = NMMA == 32 ? 4 : NMMA == 64 ? 5 : NMMA == 128 ? 6 : 7;  // log2(NMMA / 2)
  // tile bits of the gathered element grid (a paired leg is inside the element)
  static constexpr int kXBits = 7 + kLogK - (PX ? 1 : 0);
  static constexpr int kYBits = kLogN + kLogK - (PY ? 1 : 0);
  static constexpr int kXPer = 1 << (kXBits - 8);  // X elements (or pairs) per thread per k-block
  static constexpr int kYPer = 1 << (kYBits - 8);
  using XT = typename std::conditional<PX, float4, float2>::type;
  using YT = typename std::conditional<PY, float4, float2>::type;
  static constexpr bool kPre = NMMA <= 128;       // per-thread offsets kept in registers
  static constexpr int kAtoms = KBC / 16;         // 128-byte (16 complex) K atoms per k-block
  static constexpr int kXAtom = 128 * 128;
  static constexpr int kYAtom = NMMA * 128;
  static constexpr int kXPlane = kAtoms * kXAtom;
  static constexpr int kYPlane = kAtoms * kYAtom;
  static constexpr int kStage = 2 * kXPlane + 2 * kYPlane;
  static constexpr int kSmem = STAGES * kStage + 1024;
  static constexpr int kHalf = NMMA / 2;
  static constexpr uint32_t kIdesc = idesc_f32acc(2, 128, NMMA);
  static_assert(kSmem + 4096 <= 227 * 1024, "smem budget");
  static_assert(kXBits >= 8 && kYBits >= 8, "tile smaller than the CTA");
  static_assert(PX || kXPer >= 2, "register pairs need two elements per thread");
};

__device__ __forceinline__ int64_t tab4(const int64_t* t, int64_t idx) {
  return __ldg(t + (idx & 255)) + __ldg(t + 256 + ((idx >> 8) & 255)) +
         __ldg(t + 512 + ((idx >> 16) & 255)) + __ldg(t + 768 + ((idx >> 24) & 255));
}

// Element-slot part (tile bits >= the thread bits) of an offset / address:
// thread-independent, so with i unrolled the sums come straight from the
// parameter bank on the uniform datapath (no shared-memory round trip).
template <int FIRST, int LAST>
__device__ __forceinline__ uint32_t slot_sum(const uint32_t (&tab)[kGtMaxBits], int i) {
  uint32_t s = 0;
#pragma unroll
  for (int j = FIRST; j < LAST; ++j)
    if ((i >> (j - FIRST)) & 1) s += tab[j];
  return s;
}
template <int FIRST, int LAST>
__device__ __forceinline__ uint32_t slot_xor(const uint32_t (&tab)[kGtMaxBits], int i) {
  uint32_t s = 0;
#pragma unroll
  for (int j = FIRST; j < LAST; ++j)
    if ((i >> (j - FIRST)) & 1) s ^= tab[j];
  return s;
}

__device__ __forceinline__ float2 ldg_stream(const float2* p) {
  float2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];"
               : "=f"(v.x), "=f"(v.y)
               : "l"(p));
  return v;
}

// TF32 "big" part, round-half-away on the 13 dropped mantissa bits (two
// integer ops; the tensor core reads only the top 19 bits of each fp32)
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

__device__ __forceinline__ float4 ldg_stream4(const float2* p) {
  float4 v;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void sts4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

__device__ __forceinline__ void sts2(uint32_t addr, float a, float b) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ void split_range(const GtParams& p, int split, uint32_t& lo, uint32_t& hi) {
  if (p.splits == 1) {
    lo = 0;
    hi = static_cast<uint32_t>(p.kblocks);
  } else {
    lo = static_cast<uint32_t>(p.kblocks * split / p.splits);
    hi = static_cast<uint32_t>(p.kblocks * (split + 1) / p.splits);
  }
}

// Unit / k-block cursor over this CTA's contiguous range of (m-block,
// split) units (split fastest).  Consecutive units move mb by at most one,
// so owners advance their m-block offsets with carry deltas instead of table
// lookups; the only division happens once, at init.
struct GtCursor {
  uint32_t u, u_end, mb, split;
  int carry;  // after next() == 2: the bit of mb that turned on
  uint32_t kb, kb_hi;
  __device__ __forceinline__ bool valid() const { return u < u_end; }
  __device__ __forceinline__ void init(const GtParams& p, uint32_t units) {
    u = static_cast<uint32_t>(static_cast<uint64_t>(blockIdx.x) * units / gridDim.x);
    u_end = static_cast<uint32_t>(static_cast<uint64_t>(blockIdx.x + 1) * units / gridDim.x);
    const uint32_t splits = static_cast<uint32_t>(p.splits);
    mb = splits == 1 ? u : u / splits;
    split = u - mb * splits;
    carry = 0;
    split_range(p, static_cast<int>(split), kb, kb_hi);
  }
  // advance one unit: 1 = same m-block (next split), 2 = next m-block
  __device__ __forceinline__ int next_unit(const GtParams& p) {
    ++u;
    int moved = 1;
    if (++split == static_cast<uint32_t>(p.splits)) {
      split = 0;
      ++mb;
      carry = __ffs(mb) - 1;
      moved = 2;
    }
    if (valid()) split_range(p, static_cast<int>(split), kb, kb_hi);
    return moved;
  }
  // advance one k-block: 0 = same unit, else next_unit()'s code
  __device__ __forceinline__ int next(const GtParams& p) {
    if (++kb < kb_hi) return 0;
    return next_unit(p);
  }
};

// MW (256-column tiles): a third warpgroup holds a dedicated MMA-issue warp.
// A clock64 trace showed warp 0 spending a third of every k-block inside the
// MMA issue (the issue blocks while the tensor pipe works through the queue)
// while the other seven workers waited half of theirs for the stage that only
// warp 0's late issue would release.  The block launches with 384 threads x
// 168 registers; the MMA warpgroup drops to 24 and the workers rise to 240.
template <int NMMA, int KBC, int STAGES, bool PX, bool PY, int OCC, bool MW = false>
__global__ void __launch_bounds__(MW ? kGtThreads + 128 : kGtThreads, OCC) gather_tc_kernel(const __grid_constant__ GtParams p) {
  using Cfg = GtCfg<NMMA, KBC, STAGES, PX, PY>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ int64_t ocol_t[128], ccol_t[128], dxk[32], dyk[32], dxm[32], dom[32], dcm[32];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int t = threadIdx.x;
  const uint32_t units = static_cast<uint32_t>(p.m_blocks * p.splits);

  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kGtWorkers);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kGtWorkerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t < 32) {
    dxk[t] = p.dxk[t];
    dyk[t] = p.dyk[t];
    dxm[t] = p.dxm[t];
    dom[t] = p.dom[t];
    dcm[t] = p.dcm[t];
  }
  if (t < 128) {
    int64_t o = 0, c = 0;
    for (int j = 0; j < p.fy; ++j)
      if ((t >> j) & 1) {
        o += p.ocol[j];
        c += p.ccol[j];
      }
    ocol_t[t] = o;
    ccol_t[t] = c;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "r"(static_cast<uint32_t>(2 * NMMA)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  fence_before_sync();
  __syncthreads();
  fence_after_sync();
  const uint32_t tmem_base = tmem_slot;
  const uint32_t smem0 = smem_u32(smem);

  // Barrier waits use the suspend-hinted try_wait: polling without the hint
  // (tried on the round-1 verdict's advice) measured 2-3 % slower on C1a / C1c,
  // and a run-time switch between the two cost another 3-7 % in registers.
  auto wait = [&](uint64_t* bar, uint32_t parity) { mbar_wait(bar, parity); };

  GtCursor ic;  // MMA issue (warp 0, or the MMA warp)
  ic.init(p, units);
  int i_in_chunk = 0;
  uint32_t i_ch = 0, i_g = 0, dcol = 0;
  // MMAs of the issue cursor's k-block (staged as k-block i_g): one elected lane
  auto issue_kblock = [&]() {
    if (i_in_chunk == 0) {
      const uint32_t b = i_ch & 1;
      wait(&tempty[b], ((i_ch >> 1) & 1) ^ 1);
      fence_after_sync();
      dcol = tmem_base + b * NMMA;
    }
    const uint32_t s = i_g % STAGES;
    wait(&full[s], (i_g / STAGES) & 1);
    fence_after_sync();
    const uint32_t st = smem0 + s * Cfg::kStage;
#pragma unroll
    for (int a = 0; a < Cfg::kAtoms; ++a) {
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t xs = st + a * Cfg::kXAtom + kk * 32;
        const uint32_t ys = st + 2 * Cfg::kXPlane + a * Cfg::kYAtom + kk * 32;
        const uint64_t x_big = umma_desc_sw128(xs);
        const uint64_t x_small = umma_desc_sw128(xs + Cfg::kXPlane);
        const uint64_t y_big = umma_desc_sw128(ys);
        const uint64_t y_small = umma_desc_sw128(ys + Cfg::kYPlane);
        const uint32_t acc0 = (i_in_chunk > 0 || a > 0 || kk > 0) ? 1u : 0u;
        // small products first: accumulated before the big one
        mma_tf32_elect(dcol, x_small, y_big, Cfg::kIdesc, acc0);
        mma_tf32_elect(dcol, x_big, y_small, Cfg::kIdesc, 1u);
        mma_tf32_elect(dcol, x_big, y_big, Cfg::kIdesc, 1u);
      }
    }
    mma_commit_elect(&empty[s]);
    ++i_g;
    const bool unit_end = ic.kb + 1 == ic.kb_hi;
    if (++i_in_chunk == p.chunk_kb || unit_end) {
      mma_commit_elect(&tfull[i_ch & 1]);
      ++i_ch;
      i_in_chunk = 0;
    }
    ic.next(p);
  };

  // Everything a worker warp does (gather, split, stage, fold, store); a lambda
  // so that, with a dedicated MMA warp, it sits inside the branch that starts
  // with the workers' setmaxnreg (ptxas allocates registers per such region).
  auto worker_body = [&]() {
  const int quad = warp & 3;
  const int half = warp >> 2;
  uint32_t xg_lo = 0, yg_lo = 0, xs_lo = 0, ys_lo = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if ((t >> j) & 1) {
      xg_lo += p.xg[j];
      xs_lo ^= p.xs[j];
      yg_lo += p.yg[j];
      ys_lo ^= p.ys[j];
    }
  }
  // per-thread element offsets / smem addresses of its tile elements
  uint32_t xo[Cfg::kPre ? Cfg::kXPer : 1], xa[Cfg::kPre ? Cfg::kXPer : 1];
  uint32_t yo[Cfg::kPre ? Cfg::kYPer : 1], ya[Cfg::kPre ? Cfg::kYPer : 1];
  if constexpr (Cfg::kPre) {
#pragma unroll
    for (int i = 0; i < Cfg::kXPer; ++i) {
      xo[i] = xg_lo + slot_sum<8, Cfg::kXBits>(p.xg, i);
      xa[i] = xs_lo ^ slot_xor<8, Cfg::kXBits>(p.xs, i);
    }
#pragma unroll
    for (int i = 0; i < Cfg::kYPer; ++i) {
      yo[i] = yg_lo + slot_sum<8, Cfg::kYBits>(p.yg, i);
      ya[i] = ys_lo ^ slot_xor<8, Cfg::kYBits>(p.ys, i);
    }
  }
  auto xoff = [&](int i) {
    if constexpr (Cfg::kPre) return xo[i];
    else return xg_lo + slot_sum<8, Cfg::kXBits>(p.xg, i);
  };
  auto xadr = [&](int i) {
    if constexpr (Cfg::kPre) return xa[i];
    else return xs_lo ^ slot_xor<8, Cfg::kXBits>(p.xs, i);
  };
  auto yoff = [&](int i) {
    if constexpr (Cfg::kPre) return yo[i];
    else return yg_lo + slot_sum<8, Cfg::kYBits>(p.yg, i);
  };
  auto yadr = [&](int i) {
    if constexpr (Cfg::kPre) return ya[i];
    else return ys_lo ^ slot_xor<8, Cfg::kYBits>(p.ys, i);
  };

  float acc[Cfg::kHalf];
#pragma unroll
  for (int j = 0; j < Cfg::kHalf; ++j) acc[j] = 0.f;
  GtCursor pc;  // loads (one k-block ahead of the smem stores)
  pc.init(p, units);
  // operand offsets of the load cursor's k-block
  int64_t xm_off = pc.valid() ? tab4(p.tabs, pc.mb) : 0, xk_off = 0, yk_off = 0;
  auto open_k = [&]() {  // first k-block of the cursor's (new) unit
    if (!pc.valid()) return;
    xk_off = pc.kb == 0 ? 0 : tab4(p.tabs + 3 * 1024, pc.kb);
    yk_off = pc.kb == 0 ? 0 : tab4(p.tabs + 4 * 1024, pc.kb);
  };
  open_k();
  GtCursor fc;  // fold: this CTA's chunk sequence
  fc.init(p, units);
  // final-output (one split) or partial-layout offset of the fold cursor's m-block
  const int64_t* dmo = p.splits == 1 ? dom : dcm;
  int64_t m_off = fc.valid() ? tab4(p.tabs + (p.splits == 1 ? 1 : 2) * 1024, fc.mb) : 0;
  int64_t f_n = fc.valid() ? fc.kb_hi - fc.kb : 0;
  int f_c = 0, f_nch = static_cast<int>((f_n + p.chunk_kb - 1) / p.chunk_kb);
  uint32_t f_base = 0, ch = 0;

  using XT = typename Cfg::XT;
  using YT = typename Cfg::YT;
  XT cx[Cfg::kXPer];
  YT cy[Cfg::kYPer];
  auto load = [&](XT (&vx)[Cfg::kXPer], YT (&vy)[Cfg::kYPer]) {
    const float2* xb = p.X + (xm_off + xk_off);
    const float2* yb = p.Y + yk_off;
#pragma unroll
    for (int i = 0; i < Cfg::kXPer; ++i) {
      if constexpr (PX) vx[i] = ldg_stream4(xb + xoff(i));
      else vx[i] = ldg_stream(xb + xoff(i));
    }
#pragma unroll
    for (int i = 0; i < Cfg::kYPer; ++i) {
      if constexpr (PY) vy[i] = __ldg(reinterpret_cast<const float4*>(yb + yoff(i)));
      else vy[i] = __ldg(yb + yoff(i));
    }
    const int b = __ffs(pc.kb + 1) - 1;  // carry bit of kb -> kb + 1
    const int moved = pc.next(p);
    if (moved == 0) {
      xk_off += dxk[b];
      yk_off += dyk[b];
    } else {
      if (moved == 2) xm_off += dxm[pc.carry];
      open_k();
    }
  };
  bool have = pc.valid();
  if (have) load(cx, cy);
  // Iteration with s0 = k-blocks staged so far:
  //   1. prefetch k-block s0 + 1 into registers
  //   2. warp 0 issues the MMAs of k-block s0 - 1 (staged last iteration), so
  //      the tensor pipe has work while k-block s0 is being staged
  //   3. stage k-block s0 (3xTF32 split into smem); needs MMA s0 - STAGES done
  //   4. fold the TMEM chunks ending at or before s0 - 1 (their MMAs were issued
  //      in step 2 at the latest); once nothing is left to stage, fold everything
  // A chunk's TMEM buffer is folded (step 4) before the MMAs that reuse it
  // are issued (step 2 of a later iteration), so no step waits on a later one.
  uint32_t staged = 0;
  while (true) {
    const uint32_t s0 = staged;
    XT nx[Cfg::kXPer];
    YT ny[Cfg::kYPer];
    bool have_next = false;
    if (have) {
      have_next = pc.valid();
      if (have_next) load(nx, ny);
    }
    if constexpr (!MW) {
      if (warp == 0) {
        while (i_g < s0) issue_kblock();
      }
    }
    if (have) {
      const uint32_t s = s0 % STAGES;
      wait(&empty[s], ((s0 / STAGES) & 1) ^ 1);
      const uint32_t st = smem0 + s * Cfg::kStage;
#pragma unroll
      for (int i = 0; i < Cfg::kXPer; ++i) {
        const uint32_t a = st + xadr(i);
        if constexpr (PX) {  // (k, k + 1) pair: 16 contiguous bytes per plane
          const float r0 = tf32_hi(cx[i].x), i0 = tf32_hi(cx[i].y), r1 = tf32_hi(cx[i].z), i1 = tf32_hi(cx[i].w);
          sts4(a, r0, i0, r1, i1);
          sts4(a + Cfg::kXPlane, cx[i].x - r0, cx[i].y - i0, cx[i].z - r1, cx[i].w - i1);
        } else if ((i & 1) == 0) {
          // register pair: elements i, i + 1 differ in k bit 0 (tile bit 8),
          // 16 contiguous bytes of the plane
          const float r0 = tf32_hi(cx[i].x), i0 = tf32_hi(cx[i].y);
          const float r1 = tf32_hi(cx[i + 1].x), i1 = tf32_hi(cx[i + 1].y);
          sts4(a, r0, i0, r1, i1);
          sts4(a + Cfg::kXPlane, cx[i].x - r0, cx[i].y - i0, cx[i + 1].x - r1, cx[i + 1].y - i1);
        }
      }
#pragma unroll
      for (int i = 0; i < Cfg::kYPer; ++i) {
        const uint32_t a0 = st + 2 * Cfg::kXPlane + yadr(i);
        const uint32_t a1 = a0 ^ 0x90u;  // row 2n+1 (row bit 0 and its swizzle bit)
        if constexpr (PY) {
          const float r0 = tf32_hi(cy[i].x), i0 = tf32_hi(cy[i].y), r1 = tf32_hi(cy[i].z), i1 = tf32_hi(cy[i].w);
          const float lr0 = cy[i].x - r0, li0 = cy[i].y - i0, lr1 = cy[i].z - r1, li1 = cy[i].w - i1;
          sts4(a0, r0, -i0, r1, -i1);
          sts4(a1, i0, r0, i1, r1);
          sts4(a0 + Cfg::kYPlane, lr0, -li0, lr1, -li1);
          sts4(a1 + Cfg::kYPlane, li0, lr0, li1, lr1);
        } else {
          const float hr = tf32_hi(cy[i].x), hi = tf32_hi(cy[i].y);
          const float lr = cy[i].x - hr, li = cy[i].y - hi;
          sts2(a0, hr, -hi);
          sts2(a1, hi, hr);
          sts2(a0 + Cfg::kYPlane, lr, -li);
          sts2(a1 + Cfg::kYPlane, li, lr);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      mbar_arrive(&full[s]);
      ++staged;
#pragma unroll
      for (int i = 0; i < Cfg::kXPer; ++i) cx[i] = nx[i];
#pragma unroll
      for (int i = 0; i < Cfg::kYPer; ++i) cy[i] = ny[i];
      have = have_next;
    }
    const bool drain = staged == s0;  // nothing staged: every MMA is issued
    while (fc.valid()) {
      const int64_t end = static_cast<int64_t>(f_c + 1) * p.chunk_kb;
      const int64_t last = static_cast<int64_t>(f_base) + (end < f_n ? end : f_n) - 1;
      // one iteration of slack: the MMAs of k-block s0 - 1 were issued earlier in
      // this iteration (or by the MMA warp as soon as it was staged), so the
      // chunk that ends there is folded now.  Two iterations measured C1a 0.83
      // vs 0.79 ms; zero would wait for MMAs this very warp has yet to issue.
      if (!drain && last + 1 > static_cast<int64_t>(s0)) break;
      const uint32_t b = ch & 1;
      wait(&tfull[b], (ch >> 1) & 1);
      fence_after_sync();
      const uint32_t taddr =
          tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + b * NMMA + half * Cfg::kHalf;
#pragma unroll
      for (int gi = 0; gi < Cfg::kHalf / 16; ++gi) {
        uint32_t v[16];
        tmem_ld16(taddr + gi * 16, v);
        tmem_wait_ld();
        if (f_c == 0) {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[gi * 16 + j] = __uint_as_float(v[j]);
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j) acc[gi * 16 + j] += __uint_as_float(v[j]);
        }
      }
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      ++ch;
      if (f_c == f_nch - 1) {
        // unit finished: store this thread's row (one TMEM lane), its column half
        const int r = quad * 32 + lane;
        const uint32_t split = fc.split;
        if (r < (1 << p.rbits)) {
          const int n0 = half * (Cfg::kHalf / 2);
          const int ncols = min(Cfg::kHalf / 2, (1 << p.fy) - n0);
          if (p.splits == 1) {
            int64_t base = m_off;
            for (int j = 0; j < p.rbits; ++j)
              if ((r >> j) & 1) base += p.orow[j];
#pragma unroll
            for (int j = 0; j < Cfg::kHalf / 2; ++j)
              if (j < ncols) p.C[base + ocol_t[n0 + j]] = make_float2(acc[2 * j], acc[2 * j + 1]);
          } else {
            int64_t base = static_cast<int64_t>(split) * p.mn + m_off;
            for (int j = 0; j < p.rbits; ++j)
              if ((r >> j) & 1) base += p.crow[j];
#pragma unroll
            for (int j = 0; j < Cfg::kHalf / 2; ++j)
              if (j < ncols) p.parts[base + ccol_t[n0 + j]] = make_float2(acc[2 * j], acc[2 * j + 1]);
          }
        }
        f_base += static_cast<uint32_t>(f_n);
        if (fc.next_unit(p) == 2) m_off += dmo[fc.carry];
        f_c = 0;
        if (fc.valid()) {
          f_n = fc.kb_hi - fc.kb;
          f_nch = static_cast<int>((f_n + p.chunk_kb - 1) / p.chunk_kb);
        }
      } else {
        ++f_c;
      }
    }
    if (drain && !fc.valid()) break;
  }
  };  // worker_body
  if constexpr (MW) {
    if (warp >= kGtWorkerWarps) {
      asm volatile("setmaxnreg.dec.sync.aligned.u32 24;");
      if (warp == kGtWorkerWarps) {  // the MMA warp: every k-block as soon as the workers have staged it
        while (ic.valid()) issue_kblock();
      }
    } else {
      asm volatile("setmaxnreg.inc.sync.aligned.u32 240;");
      worker_body();
    }
  } else {
    worker_body();
  }
  fence_before_sync();
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(static_cast<uint32_t>(2 * NMMA)));
  }
}

}  // namespace

struct GatherTcPlan {
  GtParams p;
  GtParams p2;              // paired layout (16-byte K pairs), when pair_x
  bool pair_x = false, pair_y = false;
  int nmma = 0, kbc = 0, occ = 1;  // occ: CTAs per SM (2 on the narrowest tiles)
  int64_t rows_x = 0, rows_y = 0, k = 0;
  std::vector<int64_t> tabs_host;
  mutable int64_t* tabs_dev = nullptr;
  ~GatherTcPlan() {
    if (tabs_dev) cudaFree(tabs_dev);
  }
};

namespace {

// 4 levels x 256 entries: T[l][v] = sum of strides[8l + b] over set bits b of v
void build_tab4(const std::vector<int64_t>& strides, int64_t* out) {
  for (int l = 0; l < 4; ++l)
    for (int v = 0; v < 256; ++v) {
      int64_t s = 0;
      for (int b = 0; b < 8; ++b)
        if (((v >> b) & 1) && 8 * l + b < static_cast<int>(strides.size())) s += strides[8 * l + b];
      out[l * 256 + v] = s;
    }
}

// Smem byte address (XOR-linear part) of one tile bit: X rows / Y^ rows of
// 128 bytes, 16-byte chunks swizzled by (row & 7), K atoms of atom_bytes.
uint32_t row_bit_addr(int row_bit) {
  const uint32_t rho = 1u << row_bit;
  return ((rho & 7u) << 4) | (rho << 7);
}
uint32_t k_bit_addr(int j, uint32_t atom_bytes) {
  if (j == 0) return 1u << 3;
  if (j <= 3) return 1u << (4 + j - 1);
  return (1u << (j - 4)) * atom_bytes;
}
// bank-selecting bits (byte address bits 3..6: the 8-byte slot in a 128-byte
// wavefront of a half-warp's 8-byte stores)
uint32_t bank4(uint32_t addr) { return (addr >> 3) & 15u; }

// 2^(n - rank): ways of the worst bank conflict of n lane bits' address vectors
int conflict_ways(const uint32_t* v, int n) {
  uint32_t rows[8];
  for (int i = 0; i < n; ++i) rows[i] = v[i];
  int rank = 0;
  for (int bit = 3; bit >= 0; --bit) {
    int piv = -1;
    for (int i = rank; i < n; ++i)
      if ((rows[i] >> bit) & 1) {
        piv = i;
        break;
      }
    if (piv < 0) continue;
    std::swap(rows[piv], rows[rank]);
    for (int i = 0; i < n; ++i)
      if (i != rank && ((rows[i] >> bit) & 1)) rows[i] ^= rows[rank];
    ++rank;
  }
  return 1 << (n - rank);
}

double eff(int run) { return std::min(1.0, std::ldexp(1.0, run) / 4.0) + 0.1 * std::min(1.0, std::ldexp(1.0, run) / 16.0); }

}  // namespace

int gather_tc_prepare(int n_legs, const GatherTcLeg* legs, GatherTcPlan** out) {
  *out = nullptr;
  std::vector<int> xf, cm, yf;  // indices into legs
  for (int i = 0; i < n_legs; ++i) {
    if (legs[i].kind == 0) xf.push_back(i);
    else if (legs[i].kind == 1) cm.push_back(i);
    else yf.push_back(i);
  }
  const int fx = static_cast<int>(xf.size()), c = static_cast<int>(cm.size()),
            fy = static_cast<int>(yf.size());
  if (fy > 7) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: Y has more than 128 columns");
  if (fx < 6) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: X has fewer than 64 rows");
  const int nmma = std::max(32, 2 << fy);
  const int lgn = nmma == 32 ? 4 : nmma == 64 ? 5 : nmma == 128 ? 6 : 7;  // log2(nmma / 2)
  // narrowest tiles (<= 16 Y columns): 16-K k-blocks and two CTAs per SM -- the
  // loop is a latency chain, and a second CTA hides it where more bytes in
  // flight per CTA did not
  const char* occ_s = std::getenv("TNC_GT_OCC2");
  const int occ = (nmma == 32 && !(occ_s && std::atoi(occ_s) == 0)) ? 2 : 1;
  const int kbc = (nmma <= 64 && occ == 1) ? 32 : 16;
  const int kb = kbc == 32 ? 5 : 4;
  if (c < kb) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: K smaller than one k-block");
  const int rb = std::min(7, fx);
  if (fx - rb > 31 || c - kb > 31) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: outer index > 31 bits");

  // ---- which legs form the tile: greedy on the access efficiency of X
  // reads, Y reads and output writes, weighted by their bytes
  const double rows_x = std::ldexp(1.0, fx), rows_y = std::ldexp(1.0, fy), kk = std::ldexp(1.0, c);
  const double wx = rows_x * kk, wy = rows_y * kk, wo = rows_x * rows_y;
  std::vector<int> xo(xf), yo(cm), oo(xf);  // per-tensor stride orders
  xo.insert(xo.end(), cm.begin(), cm.end());
  yo.insert(yo.end(), yf.begin(), yf.end());
  oo.insert(oo.end(), yf.begin(), yf.end());
  std::sort(xo.begin(), xo.end(), [&](int a, int b) { return legs[a].x_stride < legs[b].x_stride; });
  std::sort(yo.begin(), yo.end(), [&](int a, int b) { return legs[a].y_stride < legs[b].y_stride; });
  std::sort(oo.begin(), oo.end(), [&](int a, int b) { return legs[a].out_stride < legs[b].out_stride; });
  std::vector<char> inR(n_legs, 0), inK(n_legs, 0);
  int nR = 0, nK = 0;
  auto in_x = [&](int i) { return inR[i] || inK[i]; };
  auto in_y = [&](int i) { return legs[i].kind == 2 || inK[i]; };
  auto in_o = [&](int i) { return legs[i].kind == 2 || inR[i]; };
  auto run = [&](const std::vector<int>& order, auto in) {
    int r = 0;
    while (r < static_cast<int>(order.size()) && in(order[r])) ++r;
    return r;
  };
  auto first_missing = [&](const std::vector<int>& order, auto in) {
    for (int i : order)
      if (!in(i)) return i;
    return -1;
  };
  while (nR < rb || nK < kb) {
    double best = 0;
    int pick = -1;
    auto consider = [&](int leg, double w, const std::vector<int>& order, auto in) {
      if (leg < 0) return;
      const bool free_x = legs[leg].kind == 0;
      if (free_x ? nR >= rb : nK >= kb) return;
      const int before = run(order, in);
      (free_x ? inR : inK)[leg] = 1;
      const int after = run(order, in);
      (free_x ? inR : inK)[leg] = 0;
      const double gain = w * (eff(after) - eff(before));
      if (gain > best) {
        best = gain;
        pick = leg;
      }
    };
    consider(first_missing(xo, in_x), wx, xo, in_x);
    consider(first_missing(yo, in_y), wy, yo, in_y);
    consider(first_missing(oo, in_o), wo, oo, in_o);
    if (pick < 0) break;
    if (legs[pick].kind == 0) {
      inR[pick] = 1;
      ++nR;
    } else {
      inK[pick] = 1;
      ++nK;
    }
  }
  for (int i : xo) {  // fill what is left with X's fastest legs
    if (legs[i].kind == 0 && !inR[i] && nR < rb) {
      inR[i] = 1;
      ++nR;
    }
    if (legs[i].kind == 1 && !inK[i] && nK < kb) {
      inK[i] = 1;
      ++nK;
    }
  }
  std::vector<int> R, KL, outer_m, outer_k;
  for (int i : xf) (inR[i] ? R : outer_m).push_back(i);
  for (int i : cm) (inK[i] ? KL : outer_k).push_back(i);
  std::sort(outer_m.begin(), outer_m.end(), [&](int a, int b) { return legs[a].x_stride < legs[b].x_stride; });
  std::sort(outer_k.begin(), outer_k.end(), [&](int a, int b) { return legs[a].x_stride < legs[b].x_stride; });
  // tile orders (real legs by stride; phantom bits, if any, come after)
  std::vector<int> xt(R), yt(yf);
  xt.insert(xt.end(), KL.begin(), KL.end());
  yt.insert(yt.end(), KL.begin(), KL.end());
  std::sort(xt.begin(), xt.end(), [&](int a, int b) { return legs[a].x_stride < legs[b].x_stride; });
  std::sort(yt.begin(), yt.end(), [&](int a, int b) { return legs[a].y_stride < legs[b].y_stride; });

  // ---- bit assignment: rows of R -> row bits, KL -> k bits, Y-free -> column
  // bits.  Every smem store moves a K-adjacent element pair (16 bytes): one
  // common tile leg L, the pair leg, sits on k bit 0.
  //   memory pair (px / py): L is the operand's stride-1 leg, so the pair is
  //     also 16 contiguous bytes in HBM (one 16-byte load); L is inside the
  //     element, not a tile bit;
  //   register pair (otherwise): L is tile bit 8, the thread's first
  //     iteration bit, so its elements 2m and 2m + 1 are the pair (two 8-byte
  //     loads, one 16-byte store per plane).
  // A quarter-warp's 16-byte stores hit 8 distinct 16-byte chunks iff the
  // chunk vectors (address bits 4-6) of the operand's 3 fastest tile legs
  // (thread bits 0-2) are independent; search the assignments that decide them.
  const uint32_t xatom = 128 * 128, yatom = static_cast<uint32_t>(nmma) * 128;
  // py: Y is memory-paired too; otherwise Y keeps 8-byte stores and L keeps its
  // place in Y's stride order (register pairs for Y measured no gain on C1a
  // and cost Y's load coalescing on C1c)
  auto assign = [&](bool px, bool py, GtParams& q) -> int {
    const int ymode = py ? 1 : 2;
    std::vector<int> row_of(n_legs, -1), k_of(n_legs, -1), n_of(n_legs, -1);
    int L = xt[0];  // px: X's stride-1 leg
    if (!px) {      // the common tile leg with the largest X stride (an iteration bit already, as a rule)
      L = KL[0];
      for (int leg : KL)
        if (legs[leg].x_stride > legs[L].x_stride) L = leg;
    }
    std::vector<int> xl, yl;
    for (int leg : xt)
      if (leg != L) xl.push_back(leg);
    for (int leg : yt)
      if (leg != L || ymode == 2) yl.push_back(leg);
    const int xlanes = 3, ylanes = ymode == 2 ? 4 : 3;
    const int nxl = std::min<int>(xlanes, static_cast<int>(xl.size()));
    const int nyl = std::min<int>(ylanes, static_cast<int>(yl.size()));
    auto vec_row = [&](int j) { return j < 3 ? 1u << j : 0u; };
    auto vec_k = [&](int j) { return (j >= 1 && j <= 3) ? 1u << (j - 1) : 0u; };
    auto vec_n = [&](int j) { return j < 2 ? 1u << (j + 1) : 0u; };
    // unpaired Y: a half-warp's 8-byte stores, 8-byte slots (address bits 3-6)
    auto vec_k8 = [&](int j) { return j == 0 ? 1u : (j <= 3 ? (1u << j) : 0u); };
    auto vec_n8 = [&](int j) { return j < 2 ? (1u << (2 + j)) : 0u; };
    // smem store bytes per k-block
    const double sx = 16.0 * 128 * kbc, sy = 32.0 * (nmma / 2) * kbc;
    std::vector<int> lowR, lowN;  // low-order legs whose slots matter
    for (int i = 0; i < nxl; ++i)
      if (legs[xl[i]].kind == 0) lowR.push_back(xl[i]);
    for (int i = 0; i < nyl; ++i)
      if (legs[yl[i]].kind == 2) lowN.push_back(yl[i]);
    std::vector<int> kperm(KL.size());
    for (size_t i = 0; i < KL.size(); ++i) kperm[i] = static_cast<int>(i);
    double best_score = 1e300;
    std::vector<int> best_k, best_r, best_n;
    // candidate slots: rows 0..min(rb,3)-1 or "high" (-1); columns 0..min(fy,2)-1 or high
    auto enum_slots = [](int nlegs, int nslots, std::vector<std::vector<int>>& outv) {
      std::vector<int> cur(nlegs, -1);
      std::function<void(int, unsigned)> rec = [&](int i, unsigned used) {
        if (i == nlegs) {
          outv.push_back(cur);
          return;
        }
        cur[i] = -1;
        rec(i + 1, used);
        for (int s = 0; s < nslots; ++s)
          if (!((used >> s) & 1)) {
            cur[i] = s;
            rec(i + 1, used | (1u << s));
          }
      };
      rec(0, 0);
    };
    std::vector<std::vector<int>> r_opts, n_opts;
    enum_slots(static_cast<int>(lowR.size()), std::min(rb, 3), r_opts);
    enum_slots(static_cast<int>(lowN.size()), std::min(fy, 2), n_opts);
    do {
      for (size_t i = 0; i < KL.size(); ++i) k_of[KL[kperm[i]]] = static_cast<int>(i);
      if (k_of[L] != 0) continue;  // the pair leg sits on k bit 0
      double bx = 1e300, by = 1e300;
      std::vector<int> br, bn;
      for (auto& ro : r_opts) {
        uint32_t v[4];
        for (int i = 0; i < nxl; ++i) {
          const int leg = xl[i];
          if (legs[leg].kind == 1) {
            v[i] = vec_k(k_of[leg]);
          } else {
            const int sl = ro[std::find(lowR.begin(), lowR.end(), leg) - lowR.begin()];
            v[i] = sl < 0 ? 0u : vec_row(sl);
          }
        }
        const double sc = sx * conflict_ways(v, nxl);
        if (sc < bx) {
          bx = sc;
          br = ro;
        }
      }
      for (auto& no : n_opts) {
        uint32_t v[4];
        for (int i = 0; i < nyl; ++i) {
          const int leg = yl[i];
          if (legs[leg].kind == 1) {
            v[i] = ymode == 2 ? vec_k8(k_of[leg]) : vec_k(k_of[leg]);
          } else {
            const int sl = no[std::find(lowN.begin(), lowN.end(), leg) - lowN.begin()];
            v[i] = sl < 0 ? 0u : (ymode == 2 ? vec_n8(sl) : vec_n(sl));
          }
        }
        const double sc = sy * conflict_ways(v, nyl);
        if (sc < by) {
          by = sc;
          bn = no;
        }
      }
      if (bx + by < best_score) {
        best_score = bx + by;
        best_k.assign(KL.size(), 0);
        for (size_t i = 0; i < KL.size(); ++i) best_k[i] = kperm[i];
        best_r = br;
        best_n = bn;
      }
    } while (std::next_permutation(kperm.begin(), kperm.end()));
    for (size_t i = 0; i < KL.size(); ++i) k_of[KL[best_k[i]]] = static_cast<int>(i);
    if (std::getenv("TNC_GT_DEBUG"))
      std::fprintf(stderr, "tc_gather assign: nmma=%d kbc=%d px=%d ymode=%d store cost %.0f (conflict-free %.0f)\n", nmma,
                   kbc, px, ymode, best_score, sx + sy);
    {  // rows: searched low legs first, the rest by output stride (lane-adjacent writes)
      std::vector<char> used(7, 0);
      for (size_t i = 0; i < lowR.size(); ++i)
        if (best_r[i] >= 0) {
          row_of[lowR[i]] = best_r[i];
          used[best_r[i]] = 1;
        }
      std::vector<int> rest;
      for (int leg : R)
        if (row_of[leg] < 0) rest.push_back(leg);
      std::sort(rest.begin(), rest.end(), [&](int a, int b) { return legs[a].out_stride < legs[b].out_stride; });
      int slot = 0;
      for (int leg : rest) {
        while (used[slot]) ++slot;
        row_of[leg] = slot;
        used[slot] = 1;
      }
    }
    {  // columns
      std::vector<char> used(7, 0);
      for (size_t i = 0; i < lowN.size(); ++i)
        if (best_n[i] >= 0) {
          n_of[lowN[i]] = best_n[i];
          used[best_n[i]] = 1;
        }
      int slot = 0;
      for (int leg : yf)
        if (n_of[leg] < 0) {
          while (used[slot]) ++slot;
          n_of[leg] = slot;
          used[slot] = 1;
        }
    }
    // tile bit tables: real legs by stride, phantom bits above them; a
    // register pair leg goes to tile bit 8 (a memory pair leg is the 16-byte
    // element, not a bit)
    struct Bit {
      uint32_t g, s;
    };
    std::vector<Bit> xb, yb;
    uint64_t xsum = px ? 0 : static_cast<uint64_t>(legs[L].x_stride);
    uint64_t ysum = 0;
    for (int leg : xl) {
      xsum += static_cast<uint64_t>(legs[leg].x_stride);
      xb.push_back({static_cast<uint32_t>(legs[leg].x_stride),
                    legs[leg].kind == 0 ? row_bit_addr(row_of[leg]) : k_bit_addr(k_of[leg], xatom)});
    }
    for (int r = rb; r < 7; ++r) xb.push_back({0u, row_bit_addr(r)});  // phantom rows: re-read rows, never stored
    if (!px) xb.insert(xb.begin() + 8, {static_cast<uint32_t>(legs[L].x_stride), k_bit_addr(0, xatom)});
    for (int leg : yl) {
      ysum += static_cast<uint64_t>(legs[leg].y_stride);
      yb.push_back({static_cast<uint32_t>(legs[leg].y_stride),
                    legs[leg].kind == 2 ? row_bit_addr(n_of[leg] + 1) : k_bit_addr(k_of[leg], yatom)});
    }
    for (int n = fy; n < lgn; ++n) yb.push_back({0u, row_bit_addr(n + 1)});  // phantom columns
    if (xb.size() > static_cast<size_t>(kGtMaxBits) || yb.size() > static_cast<size_t>(kGtMaxBits))
      TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: too many tile bits");
    for (size_t j = 0; j < xb.size(); ++j) {
      q.xg[j] = xb[j].g;
      q.xs[j] = xb[j].s;
    }
    for (size_t j = 0; j < yb.size(); ++j) {
      q.yg[j] = yb[j].g;
      q.ys[j] = yb[j].s;
    }
    if (xsum + 1 >= (uint64_t{1} << 32) || ysum + 1 >= (uint64_t{1} << 32))
      TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: tile offsets exceed 32 bits");
    for (int leg : R) {
      q.orow[row_of[leg]] = legs[leg].out_stride;
      q.crow[row_of[leg]] = legs[leg].canon_stride;
    }
    for (int leg : yf) {
      q.ocol[n_of[leg]] = legs[leg].out_stride;
      q.ccol[n_of[leg]] = legs[leg].canon_stride;
    }
    return TNC_OK;
  };

  auto* plan = new GatherTcPlan();
  std::memset(&plan->p, 0, sizeof(plan->p));
  GtParams& p = plan->p;
  plan->nmma = nmma;
  plan->kbc = kbc;
  plan->occ = occ;
  plan->rows_x = int64_t{1} << fx;
  plan->rows_y = int64_t{1} << fy;
  plan->k = int64_t{1} << c;
  p.rbits = rb;
  p.fy = fy;
  if (const int st = assign(false, false, p); st != TNC_OK) {
    delete plan;
    return st;
  }
  p.m_blocks = int64_t{1} << (fx - rb);
  p.kblocks = int64_t{1} << (c - kb);
  p.mn = plan->rows_x * plan->rows_y;
  // outer tables
  plan->tabs_host.assign(static_cast<size_t>(kGtTabs) * 1024, 0);
  std::vector<int64_t> sxm, som, scm, sxk, syk;
  for (int i : outer_m) {
    sxm.push_back(legs[i].x_stride);
    som.push_back(legs[i].out_stride);
    scm.push_back(legs[i].canon_stride);
  }
  for (int i : outer_k) {
    sxk.push_back(legs[i].x_stride);
    syk.push_back(legs[i].y_stride);
  }
  build_tab4(sxm, plan->tabs_host.data() + 0 * 1024);
  build_tab4(som, plan->tabs_host.data() + 1 * 1024);
  build_tab4(scm, plan->tabs_host.data() + 2 * 1024);
  build_tab4(sxk, plan->tabs_host.data() + 3 * 1024);
  build_tab4(syk, plan->tabs_host.data() + 4 * 1024);
  // carry deltas: index i -> i + 1 turns bit b = ctz(i + 1) on, bits < b off
  auto carry_deltas = [](const std::vector<int64_t>& st, int64_t* out) {
    for (int b = 0; b < 32; ++b) {
      int64_t d = 0;
      for (int i = 0; i <= b && i < static_cast<int>(st.size()); ++i) d += i == b ? st[i] : -st[i];
      out[b] = d;
    }
  };
  carry_deltas(sxk, p.dxk);
  carry_deltas(syk, p.dyk);
  carry_deltas(sxm, p.dxm);
  carry_deltas(som, p.dom);
  carry_deltas(scm, p.dcm);
  // k-splits: enough units for every SM, each SM's share within ~3% of the others
  const int sms = num_sms() * occ;
  int splits = 1;
  if (p.m_blocks < 4 * sms) {
    double best_eff = 0;
    const int64_t smax = std::min<int64_t>(p.kblocks, 4096);
    for (int64_t s = 1; s <= smax; ++s) {
      const int64_t units = p.m_blocks * s;
      const double e = static_cast<double>(units) / (ceil_div(units, sms) * sms);
      if (e > best_eff + 1e-9) {
        best_eff = e;
        splits = static_cast<int>(s);
      }
      if (units >= sms && e >= 0.97) break;
    }
  }
  if (const char* env = std::getenv("TNC_GT_SPLITS")) {
    const int64_t forced = std::atoll(env);
    if (forced >= 1) splits = static_cast<int>(std::min<int64_t>(forced, p.kblocks));
  }
  p.splits = splits;
  p.chunk_kb = std::max(1, 128 / kbc);  // 128 complex K per TMEM chain (as K2)
  if (const char* env = std::getenv("TNC_GT_CHUNK")) p.chunk_kb = std::max(1, std::atoi(env));
  // paired layout: X's stride-1 leg is a tile common leg (it goes to k bit 0);
  // Y pairs too when that leg is also Y's stride-1 leg.  Used at launch when
  // the operand pointers are 16-byte aligned.
  const bool px = legs[xt[0]].kind == 1 && legs[xt[0]].x_stride == 1;
  // (not for 256-column tiles: the paired Y registers spill there, measured slower)
  const bool py = px && nmma <= 128 && occ == 1 && yt[0] == xt[0] && legs[yt[0]].y_stride == 1;
  const char* pair_env = std::getenv("TNC_GT_PAIR");
  if (px && !(pair_env && std::atoi(pair_env) == 0)) {
    plan->p2 = p;
    if (assign(true, py, plan->p2) == TNC_OK) {
      plan->pair_x = true;
      plan->pair_y = py;
    }
  }
  const int up = upload_table(plan->tabs_host.data(), plan->tabs_host.size(), &plan->tabs_dev);
  if (up != TNC_OK) {
    delete plan;
    return up;
  }
  *out = plan;
  return TNC_OK;
}

int gather_tc_splits(const GatherTcPlan* plan) { return plan->p.splits; }

void gather_tc_destroy(GatherTcPlan* plan) { delete plan; }

namespace {

template <int NMMA, int KBC, int STAGES, bool PX, bool PY, int OCC, bool MW = false>
int launch_gt(const GtParams& p, int64_t units, double flops, double bytes, cudaStream_t stream) {
  using Cfg = GtCfg<NMMA, KBC, STAGES, PX, PY>;
  auto kern = gather_tc_kernel<NMMA, KBC, STAGES, PX, PY, OCC, MW>;
  TNC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
  const int grid = static_cast<int>(std::min<int64_t>(units, static_cast<int64_t>(num_sms()) * OCC));
  ProfScope prof(PROF_TC_GATHER, flops, bytes, stream);
  kern<<<grid, MW ? kGtThreads + 128 : kGtThreads, Cfg::kSmem, stream>>>(p);
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

}  // namespace

int gather_tc_launch(const GatherTcPlan* plan, const void* x, const void* y, void* c_final, void* parts,
                     cudaStream_t stream) {
  if (!plan->tabs_dev && !plan->tabs_host.empty()) TNC_RET(TNC_ERR_INVALID, "tc_gather: plan tables missing");
  // paired layout when the plan has one and the operands are 16-byte aligned
  const bool aligned = (reinterpret_cast<uintptr_t>(x) & 15) == 0 &&
                       (!plan->pair_y || (reinterpret_cast<uintptr_t>(y) & 15) == 0);
  const bool px = plan->pair_x && aligned, py = px && plan->pair_y;
  GtParams p = px ? plan->p2 : plan->p;
  p.X = static_cast<const float2*>(x);
  p.Y = static_cast<const float2*>(y);
  p.C = static_cast<float2*>(c_final);
  p.parts = static_cast<float2*>(parts);
  p.tabs = plan->tabs_dev;
  if (p.splits == 1 && !p.C) TNC_RET(TNC_ERR_INVALID, "tc_gather: null output");
  if (p.splits > 1 && !p.parts) TNC_RET(TNC_ERR_INVALID, "tc_gather: null partials");
  const int64_t units = p.m_blocks * p.splits;
  const double M = static_cast<double>(plan->rows_x), N = static_cast<double>(plan->rows_y),
               K = static_cast<double>(plan->k);
  const double flops = 8.0 * M * N * K, bytes = 8.0 * (M * K + N * K + M * N);
#define TNC_GT_MODES(N, KBC, ST)                                                           \
  do {                                                                                     \
    if (py) return launch_gt<N, KBC, ST, true, true, 1>(p, units, flops, bytes, stream);   \
    if (px) return launch_gt<N, KBC, ST, true, false, 1>(p, units, flops, bytes, stream);  \
    return launch_gt<N, KBC, ST, false, false, 1>(p, units, flops, bytes, stream);         \
  } while (0)
  switch (plan->nmma) {
    case 32:
      if (plan->occ == 2) {  // (a memory-paired Y would leave fewer Y elements than threads)
        if (px) return launch_gt<32, 16, 2, true, false, 2>(p, units, flops, bytes, stream);
        return launch_gt<32, 16, 2, false, false, 2>(p, units, flops, bytes, stream);
      }
      TNC_GT_MODES(32, 32, 2);
    case 64: TNC_GT_MODES(64, 32, 2);
    case 128: TNC_GT_MODES(128, 16, 3);
    case 256: {
      const char* mw_s = std::getenv("TNC_GT_MMAWARP");
      if (!(mw_s && std::atoi(mw_s) == 0)) {
        if (px) return launch_gt<256, 16, 2, true, false, 1, true>(p, units, flops, bytes, stream);
        return launch_gt<256, 16, 2, false, false, 1, true>(p, units, flops, bytes, stream);
      }
      if (px) return launch_gt<256, 16, 2, true, false, 1>(p, units, flops, bytes, stream);
      return launch_gt<256, 16, 2, false, false, 1>(p, units, flops, bytes, stream);
    }
    default: TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: bad tile width");
  }
#undef TNC_GT_MODES
}

}  // namespace tnc
