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
//   accuracy = chunks of 32 complex K accumulate in alternating TMEM buffers
//              and are folded into fp32 registers (same scheme as K2)
//   output   = one split: C written in its FINAL (caller's) leg order; more
//              splits: fp32 partials [split][row][col] (canonical order),
//              then the fixed-order tree reduction
//
// Roles (256 threads, 8 warps = 2 per SM sub-partition so each thread can
// hold up to 255 registers): every warp gathers + splits (loads run one
// k-block ahead of the smem stores), folds TMEM lane quadrant w % 4, column
// half w / 4, and stores; warp 0 also owns TMEM and issues the MMAs of
// k-block g-1 right after staging k-block g (one elected lane).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <mutex>
#include <vector>

#include "tnc_common.cuh"
#include "tnc_gather_tc.cuh"
#include "tnc_tcgen05.cuh"

namespace tnc {

namespace {

using namespace tc5;

constexpr int kGtWorkers = 256;
constexpr int kGtWorkerWarps = kGtWorkers / 32;
constexpr int kGtThreads = kGtWorkers;  // warp 0 also issues the MMAs
constexpr int kGtMaxBits = 12;          // tile bits per operand (7 rows + 4 k; 6 cols + 4 k)
constexpr int kGtTabs = 5;              // outer tables: xm, om, cm (m-block), xk, yk (k-block)
constexpr int kGtKbc = 16;              // complex K per k-block: one 128-byte TF32 atom

struct GtParams {
  const float2* X;
  const float2* Y;
  float2* C;            // final output (splits == 1)
  float2* parts;        // [splits][rows_x * rows_y] canonical order (splits > 1)
  const int64_t* tabs;  // [kGtTabs][4][256] outer-index offset tables
  int64_t m_blocks, kblocks, mn;
  int splits, chunk_kb, depth;
  int nblocks;          // 1, or 2 when Y has 128 columns (one Y-free leg outside the tile)
  int64_t y_nb, o_nb, c_nb;  // offsets of column block 1 in Y / the output / the partials
  int rbits, fy;        // real row / column bits of the tile (phantom bits, stride 0, above)
  // tile bit j (thread bit j for j < 8, element-slot bit j - 8 above): element
  // offset in the operand and XOR-linear smem byte address in the stage plane
  uint32_t xg[kGtMaxBits], xs[kGtMaxBits];
  uint32_t yg[kGtMaxBits], ys[kGtMaxBits];
  int64_t orow[7], crow[7];  // per tile-row bit: final / partial-layout stride
  int64_t ocol[7], ccol[7];  // per column bit
  // outer k-block index kb -> kb + 1 flips bit b = ctz(kb + 1) on and the bits
  // below it off: X / Y offsets move by these carry deltas
  int64_t dxk[32], dyk[32];
};

template <int NMMA, int STAGES>
struct GtCfg {
  static constexpr int kLogN = NMMA == 32 ? 4 : NMMA == 64 ? 5 : 6;  // log2(NMMA / 2)
  static constexpr int kXBits = 7 + 4;
  static constexpr int kYBits = kLogN + 4;
  static constexpr int kXPer = 1 << (kXBits - 8);  // X elements per thread per k-block
  static constexpr int kYPer = 1 << (kYBits - 8);
  static constexpr int kXPlane = 128 * 128;         // one 128-row atom of TF32
  static constexpr int kYPlane = NMMA * 128;
  static constexpr int kStage = 2 * kXPlane + 2 * kYPlane;
  static constexpr int kSmem = STAGES * kStage + 1024;
  static constexpr int kHalf = NMMA / 2;
  static constexpr uint32_t kIdesc = idesc_f32acc(2, 128, NMMA);
  static_assert(kSmem + 4096 <= 227 * 1024, "smem budget");
  static_assert(kYBits >= 8, "Y tile smaller than the CTA");
  static_assert((NMMA / 2) * kGtKbc * 8 <= kXPlane, "raw Y tile must fit the X small plane");
};

__device__ __forceinline__ int64_t tab4(const int64_t* t, int64_t idx) {
  return __ldg(t + (idx & 255)) + __ldg(t + 256 + ((idx >> 8) & 255)) +
         __ldg(t + 512 + ((idx >> 16) & 255)) + __ldg(t + 768 + ((idx >> 24) & 255));
}

__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

// arrive on `bar` once every cp.async this thread issued so far has landed
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ float2 lds2(uint32_t a) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
  return v;
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}

__device__ __forceinline__ void sts2(uint32_t addr, float a, float b) {
  asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(addr), "f"(a), "f"(b) : "memory");
}

__device__ __forceinline__ void sts4(uint32_t addr, float a, float b, float c, float d) {
  asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "f"(a), "f"(b), "f"(c), "f"(d)
               : "memory");
}

// TF32 "big" part, round-half-away on the 13 dropped mantissa bits
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}

// x minus its TF32 truncation: the tensor core reads an fp32 operand as its
// top 19 bits, so a raw fp32 plane is the "big" part and this is the "small"
__device__ __forceinline__ float tf32_rem(float x) {
  return x - __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
}

__device__ __forceinline__ void split_range(const GtParams& p, int split, int64_t& lo, int64_t& hi) {
  if (p.splits == 1) {
    lo = 0;
    hi = p.kblocks;
  } else {
    lo = p.kblocks * split / p.splits;
    hi = p.kblocks * (split + 1) / p.splits;
  }
}

// Unit / k-block cursor over this CTA's share of the (m-block, column block,
// split) units; the unit's decomposition is computed once when it is opened
// (32-bit divisions), never per k-block.
struct GtCursor {
  uint32_t u, units;
  uint32_t mb, split;
  bool nb1;
  int64_t kb, kb_hi;
  __device__ __forceinline__ bool valid() const { return u < units; }
  __device__ __forceinline__ void open(const GtParams& p) {
    if (u >= units) return;
    const uint32_t splits = static_cast<uint32_t>(p.splits);
    const uint32_t rest = splits == 1 ? u : u / splits;
    split = u - rest * splits;
    if (p.nblocks == 1) {
      mb = rest;
      nb1 = false;
    } else {
      mb = rest >> 1;
      nb1 = rest & 1;
    }
    split_range(p, static_cast<int>(split), kb, kb_hi);
  }
  __device__ __forceinline__ void init(const GtParams& p, uint32_t n_units) {
    u = blockIdx.x;
    units = n_units;
    open(p);
  }
  // advance one k-block; true when the cursor entered a new unit
  __device__ __forceinline__ bool next(const GtParams& p) {
    if (++kb < kb_hi) return false;
    u += gridDim.x;
    open(p);
    return true;
  }
};

template <int NMMA, int STAGES>
__global__ void __launch_bounds__(kGtThreads, 1) gather_tc_kernel(const __grid_constant__ GtParams p) {
  using Cfg = GtCfg<NMMA, STAGES>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  __shared__ uint64_t landed[STAGES], full[STAGES], empty[STAGES], tfull[2], tempty[2];
  __shared__ uint32_t tmem_slot;
  __shared__ uint32_t xhi_g[16], xhi_s[16], yhi_g[16], yhi_s[16];
  __shared__ int64_t ocol_t[64], ccol_t[64], dxk[32], dyk[32];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int t = threadIdx.x;
  const uint32_t units = static_cast<uint32_t>(p.m_blocks * p.nblocks * p.splits);

  if (t == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&landed[s], kGtWorkers);
      mbar_init(&full[s], kGtWorkers);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tfull[b], 1);
      mbar_init(&tempty[b], kGtWorkerWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (t < 16) {
    uint32_t g = 0, s = 0, h = 0, q = 0;
    for (int j = 8; j < Cfg::kXBits; ++j)
      if ((t >> (j - 8)) & 1) {
        g += p.xg[j];
        s ^= p.xs[j];
      }
    for (int j = 8; j < Cfg::kYBits; ++j)
      if ((t >> (j - 8)) & 1) {
        h += p.yg[j];
        q ^= p.ys[j];
      }
    xhi_g[t] = g;
    xhi_s[t] = s;
    yhi_g[t] = h;
    yhi_s[t] = q;
  }
  if (t < 32) {
    dxk[t] = p.dxk[t];
    dyk[t] = p.dyk[t];
  }
  if (t < 64) {
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
  // this thread's tile elements: operand offsets and smem byte addresses
  uint32_t xo[Cfg::kXPer], xa[Cfg::kXPer], yo[Cfg::kYPer], ya[Cfg::kYPer];
#pragma unroll
  for (int i = 0; i < Cfg::kXPer; ++i) {
    xo[i] = xg_lo + xhi_g[i];
    xa[i] = xs_lo ^ xhi_s[i];
  }
#pragma unroll
  for (int i = 0; i < Cfg::kYPer; ++i) {
    yo[i] = yg_lo + yhi_g[i];
    ya[i] = ys_lo ^ yhi_s[i];
  }

  float acc[Cfg::kHalf];
#pragma unroll
  for (int j = 0; j < Cfg::kHalf; ++j) acc[j] = 0.f;

  GtCursor pc;  // loads (depth k-blocks ahead)
  pc.init(p, units);
  // operand offsets of the load cursor's k-block: unit part + k-block part
  int64_t xm_off = 0, xk_off = 0, yk_off = 0;
  auto open_offsets = [&]() {
    if (!pc.valid()) return;
    xm_off = tab4(p.tabs, pc.mb);
    xk_off = tab4(p.tabs + 3 * 1024, pc.kb);
    yk_off = tab4(p.tabs + 4 * 1024, pc.kb) + (pc.nb1 ? p.y_nb : 0);
  };
  open_offsets();
  GtCursor ic;  // MMA issue (warp 0)
  ic.init(p, units);
  int i_in_chunk = 0;
  uint32_t i_ch = 0;
  GtCursor fc;  // fold: this CTA's chunk sequence
  fc.init(p, units);
  int64_t f_n = fc.valid() ? fc.kb_hi - fc.kb : 0;
  int f_c = 0, f_nch = static_cast<int>((f_n + p.chunk_kb - 1) / p.chunk_kb);
  uint32_t f_base = 0, ch = 0;

  // X tile: cp.async straight into the swizzled "big" plane of the stage.
  // Raw Y tile: cp.async into the (still unused) "small" X plane, in a
  // thread-linear layout; the conversion pass expands it into Y^.
  uint32_t loaded = 0;
  auto issue_loads = [&]() {
    const uint32_t s = loaded % STAGES;
    mbar_wait(&empty[s], ((loaded / STAGES) & 1) ^ 1);
    const uint32_t st = smem0 + s * Cfg::kStage;
    const float2* xb = p.X + (xm_off + xk_off);
    const float2* yb = p.Y + yk_off;
#pragma unroll
    for (int i = 0; i < Cfg::kXPer; ++i) cp_async8(st + xa[i], xb + xo[i]);
#pragma unroll
    for (int i = 0; i < Cfg::kYPer; ++i) cp_async8(st + Cfg::kXPlane + (i * kGtWorkers + t) * 8, yb + yo[i]);
    cp_async_arrive(&landed[s]);
    ++loaded;
    const int b = __ffsll(pc.kb + 1) - 1;  // carry bit of kb -> kb + 1
    if (pc.next(p)) {
      open_offsets();
    } else {
      xk_off += dxk[b];
      yk_off += dyk[b];
    }
  };
  for (int d = 0; d < p.depth && pc.valid(); ++d) issue_loads();

  // Iteration j:
  //   1. issue the loads of k-block j + depth (its stage is free once MMA
  //      j + depth - STAGES is done: depth <= STAGES - 1)
  //   2. fold the TMEM chunks ending at or before j - 2 (MMA j - 1 is queued
  //      behind them); once k-blocks run out, fold everything
  //   3. convert k-block j: Y raw -> Y^ big/small, X big -> X small
  //   4. warp 0 issues the 12 MMAs of k-block j
  // A chunk's TMEM buffer is folded (step 2) at least an iteration before the
  // MMAs that reuse it are issued (step 4): no step waits on a later one.
  for (uint32_t j = 0;; ++j) {
    if (pc.valid()) issue_loads();
    const bool more = j < loaded;
    while (fc.valid()) {
      const int64_t end = static_cast<int64_t>(f_c + 1) * p.chunk_kb;
      const int64_t last = static_cast<int64_t>(f_base) + (end < f_n ? end : f_n) - 1;
      if (more && last + 2 > static_cast<int64_t>(j)) break;
      const uint32_t b = ch & 1;
      mbar_wait(&tfull[b], (ch >> 1) & 1);
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
          for (int q = 0; q < 16; ++q) acc[gi * 16 + q] = __uint_as_float(v[q]);
        } else {
#pragma unroll
          for (int q = 0; q < 16; ++q) acc[gi * 16 + q] += __uint_as_float(v[q]);
        }
      }
      fence_before_sync();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
      ++ch;
      if (f_c == f_nch - 1) {
        // unit finished: store this thread's row (one TMEM lane), its column half
        const int r = quad * 32 + lane;
        const uint32_t mb = fc.mb, split = fc.split;
        const bool nb1 = fc.nb1;
        if (r < (1 << p.rbits)) {
          const int n0 = half * (Cfg::kHalf / 2);
          const int ncols = min(Cfg::kHalf / 2, (1 << p.fy) - n0);
          if (p.splits == 1) {
            int64_t base = tab4(p.tabs + 1 * 1024, mb) + (nb1 ? p.o_nb : 0);
            for (int q = 0; q < p.rbits; ++q)
              if ((r >> q) & 1) base += p.orow[q];
#pragma unroll
            for (int q = 0; q < Cfg::kHalf / 2; ++q)
              if (q < ncols) p.C[base + ocol_t[n0 + q]] = make_float2(acc[2 * q], acc[2 * q + 1]);
          } else {
            int64_t base = static_cast<int64_t>(split) * p.mn + tab4(p.tabs + 2 * 1024, mb) + (nb1 ? p.c_nb : 0);
            for (int q = 0; q < p.rbits; ++q)
              if ((r >> q) & 1) base += p.crow[q];
#pragma unroll
            for (int q = 0; q < Cfg::kHalf / 2; ++q)
              if (q < ncols) p.parts[base + ccol_t[n0 + q]] = make_float2(acc[2 * q], acc[2 * q + 1]);
          }
        }
        f_base += static_cast<uint32_t>(f_n);
        fc.u += gridDim.x;
        fc.open(p);
        f_c = 0;
        if (fc.valid()) {
          f_n = fc.kb_hi - fc.kb;
          f_nch = static_cast<int>((f_n + p.chunk_kb - 1) / p.chunk_kb);
        }
      } else {
        ++f_c;
      }
    }
    if (!more) break;

    const uint32_t s = j % STAGES;
    const uint32_t st = smem0 + s * Cfg::kStage;
    mbar_wait(&landed[s], (j / STAGES) & 1);
#pragma unroll
    for (int i = 0; i < Cfg::kYPer; ++i) {
      const float2 y = lds2(st + Cfg::kXPlane + (i * kGtWorkers + t) * 8);
      const uint32_t a0 = st + 2 * Cfg::kXPlane + ya[i];
      const uint32_t a1 = a0 ^ 0x90u;  // row 2n+1 (row bit 0 and its swizzle bit)
      const float hr = tf32_hi(y.x), hi = tf32_hi(y.y);
      const float lr = y.x - hr, li = y.y - hi;
      sts2(a0, hr, -hi);
      sts2(a1, hi, hr);
      sts2(a0 + Cfg::kYPlane, lr, -li);
      sts2(a1 + Cfg::kYPlane, li, lr);
    }
    asm volatile("bar.sync 1, 256;" ::: "memory");  // raw Y read before X small overwrites it
#pragma unroll
    for (int c = 0; c < Cfg::kXPlane / (16 * kGtWorkers); ++c) {
      const uint32_t a = st + (c * kGtWorkers + t) * 16;
      const float4 v = lds4(a);
      sts4(a + Cfg::kXPlane, tf32_rem(v.x), tf32_rem(v.y), tf32_rem(v.z), tf32_rem(v.w));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_arrive(&full[s]);

    if (warp == 0) {
      if (i_in_chunk == 0) {
        const uint32_t b = i_ch & 1;
        mbar_wait_spin(&tempty[b], ((i_ch >> 1) & 1) ^ 1);
        fence_after_sync();
      }
      const uint32_t dcol = tmem_base + (i_ch & 1) * NMMA;
      mbar_wait_spin(&full[s], (j / STAGES) & 1);
      fence_after_sync();
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t xs = st + kk * 32;
        const uint32_t ys = st + 2 * Cfg::kXPlane + kk * 32;
        const uint64_t x_big = umma_desc_sw128(xs);
        const uint64_t x_small = umma_desc_sw128(xs + Cfg::kXPlane);
        const uint64_t y_big = umma_desc_sw128(ys);
        const uint64_t y_small = umma_desc_sw128(ys + Cfg::kYPlane);
        const uint32_t acc0 = (i_in_chunk > 0 || kk > 0) ? 1u : 0u;
        // small products first: accumulated before the big one
        mma_tf32_elect(dcol, x_small, y_big, Cfg::kIdesc, acc0);
        mma_tf32_elect(dcol, x_big, y_small, Cfg::kIdesc, 1u);
        mma_tf32_elect(dcol, x_big, y_big, Cfg::kIdesc, 1u);
      }
      mma_commit_elect(&empty[s]);
      const bool unit_end = ic.kb + 1 == ic.kb_hi;
      if (++i_in_chunk == p.chunk_kb || unit_end) {
        mma_commit_elect(&tfull[i_ch & 1]);
        ++i_ch;
        i_in_chunk = 0;
      }
      ic.next(p);
    }
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
  int nmma = 0, kbc = 0, stages = 0;
  int64_t rows_x = 0, rows_y = 0, k = 0;
  std::vector<int64_t> tabs_host;
  mutable std::mutex mu;
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
  const int fx = static_cast<int>(xf.size()), c = static_cast<int>(cm.size());
  if (yf.size() > 7) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: Y has more than 128 columns");
  if (fx < 6) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: X has fewer than 64 rows");
  // 128 Y columns: the slowest Y-free leg selects one of two 64-column blocks
  int nb_leg = -1;
  if (yf.size() == 7) {
    auto it = std::max_element(yf.begin(), yf.end(),
                               [&](int a, int b) { return legs[a].y_stride < legs[b].y_stride; });
    nb_leg = *it;
    yf.erase(it);
  }
  const int fy = static_cast<int>(yf.size());
  const int nmma = std::max(32, 2 << fy);
  const int lgn = nmma == 32 ? 4 : nmma == 64 ? 5 : 6;  // log2(nmma / 2)
  const int kbc = kGtKbc;
  const int kb = 4;
  if (c < kb) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: K smaller than one k-block");
  const int rb = std::min(7, fx);
  if (fx - rb > 32 || c - kb > 32) TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: outer index > 32 bits");

  // ---- which legs form the tile: greedy on the access efficiency of X
  // reads, Y reads and output writes, weighted by their bytes
  const double rows_x = std::ldexp(1.0, fx), rows_y = std::ldexp(1.0, fy + (nb_leg >= 0)), kk = std::ldexp(1.0, c);
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
  // bits.  A half-warp's 8-byte smem stores hit 16 distinct 8-byte slots iff
  // the bank vectors of the operand's 4 fastest tile legs (thread bits 0-3)
  // are independent; search the assignments that decide those vectors.
  std::vector<int> row_of(n_legs, -1), k_of(n_legs, -1), n_of(n_legs, -1);
  const int nxl = std::min<int>(4, static_cast<int>(xt.size())), nyl = std::min<int>(4, static_cast<int>(yt.size()));
  auto vec_row = [](int j) { return j < 3 ? (1u << (1 + j)) : 0u; };
  auto vec_k = [](int j) { return j == 0 ? 1u : (j <= 3 ? (1u << j) : 0u); };
  auto vec_n = [](int j) { return j < 2 ? (1u << (2 + j)) : 0u; };
  const double sx = 2.0 * 128 * kbc, sy = 4.0 * (nmma / 2) * kbc;  // smem store instructions
  std::vector<int> lowR, lowN;  // low-order legs whose slots matter
  for (int i = 0; i < nxl; ++i)
    if (legs[xt[i]].kind == 0) lowR.push_back(xt[i]);
  for (int i = 0; i < nyl; ++i)
    if (legs[yt[i]].kind == 2) lowN.push_back(yt[i]);
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
    double bx = 1e300, by = 1e300;
    std::vector<int> br, bn;
    for (auto& ro : r_opts) {
      uint32_t v[4];
      for (int i = 0; i < nxl; ++i) {
        const int leg = xt[i];
        if (legs[leg].kind == 1) {
          v[i] = vec_k(k_of[leg]);
        } else {
          const int s = ro[std::find(lowR.begin(), lowR.end(), leg) - lowR.begin()];
          v[i] = s < 0 ? 0u : vec_row(s);
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
        const int leg = yt[i];
        if (legs[leg].kind == 1) {
          v[i] = vec_k(k_of[leg]);
        } else {
          const int s = no[std::find(lowN.begin(), lowN.end(), leg) - lowN.begin()];
          v[i] = s < 0 ? 0u : vec_n(s);
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

  auto* plan = new GatherTcPlan();
  std::memset(&plan->p, 0, sizeof(plan->p));
  GtParams& p = plan->p;
  plan->nmma = nmma;
  plan->kbc = kbc;
  plan->rows_x = int64_t{1} << fx;
  plan->rows_y = int64_t{1} << (fy + (nb_leg >= 0));
  plan->k = int64_t{1} << c;
  p.rbits = rb;
  p.fy = fy;
  const uint32_t xatom = 128 * 128, yatom = static_cast<uint32_t>(nmma) * 128;
  uint64_t xsum = 0, ysum = 0;
  int j = 0;
  for (int leg : xt) {
    xsum += static_cast<uint64_t>(legs[leg].x_stride);
    p.xg[j] = static_cast<uint32_t>(legs[leg].x_stride);
    p.xs[j++] = legs[leg].kind == 0 ? row_bit_addr(row_of[leg]) : k_bit_addr(k_of[leg], xatom);
  }
  for (int r = rb; r < 7; ++r) {  // phantom rows: re-read rows, never stored
    p.xg[j] = 0;
    p.xs[j++] = row_bit_addr(r);
  }
  j = 0;
  for (int leg : yt) {
    ysum += static_cast<uint64_t>(legs[leg].y_stride);
    p.yg[j] = static_cast<uint32_t>(legs[leg].y_stride);
    p.ys[j++] = legs[leg].kind == 2 ? row_bit_addr(n_of[leg] + 1) : k_bit_addr(k_of[leg], yatom);
  }
  for (int n = fy; n < lgn; ++n) {  // phantom columns
    p.yg[j] = 0;
    p.ys[j++] = row_bit_addr(n + 1);
  }
  if (xsum >= (uint64_t{1} << 32) || ysum >= (uint64_t{1} << 32)) {
    delete plan;
    TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: tile offsets exceed 32 bits");
  }
  for (int leg : R) {
    p.orow[row_of[leg]] = legs[leg].out_stride;
    p.crow[row_of[leg]] = legs[leg].canon_stride;
  }
  for (int leg : yf) {
    p.ocol[n_of[leg]] = legs[leg].out_stride;
    p.ccol[n_of[leg]] = legs[leg].canon_stride;
  }
  p.m_blocks = int64_t{1} << (fx - rb);
  p.nblocks = nb_leg >= 0 ? 2 : 1;
  if (nb_leg >= 0) {
    p.y_nb = legs[nb_leg].y_stride;
    p.o_nb = legs[nb_leg].out_stride;
    p.c_nb = legs[nb_leg].canon_stride;
  }
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
  for (int b = 0; b < 32; ++b) {
    int64_t dx = 0, dy = 0;
    for (int i = 0; i <= b && i < static_cast<int>(sxk.size()); ++i) {
      dx += i == b ? sxk[i] : -sxk[i];
      dy += i == b ? syk[i] : -syk[i];
    }
    p.dxk[b] = dx;
    p.dyk[b] = dy;
  }
  // k-splits: enough units for every SM, each SM's share within ~3% of the others
  const int sms = num_sms();
  int splits = 1;
  if (p.m_blocks * p.nblocks < 4 * sms) {
    double best_eff = 0;
    const int64_t smax = std::min<int64_t>(p.kblocks, 4096);
    for (int64_t s = 1; s <= smax; ++s) {
      const int64_t units = p.m_blocks * p.nblocks * s;
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
  p.chunk_kb = std::max(1, 32 / kbc);
  if (const char* env = std::getenv("TNC_GT_CHUNK")) p.chunk_kb = std::max(1, std::atoi(env));
  // loads in flight: every free stage for narrow tiles (short MMAs); one
  // stage kept back for 64-column tiles so a load never waits on the MMA
  // just issued
  plan->stages = nmma == 32 ? 5 : nmma == 64 ? 4 : 3;
  p.depth = plan->stages - 2;
  if (const char* env = std::getenv("TNC_GT_DEPTH"))
    p.depth = std::max(1, std::min(plan->stages - 1, std::atoi(env)));
  *out = plan;
  return TNC_OK;
}

int gather_tc_splits(const GatherTcPlan* plan) { return plan->p.splits; }

void gather_tc_destroy(GatherTcPlan* plan) { delete plan; }

namespace {

template <int NMMA, int STAGES>
int launch_gt(const GtParams& p, int64_t units, double flops, double bytes, cudaStream_t stream) {
  using Cfg = GtCfg<NMMA, STAGES>;
  auto kern = gather_tc_kernel<NMMA, STAGES>;
  TNC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmem));
  const int grid = static_cast<int>(std::min<int64_t>(units, num_sms()));
  ProfScope prof(PROF_TC_GATHER, flops, bytes, stream);
  kern<<<grid, kGtThreads, Cfg::kSmem, stream>>>(p);
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

}  // namespace

int gather_tc_launch(const GatherTcPlan* plan, const void* x, const void* y, void* c_final, void* parts,
                     cudaStream_t stream) {
  {
    std::lock_guard<std::mutex> lk(plan->mu);
    if (!plan->tabs_dev) {
      const size_t bytes = plan->tabs_host.size() * sizeof(int64_t);
      TNC_CUDA_TRY(cudaMalloc(&plan->tabs_dev, bytes));
      TNC_CUDA_TRY(cudaMemcpy(plan->tabs_dev, plan->tabs_host.data(), bytes, cudaMemcpyHostToDevice));
    }
  }
  GtParams p = plan->p;
  p.X = static_cast<const float2*>(x);
  p.Y = static_cast<const float2*>(y);
  p.C = static_cast<float2*>(c_final);
  p.parts = static_cast<float2*>(parts);
  p.tabs = plan->tabs_dev;
  if (p.splits == 1 && !p.C) TNC_RET(TNC_ERR_INVALID, "tc_gather: null output");
  if (p.splits > 1 && !p.parts) TNC_RET(TNC_ERR_INVALID, "tc_gather: null partials");
  const int64_t units = p.m_blocks * p.nblocks * p.splits;
  const double M = static_cast<double>(plan->rows_x), N = static_cast<double>(plan->rows_y),
               K = static_cast<double>(plan->k);
  const double flops = 8.0 * M * N * K, bytes = 8.0 * (M * K + N * K + M * N);
  switch (plan->nmma) {
    case 32: return launch_gt<32, 5>(p, units, flops, bytes, stream);
    case 64: return launch_gt<64, 4>(p, units, flops, bytes, stream);
    case 128: return launch_gt<128, 3>(p, units, flops, bytes, stream);
    default: TNC_RET(TNC_ERR_UNSUPPORTED, "tc_gather: bad tile width");
  }
}

}  // namespace tnc
