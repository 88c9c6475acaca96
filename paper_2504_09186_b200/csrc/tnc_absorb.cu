// K4: step fusion -- a chain of two-leg gate absorptions into one resident
// tensor, with the gate math on tensor cores, in the fewest HBM passes.
//
// Reference semantics: successive contract_pair(T, G) along a stem
// (execute.py:137-178 over tree.py:278-384 stems; contract.py:149-165):
// gate g = (out_a, out_b, in_a, in_b) contracts T's legs at logical
// positions axes[2g] (in_a) and axes[2g+1] (in_b); the two legs leave the
// order and (out_a, out_b) are appended at the end.
//
// B200 design.
//  * Physical axes.  Data never moves between gates: out_a lands on in_a's
//    physical axis, so the chain is "apply 4x4 unitaries on axis pairs", then
//    write the final logical order.
//  * Passes.  A pass streams the tensor HBM -> smem tile (2^13 complex64 =
//    64 KB, 13 tile axes) -> gates on tile axes -> HBM.  The host packs gates
//    into passes greedily in dependency order (gates on disjoint axes commute,
//    so a gate that does not fit is deferred together with every later gate on
//    its axes).  Between passes the intermediate layout is free: its 3 fastest
//    axes ("link") are tile axes of both passes (coalesced writes and reads)
//    and the next pass's tile axes come next (its reads are contiguous runs).
//    C2 (16 random gates on a rank-30 tensor): 2 passes (was 3 with 12-bit
//    tiles and in-order sections).
//  * Math.  Within a pass the gates are grouped on 3 tile axes and multiplied
//    into one 8x8 complex unitary per group (device kernel, double, no host
//    round trip for the gate values).  A group is applied to the tile as the
//    real GEMM  [1024 rows x 16] x [16 x 16]  on mma.sync.m16n8k16 (fp16 in,
//    fp32 accumulate) with a 3-product split: each 8-element row is scaled by
//    a power of two to the top of the fp16 range (f16_row_exponent), split
//    into hi + lo halves, and  lo*U_hi + hi*U_lo + hi*U_hi  are accumulated,
//    then the row scale is undone.  The A fragment of a thread is 4 complex
//    elements (rows g, g+8 x cols q, q+4) and its D fragment is the same 4
//    positions, so every group is an in-place smem read-modify-write: 16 B of
//    smem traffic and 192 tensor flops per element per group (vs 64 FP32 FMA
//    per element for the same 3 gates on CUDA cores).
//  * Banks.  8-byte smem slots are XOR-swizzled (swz); a tile bit's bank class
//    is (bit mod 4).  The host places tile axes so that the 4 fastest load
//    axes, the 4 fastest store axes, and each group's lane bits (2 column +
//    2 row bits) cover 4 distinct classes: every half-warp access is
//    conflict-free.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tnc_common.cuh"
#include "tnc_tcgen05.cuh"

namespace tnc {

namespace {

using namespace tc5;

constexpr int kTB = 13;                       // tile bits
constexpr int kTile = 1 << kTB;               // 8192 complex64 = 64 KB
constexpr int kMathThreads = 256;             // 8 math warps (tensor-core group application)
constexpr int kMemThreads = 128;              // 4 memory warps (HBM <-> smem)
constexpr int kThreads = kMathThreads + kMemThreads;
constexpr int kBufs = 3;                      // tile ring: loading / math / storing
constexpr int kMemPer = kTile / kMemThreads;  // 64 elements per memory thread per tile
constexpr int kMemThrBits = 7;
constexpr int kMaxGroups = 5;                 // groups per pass (B fragments in smem: 6 KB each)
constexpr int kMaxChainGates = 512;
constexpr int kMaxAllGroups = 512;            // groups over all passes (fragment table)
constexpr int kGroupWords = 48;               // B-fragment u32 per lane per group

// A group is a 16x16 complex unitary on 4 tile bits (gates on up to 4 axes
// multiplied together; a smaller group is padded with identity axes),
// applied to the tile viewed as [512 rows x 16] on mma.sync.m16n8k16:
// K = 32 real (2 k-steps), N = 32 real (4 n8 tiles), 4 m16 tiles per warp.
// B fragments per lane: 2 regs x 4 n-tiles x 2 k-steps x (B_hi, -B_hi, -B_lo) = 48 u32.
struct GroupParams {
  int frag_off;      // offset of the group's fragments in the table, in units of 32 u32
  int lane_slot[5];  // slot vectors of lane bits 0..4 = (q0, q1, g0, g1, g2)
  int warp_slot[3];  // math warp id bits
  int iter[4];       // slot XOR of m16-tile iteration m
  int h_slot;        // row + 8
  int q2_slot;       // column + 4
  int q3_slot;       // column + 8 (second k-step)
};

struct AbsorbParams {
  int n_outer;
  int n_groups;
  int frag_base;     // the pass's first group in the fragment table (units of 32 u32)
  int64_t n_tiles;
  // memory-thread enumeration e = mt + 128 i: offset = thread part + [i] part
  int64_t in_bit[kMemThrBits];
  int in_slot_bit[kMemThrBits];
  int64_t in_i[kMemPer];
  int in_slot_i[kMemPer];
  int64_t out_bit[kMemThrBits];
  int out_slot_bit[kMemThrBits];
  int64_t out_i[kMemPer];
  int out_slot_i[kMemPer];
  GroupParams g[kMaxGroups];
  int64_t outer_in[TNC_MAX_RANK];   // outer bit k of the tile index: input / output stride
  int64_t outer_out[TNC_MAX_RANK];
};

// Fragment-table job: group k (width w_k column bits, fragments at u32 offset
// off_k * 32) multiplies gates grp_gate[grp_first[k] .. grp_first[k+1]) in
// order; gate j acts on column bits (ca, cb).
struct FragParams {
  int n_groups;
  int grp_first[kMaxAllGroups + 1];
  int grp_off[kMaxAllGroups];
  signed char grp_w[kMaxAllGroups];
  short grp_gate[kMaxChainGates];
  signed char grp_ca[kMaxChainGates], grp_cb[kMaxChainGates];
  const float2* gate[kMaxChainGates];
  int64_t gstride[kMaxChainGates][4];  // element strides of the (out_a, out_b, in_a, in_b) legs
};

__host__ __device__ __forceinline__ int swz(int e) { return e ^ (((e >> 4) ^ (e >> 8) ^ (e >> 12)) & 15); }

__device__ __forceinline__ void cp_async8(uint32_t smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_dst), "l"(gmem_src) : "memory");
}

__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t h2_bits(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }

typedef unsigned long long u64;
__device__ __forceinline__ u64 pk(float2 v) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 upk(u64 r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
// packed fp32x2 FMA (one issue slot for a complex element)
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}



__device__ __forceinline__ float amax2(float2 a, float2 b) {
  return fmaxf(fmaxf(fabsf(a.x), fabsf(a.y)), fmaxf(fabsf(b.x), fabsf(b.y)));
}

// Group unitaries -> per-lane mma B fragments (hi / lo fp16) in global memory.
// One warp per group; lane 0 multiplies the embedded gates in double.
__global__ void absorb_frag_kernel(const FragParams p, uint32_t* __restrict__ table) {
  __shared__ double mr[16][16], mi[16][16], nr[16][16], ni[16][16];
  const int grp = blockIdx.x;
  const int lane = threadIdx.x;
  const int w = p.grp_w[grp], D = 1 << w;
  for (int e = lane; e < D * D; e += 32) {
    mr[e / D][e % D] = (e / D == e % D) ? 1.0 : 0.0;
    mi[e / D][e % D] = 0.0;
  }
  __syncwarp();
  for (int j = p.grp_first[grp]; j < p.grp_first[grp + 1]; ++j) {
    const int gi = p.grp_gate[j], ca = p.grp_ca[j], cb = p.grp_cb[j];
    const float2* u = p.gate[gi];
    const int64_t* st = p.gstride[gi];
    const int keep = ~((1 << ca) | (1 << cb));
    for (int e = lane; e < D * D; e += 32) {
      const int o = e / D, i = e % D;
      const int oa = (o >> ca) & 1, ob = (o >> cb) & 1;
      double sr = 0.0, si = 0.0;
      for (int q = 0; q < 4; ++q) {  // embedded gate G[o][k]: k differs from o only on (ca, cb)
        const int ka = q >> 1, kb = q & 1;
        const int k = (o & keep) | (ka << ca) | (kb << cb);
        const float2 g = u[oa * st[0] + ob * st[1] + ka * st[2] + kb * st[3]];
        sr += g.x * mr[k][i] - g.y * mi[k][i];
        si += g.x * mi[k][i] + g.y * mr[k][i];
      }
      nr[o][i] = sr;
      ni[o][i] = si;
    }
    __syncwarp();
    for (int e = lane; e < D * D; e += 32) {
      mr[e / D][e % D] = nr[e / D][e % D];
      mi[e / D][e % D] = ni[e / D][e % D];
    }
    __syncwarp();
  }
  // real B[k][n], k = 2i + d (input column i, d = re/im), n = 2o + c:
  //   B[2i][2o] = Mr[o][i], B[2i+1][2o] = -Mi[o][i], B[2i][2o+1] = Mi[o][i], B[2i+1][2o+1] = Mr[o][i]
  auto bval = [&](int k, int n) -> double {
    const int i = k >> 1, d = k & 1, o = n >> 1, c = n & 1;
    if (c == 0) return d == 0 ? mr[o][i] : -mi[o][i];
    return d == 0 ? mi[o][i] : mr[o][i];
  };
  const int n_tiles = D / 4, k_steps = D / 8;
  uint32_t* out = table + static_cast<int64_t>(p.grp_off[grp]) * 32 + lane * (6 * n_tiles * k_steps);
  const int q = lane & 3, gq = lane >> 2;
  // layout per lane: [set][n-tile][k-step][2 regs], sets (B_hi, -B_hi, -B_lo):
  // the tile side is split as (-hi, lo) so that  lo*B_hi + (-hi)*(-B_lo) +
  // (-hi)*(-B_hi)  is the 3-product sum (see split_nhi)
  for (int hl = 0; hl < 3; ++hl)
    for (int nt = 0; nt < n_tiles; ++nt)
      for (int ks = 0; ks < k_steps; ++ks) {
        const int n = 8 * nt + gq;
        const int kk[4] = {16 * ks + 2 * q, 16 * ks + 2 * q + 1, 16 * ks + 2 * q + 8, 16 * ks + 2 * q + 9};
        __half h[4];
        for (int j = 0; j < 4; ++j) {
          const double v = bval(kk[j], n);
          const __half hi = __double2half(v);
          const __half lo = __double2half(v - static_cast<double>(__half2float(hi)));
          h[j] = hl == 0 ? hi : hl == 1 ? __hneg(hi) : __hneg(lo);
        }
        uint32_t* o = out + 2 * ((hl * n_tiles + nt) * k_steps + ks);
        o[0] = h2_bits(__halves2half2(h[0], h[1]));
        o[1] = h2_bits(__halves2half2(h[2], h[3]));
      }
}

// Tile-side split of one complex element (x * 2^-e as fp16 pieces), 5 issue
// slots: t = x*s + M rounds x*s to a multiple of 16 (M = 1.5 * 2^27; the row
// max is scaled into [2^14, 2^15), so the rounded value has <= 11 significant
// bits and is exact in fp16), nh = M - t = -hi exactly, lo = x*s - hi exactly
// (fp16-rounded to 2^-22 of the row max).  Returns (-hi, lo) as half2 pairs.
constexpr u64 kM2 = 0x4d4000004d400000ull;    // (1.5 * 2^27, 1.5 * 2^27)
constexpr u64 kNeg1 = 0xbf800000bf800000ull;  // (-1, -1)
__device__ __forceinline__ void split_nhi(float2 x, u64 s, uint32_t& nhi, uint32_t& lo) {
  const u64 xv = pk(x);
  const u64 t = ffma2(xv, s, kM2);
  const u64 nh = ffma2(t, kNeg1, kM2);
  const u64 l = ffma2(xv, s, nh);
  nhi = h2_bits(__float22half2_rn(upk(nh)));
  lo = h2_bits(__float22half2_rn(upk(l)));
}

__device__ __forceinline__ u64 pow2_pair(uint32_t bits) { return (static_cast<u64>(bits) << 32) | bits; }

// One group on the tile: per m16 tile a thread holds rows (g, g+8) x columns
// (q, q+4, q+8, q+12); k-step s covers columns 8s..8s+7.  Two m16 tiles are
// processed together (independent chains for latency hiding; their 4 row
// exponents share one pair of shuffles).
__device__ __forceinline__ void apply_group(float2* tile, const GroupParams& gp, const uint32_t* fr,
                                            int base) {
  uint32_t fb[48];  // [set: B_hi, -B_hi, -B_lo][n-tile 4][k-step 2][2]
#pragma unroll
  for (int v = 0; v < 12; ++v) {
    const uint4 t = reinterpret_cast<const uint4*>(fr)[v];  // shared memory
    fb[4 * v + 0] = t.x;
    fb[4 * v + 1] = t.y;
    fb[4 * v + 2] = t.z;
    fb[4 * v + 3] = t.w;
  }
  // loop-invariant slot vectors in registers (no indexed param loads in the loop)
  const int h_slot = gp.h_slot, q2_slot = gp.q2_slot, q3_slot = gp.q3_slot;
  const int it_slot[4] = {gp.iter[0], gp.iter[1], gp.iter[2], gp.iter[3]};
#pragma unroll 1
  for (int mp = 0; mp < 4; mp += 2) {
    int sl[2][8];  // element e = h + 2 j + 4 s : row g + 8h, column q + 4j + 8s
    float2 x[2][8];
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      sl[u][0] = base ^ (mp ? it_slot[2 + u] : it_slot[u]);
      sl[u][1] = sl[u][0] ^ h_slot;
      sl[u][2] = sl[u][0] ^ q2_slot;
      sl[u][3] = sl[u][1] ^ q2_slot;
#pragma unroll
      for (int e = 0; e < 4; ++e) sl[u][4 + e] = sl[u][e] ^ q3_slot;
#pragma unroll
      for (int e = 0; e < 8; ++e) x[u][e] = tile[sl[u][e]];
    }
    // row maxima -> 4 exponent bytes, quad max with two shuffles
    uint32_t ex = 0;
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const float mx = fmaxf(amax2(x[u][h], x[u][h + 2]), amax2(x[u][h + 4], x[u][h + 6]));
        ex |= (__float_as_uint(mx) >> 23) << (8 * (2 * u + h));
      }
    ex = __vmaxu4(ex, __shfl_xor_sync(0xffffffffu, ex, 1));
    ex = __vmaxu4(ex, __shfl_xor_sync(0xffffffffu, ex, 2));
    ex = __vmaxu4(ex, 0x0f0f0f0fu);
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      u64 sc[2], un[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t E = (ex >> (8 * (2 * u + h))) & 0xffu;
        sc[h] = pow2_pair((268u - E) << 23);  // 2^(141 - E): row max -> [2^14, 2^15)
        un[h] = pow2_pair((E - 14u) << 23);   // 2^(E - 141)
      }
      uint32_t ah[2][4], al[2][4];
#pragma unroll
      for (int ks = 0; ks < 2; ++ks)
#pragma unroll
        for (int r = 0; r < 4; ++r) split_nhi(x[u][4 * ks + r], sc[r & 1], ah[ks][r], al[ks][r]);
      // two accumulation chains per n-tile (small terms / main term), summed
      // after: halves the dependent-HMMA chain length
      float d[4][4], c[4][4];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        d[nt][0] = d[nt][1] = d[nt][2] = d[nt][3] = 0.f;
        c[nt][0] = c[nt][1] = c[nt][2] = c[nt][3] = 0.f;
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
          const int o = 2 * (nt * 2 + ks);
          mma16816(c[nt], al[ks], fb[o], fb[o + 1]);            // lo * B_hi
          mma16816(d[nt], ah[ks], fb[16 + o], fb[16 + o + 1]);  // (-hi) * (-B_hi)
          mma16816(c[nt], ah[ks], fb[32 + o], fb[32 + o + 1]);  // (-hi) * (-B_lo)
        }
#pragma unroll
        for (int v = 0; v < 4; ++v) d[nt][v] += c[nt][v];
      }
      // output column o = 4 nt + q = q + 4 j + 8 s with j = nt & 1, s = nt >> 1
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int e0 = 2 * (nt & 1) + 4 * (nt >> 1);
        tile[sl[u][e0]] = upk(ffma2(pk(make_float2(d[nt][0], d[nt][1])), un[0], 0ull));
        tile[sl[u][e0 + 1]] = upk(ffma2(pk(make_float2(d[nt][2], d[nt][3])), un[1], 0ull));
      }
    }
  }
}

__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Sum over the outer (non-tile) axes of tile t: one warp, lanes split the axes.
__device__ __forceinline__ int64_t tile_base(int64_t t, const int64_t* __restrict__ st, int n_outer, int lane) {
  int64_t b = 0;
  for (int a = lane; a < n_outer; a += 32)
    if ((t >> a) & 1) b += st[a];
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) b += __shfl_xor_sync(0xffffffffu, b, s);
  return b;
}

// One pass over the tensor, one persistent CTA per SM, warp-specialised over a
// ring of 3 tile buffers (192 KB of smem):
//   memory warps (4):  cp.async gather of tile k (HBM -> smem, 8-byte elements,
//                      completion tracked by mbarrier full[b]), then the store
//                      of tile k-1 (smem -> HBM in the output layout) once the
//                      math warps released it (computed[b]), then empty[b];
//   math warps (8):    the pass's gate groups on tensor cores, in place.
// Loads, math and stores of three consecutive tiles overlap.
__global__ void __launch_bounds__(kThreads, 1) absorb_mma_kernel(const float2* __restrict__ in,
                                                                  float2* __restrict__ out,
                                                                  const uint32_t* __restrict__ frags,
                                                                  const AbsorbParams p) {
  extern __shared__ __align__(16) float2 tiles[];  // kBufs x kTile, then the pass's B fragments
  __shared__ __align__(8) uint64_t full[kBufs], computed[kBufs], empty[kBufs];
  __shared__ int64_t s_oin[TNC_MAX_RANK], s_oout[TNC_MAX_RANK];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  const int warp = tid >> 5;
  if (tid < p.n_outer) {
    s_oin[tid] = p.outer_in[tid];
    s_oout[tid] = p.outer_out[tid];
  }
  // the pass's group B fragments (48 u32 per lane per group) -> smem once
  uint32_t* sfrag = reinterpret_cast<uint32_t*>(tiles + kBufs * kTile);
  {
    const uint4* src = reinterpret_cast<const uint4*>(frags + static_cast<int64_t>(p.frag_base) * 32);
    uint4* dst = reinterpret_cast<uint4*>(sfrag);
    for (int i = tid; i < p.n_groups * kGroupWords * 32 / 4; i += kThreads) dst[i] = __ldg(src + i);
  }
  if (tid == 0) {
    for (int b = 0; b < kBufs; ++b) {
      mbar_init(&full[b], kMemThreads);
      mbar_init(&computed[b], 1);
      mbar_init(&empty[b], kMemThreads);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= kMathThreads / 32) {
    // ---- memory warps
    const int mt = tid - kMathThreads;
    int64_t my_in = 0, my_out = 0;
    int my_in_slot = 0, my_out_slot = 0;
#pragma unroll
    for (int j = 0; j < kMemThrBits; ++j)
      if ((mt >> j) & 1) {
        my_in += p.in_bit[j];
        my_out += p.out_bit[j];
        my_in_slot ^= p.in_slot_bit[j];
        my_out_slot ^= p.out_slot_bit[j];
      }
    const uint32_t tiles_s = smem_u32(tiles);
    for (int64_t k = 0;; ++k) {
      const int64_t t = blockIdx.x + k * gridDim.x;
      const bool have = t < p.n_tiles;
      if (have) {
        const int b = static_cast<int>(k % kBufs);
        if (k >= kBufs) mbar_wait(&empty[b], static_cast<uint32_t>((k / kBufs - 1) & 1));
        const float2* src = in + tile_base(t, s_oin, p.n_outer, lane) + my_in;
        const uint32_t dst = tiles_s + b * kTile * 8;
#pragma unroll 16
        for (int i = 0; i < kMemPer; ++i) cp_async8(dst + ((my_in_slot ^ p.in_slot_i[i]) << 3), src + p.in_i[i]);
        cp_async_arrive(&full[b]);
      }
      if (k >= 1) {
        const int64_t kp = k - 1;
        const int bp = static_cast<int>(kp % kBufs);
        mbar_wait(&computed[bp], static_cast<uint32_t>((kp / kBufs) & 1));
        const float2* tile = tiles + bp * kTile;
        float2* dst = out + tile_base(t - gridDim.x, s_oout, p.n_outer, lane) + my_out;
#pragma unroll 16
        for (int i = 0; i < kMemPer; ++i) __stcs(dst + p.out_i[i], tile[my_out_slot ^ p.out_slot_i[i]]);
        mbar_arrive(&empty[bp]);
      }
      if (!have) break;
    }
  } else {
    // ---- math warps
    for (int64_t k = 0;; ++k) {
      const int64_t t = blockIdx.x + k * gridDim.x;
      if (t >= p.n_tiles) break;
      const int b = static_cast<int>(k % kBufs);
      mbar_wait(&full[b], static_cast<uint32_t>((k / kBufs) & 1));
      float2* tile = tiles + b * kTile;
      for (int g = 0; g < p.n_groups; ++g) {
        const GroupParams& gp = p.g[g];
        int base = 0;
#pragma unroll
        for (int j = 0; j < 5; ++j)
          if ((lane >> j) & 1) base ^= gp.lane_slot[j];
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if ((warp >> j) & 1) base ^= gp.warp_slot[j];
        apply_group(tile, gp, sfrag + (g * 32 + lane) * kGroupWords, base);
        asm volatile("bar.sync 1, %0;" ::"n"(kMathThreads) : "memory");
      }
      if (tid == 0) mbar_arrive(&computed[b]);
    }
  }
}

// ---------------------------------------------------------------------------
// host planning

struct GateRef {
  int pa, pb;  // physical axes of in_a, in_b
};

struct Pass {
  std::vector<int> gates;                 // gate indices, dependency order
  std::vector<int> tile;                  // tile axes (set, before bit placement)
  std::vector<std::vector<int>> groups;   // gate indices per 3-axis group
  std::vector<std::vector<int>> gaxes;    // the group's axes (2 or 3)
};

bool has(const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); }
void add(std::vector<int>& v, int x) {
  if (!has(v, x)) v.push_back(x);
}

// Greedy packing with deferral: walk `todo` in order; a gate joins if it is
// not blocked (no earlier deferred gate on its axes) and the set stays within
// `cap` axes; otherwise it is deferred and blocks its axes.
std::vector<int> pack(const std::vector<GateRef>& gates, const std::vector<int>& todo, std::vector<int>& axes,
                      int cap, std::vector<int>& rest) {
  std::vector<int> chosen, blocked;
  rest.clear();
  for (int gi : todo) {
    const int a = gates[gi].pa, b = gates[gi].pb;
    if (has(blocked, a) || has(blocked, b)) {
      add(blocked, a);
      add(blocked, b);
      rest.push_back(gi);
      continue;
    }
    std::vector<int> trial = axes;
    add(trial, a);
    add(trial, b);
    if (static_cast<int>(trial.size()) <= cap) {
      axes = trial;
      chosen.push_back(gi);
    } else {
      add(blocked, a);
      add(blocked, b);
      rest.push_back(gi);
    }
  }
  return chosen;
}

std::vector<int> fastest(const std::vector<int64_t>& stride, int r, int n) {
  std::vector<int> ax(r);
  for (int i = 0; i < r; ++i) ax[i] = i;
  std::sort(ax.begin(), ax.end(), [&](int x, int y) { return stride[x] < stride[y]; });
  ax.resize(std::min(n, r));
  return ax;
}

constexpr int kLink = 3;  // fastest axes shared by consecutive layouts (64-byte runs)

int plan_passes(int r, const std::vector<GateRef>& gates, const std::vector<int64_t>& in_stride,
                const std::vector<int64_t>& final_stride, std::vector<Pass>& passes) {
  passes.clear();
  const std::vector<int> out_fast = fastest(final_stride, r, kLink);
  std::vector<int> link = fastest(in_stride, r, kLink);
  std::vector<int> todo(gates.size());
  for (size_t i = 0; i < gates.size(); ++i) todo[i] = static_cast<int>(i);
  for (int guard = 0; guard < 4 * static_cast<int>(gates.size()) + 4; ++guard) {
    Pass ps;
    ps.tile = link;
    std::vector<int> rest;
    ps.gates = pack(gates, todo, ps.tile, kTB, rest);
    if (ps.gates.empty() && !todo.empty()) return set_error("absorb: a gate does not fit a tile"), TNC_ERR_UNSUPPORTED;
    // groups of <= 4 axes (same deferral rule); groups beyond kMaxGroups go
    // back to the remaining gates (the first k groups are a dependency-closed
    // prefix of the pass's gates)
    {
      std::vector<int> todo2 = ps.gates;
      while (!todo2.empty()) {
        std::vector<int> axes, rest2;
        std::vector<int> grp = pack(gates, todo2, axes, 4, rest2);
        if (static_cast<int>(ps.groups.size()) == kMaxGroups) {
          rest.insert(rest.end(), todo2.begin(), todo2.end());
          std::sort(rest.begin(), rest.end());
          break;
        }
        ps.groups.push_back(grp);
        ps.gaxes.push_back(axes);
        todo2 = rest2;
      }
      ps.gates.clear();
      for (const auto& grp : ps.groups) ps.gates.insert(ps.gates.end(), grp.begin(), grp.end());
    }
    if (rest.empty()) {
      std::vector<int> with_out = ps.tile;
      for (int a : out_fast) add(with_out, a);
      if (static_cast<int>(with_out.size()) <= kTB) {
        ps.tile = with_out;
        passes.push_back(ps);
        break;
      }
      // final layout's fast axes do not fit: this pass hands over to a pure
      // permutation pass through link axes
      std::vector<int> nl;
      for (int a : out_fast)
        if (has(ps.tile, a)) nl.push_back(a);
      for (int a : ps.tile)
        if (static_cast<int>(nl.size()) < kLink) add(nl, a);
      passes.push_back(ps);
      Pass fin;
      fin.tile = nl;
      for (int a : out_fast) add(fin.tile, a);
      passes.push_back(fin);
      break;
    }
    // link to the next pass: tile axes the remaining gates touch, then final
    // fast axes, then any tile axis
    std::vector<int> nl;
    for (int gi : rest)
      for (int a : {gates[gi].pa, gates[gi].pb})
        if (has(ps.tile, a) && static_cast<int>(nl.size()) < kLink) add(nl, a);
    for (int a : out_fast)
      if (has(ps.tile, a) && static_cast<int>(nl.size()) < kLink) add(nl, a);
    for (int a : ps.tile)
      if (static_cast<int>(nl.size()) < kLink) add(nl, a);
    passes.push_back(ps);
    link = nl;
    todo = rest;
  }
  if (passes.empty()) return set_error("absorb: planning failed"), TNC_ERR_UNSUPPORTED;
  return TNC_OK;
}

// Intermediate layout feeding pass `next`: [outer axes][next tile axes][link]
std::vector<int64_t> handover_layout(int r, const Pass& next, const std::vector<int>& link) {
  std::vector<int> order;  // most significant first
  for (int a = 0; a < r; ++a)
    if (!has(next.tile, a)) order.push_back(a);
  for (int a : next.tile)
    if (!has(link, a)) order.push_back(a);
  for (int a : link) order.push_back(a);
  std::vector<int64_t> st(r);
  for (int i = 0; i < r; ++i) st[order[i]] = static_cast<int64_t>(1) << (r - 1 - i);
  return st;
}

// Place the pass's 13 tile axes on tile bits: the 4 fastest load axes and the
// 4 fastest store axes each cover the 4 bank classes (bit mod 4).
std::vector<int> place_bits(const std::vector<int>& tile, const std::vector<int64_t>& in_st,
                            const std::vector<int64_t>& out_st) {
  auto by = [&](const std::vector<int64_t>& st) {
    std::vector<int> v = tile;
    std::sort(v.begin(), v.end(), [&](int x, int y) { return st[x] < st[y]; });
    v.resize(4);
    return v;
  };
  const std::vector<int> A = by(in_st), B = by(out_st);
  std::vector<int> cls(tile.size(), -1);  // class per tile-vector index
  auto idx = [&](int a) { return static_cast<int>(std::find(tile.begin(), tile.end(), a) - tile.begin()); };
  std::vector<int> usedA, usedB;
  for (int a : A)
    if (has(B, a)) {
      int c = 0;
      while (has(usedA, c) || has(usedB, c)) ++c;
      cls[idx(a)] = c;
      usedA.push_back(c);
      usedB.push_back(c);
    }
  for (int a : A)
    if (cls[idx(a)] < 0) {
      int c = 0;
      while (has(usedA, c)) ++c;
      cls[idx(a)] = c;
      usedA.push_back(c);
    }
  for (int a : B)
    if (cls[idx(a)] < 0) {
      int c = 0;
      while (has(usedB, c)) ++c;
      cls[idx(a)] = c;
      usedB.push_back(c);
    }
  std::vector<int> bit_axis(kTB, -1);
  for (size_t i = 0; i < tile.size(); ++i)
    if (cls[i] >= 0)
      for (int b = cls[i]; b < kTB; b += 4)
        if (bit_axis[b] < 0) {
          bit_axis[b] = tile[i];
          break;
        }
  for (size_t i = 0; i < tile.size(); ++i)
    if (cls[i] < 0)
      for (int b = 0; b < kTB; ++b)
        if (bit_axis[b] < 0) {
          bit_axis[b] = tile[i];
          break;
        }
  return bit_axis;  // bit position -> physical axis
}

int build_pass_params(int r, const Pass& ps, const std::vector<int>& bit_axis, const std::vector<int64_t>& in_st,
                      const std::vector<int64_t>& out_st, int frag_base /* u32 x 32 units */, AbsorbParams& p,
                      std::vector<std::vector<int>>& group_colbits) {
  std::memset(&p, 0, sizeof(p));
  std::vector<int> pos(r, -1);
  for (int b = 0; b < kTB; ++b) pos[bit_axis[b]] = b;
  if (std::getenv("TNC_ABSORB_DEBUG")) {
    std::fprintf(stderr, "pass: %zu gates, %zu groups; tile bits->axis:", ps.gates.size(), ps.groups.size());
    for (int b = 0; b < kTB; ++b) std::fprintf(stderr, " %d", bit_axis[b]);
    std::fprintf(stderr, "\n");
  }
  auto enum_order = [&](const std::vector<int64_t>& st) {
    std::vector<int> v(bit_axis);
    std::sort(v.begin(), v.end(), [&](int x, int y) { return st[x] < st[y]; });
    return v;
  };
  const std::vector<int> lo = enum_order(in_st), so = enum_order(out_st);
  for (int j = 0; j < kMemThrBits; ++j) {
    p.in_bit[j] = in_st[lo[j]];
    p.in_slot_bit[j] = swz(1 << pos[lo[j]]);
    p.out_bit[j] = out_st[so[j]];
    p.out_slot_bit[j] = swz(1 << pos[so[j]]);
  }
  for (int i = 0; i < kMemPer; ++i) {
    int64_t oi = 0, oo = 0;
    int si = 0, so_ = 0;
    for (int j = 0; j < kTB - kMemThrBits; ++j)
      if ((i >> j) & 1) {
        oi += in_st[lo[kMemThrBits + j]];
        si ^= swz(1 << pos[lo[kMemThrBits + j]]);
        oo += out_st[so[kMemThrBits + j]];
        so_ ^= swz(1 << pos[so[kMemThrBits + j]]);
      }
    p.in_i[i] = oi;
    p.in_slot_i[i] = si;
    p.out_i[i] = oo;
    p.out_slot_i[i] = so_;
  }
  // outer axes: least significant tile-index bits = smallest input stride
  std::vector<int> outer;
  for (int a = 0; a < r; ++a)
    if (pos[a] < 0) outer.push_back(a);
  std::sort(outer.begin(), outer.end(), [&](int x, int y) { return in_st[x] < in_st[y]; });
  p.n_outer = static_cast<int>(outer.size());
  for (int k = 0; k < p.n_outer; ++k) {
    p.outer_in[k] = in_st[outer[k]];
    p.outer_out[k] = out_st[outer[k]];
  }
  p.n_tiles = static_cast<int64_t>(1) << p.n_outer;
  p.n_groups = static_cast<int>(ps.groups.size());
  group_colbits.clear();
  int foff = frag_base;
  p.frag_base = frag_base;
  for (int g = 0; g < p.n_groups; ++g) {
    std::vector<int> gb;  // tile bits of the group's axes
    for (int a : ps.gaxes[g]) gb.push_back(pos[a]);
    auto cl = [](int b) { return b & 3; };
    const int w = 4;
    // pad a smaller group to 4 column bits with row bits of fresh classes
    while (static_cast<int>(gb.size()) < w) {
      int best = -1;
      for (int b = 0; b < kTB && best < 0; ++b) {
        bool fresh = !has(gb, b);
        for (int x : gb) fresh = fresh && cl(x) != cl(b);
        if (fresh) best = b;
      }
      for (int b = 0; b < kTB && best < 0; ++b)
        if (!has(gb, b)) best = b;
      gb.push_back(best);
    }
    // q0, q1 (lane bits 0, 1): two column bits of distinct classes
    std::vector<int> cols = gb;
    for (size_t i = 0; i < cols.size(); ++i)
      for (size_t j = i + 1; j < cols.size(); ++j)
        if (cl(cols[i]) != cl(cols[j]) && !(i == 0 && j == 1) && cl(cols[0]) == cl(cols[1])) {
          std::swap(cols[0], cols[i]);
          std::swap(cols[1], cols[j]);
        }
    std::vector<int> rows;
    for (int b = 0; b < kTB; ++b)
      if (!has(cols, b)) rows.push_back(b);
    // g0, g1: row bits completing the 4 classes of a half-warp
    std::vector<int> lane_bits = {cols[0], cols[1]};
    for (int pass_ = 0; pass_ < 2; ++pass_) {
      for (int b : rows) {
        if (static_cast<int>(lane_bits.size()) >= 4) break;
        if (has(lane_bits, b)) continue;
        bool distinct = true;
        for (int x : lane_bits) distinct = distinct && cl(x) != cl(b);
        if (distinct || pass_ == 1) lane_bits.push_back(b);
      }
    }
    std::vector<int> others;
    for (int b : rows)
      if (!has(lane_bits, b)) others.push_back(b);
    // others (7 bits): g2, h, warp x3, iteration x2
    GroupParams& gp = p.g[g];
    gp.frag_off = foff;
    foff += kGroupWords;
    for (int j = 0; j < 4; ++j) gp.lane_slot[j] = swz(1 << lane_bits[j]);
    gp.lane_slot[4] = swz(1 << others[0]);
    gp.h_slot = swz(1 << others[1]);
    for (int j = 0; j < 3; ++j) gp.warp_slot[j] = swz(1 << others[2 + j]);
    for (int m = 0; m < 4; ++m) {
      int x = 0;
      for (int j = 0; j < 2; ++j)
        if ((m >> j) & 1) x ^= swz(1 << others[5 + j]);
      gp.iter[m] = x;
    }
    gp.q2_slot = swz(1 << cols[2]);
    gp.q3_slot = swz(1 << cols[3]);
    // column bit c of the group unitary <-> tile bit cols[c]
    group_colbits.push_back(cols);
    if (std::getenv("TNC_ABSORB_DEBUG")) {
      auto cl = [](int b) { return b & 3; };
      std::fprintf(stderr, "  group %d: gates %zu axes %zu cols [%d %d %d %d] lanes [%d %d %d %d] classes [%d %d %d %d]\n", g,
                   ps.groups[g].size(), ps.gaxes[g].size(), cols[0], cols[1], cols[2], cols[3], lane_bits[0],
                   lane_bits[1], lane_bits[2], lane_bits[3], cl(lane_bits[0]), cl(lane_bits[1]), cl(lane_bits[2]),
                   cl(lane_bits[3]));
    }
  }
  return TNC_OK;
}

struct ChainPlan {
  std::vector<GateRef> refs;
  std::vector<int> lorder;
  std::vector<Pass> passes;
  std::vector<std::vector<int64_t>> in_st, out_st;  // per pass
  int total_groups = 0;
};

int plan_chain(int r, int n_gates, const int32_t* axes, ChainPlan& cp) {
  if (r < kTB || r > TNC_MAX_RANK - 2) TNC_RET(TNC_ERR_UNSUPPORTED, "absorb: rank must be in [13, 62]");
  if (n_gates < 0 || n_gates > kMaxChainGates) TNC_RET(TNC_ERR_INVALID, "absorb: gate count out of range");
  cp.lorder.resize(r);
  for (int i = 0; i < r; ++i) cp.lorder[i] = i;
  cp.refs.clear();
  for (int g = 0; g < n_gates; ++g) {
    const int la = axes[2 * g], lb = axes[2 * g + 1];
    if (la < 0 || la >= r || lb < 0 || lb >= r || la == lb)
      TNC_RET(TNC_ERR_CONTRACTION, "absorb: gate axes out of range");
    GateRef ref{cp.lorder[la], cp.lorder[lb]};
    cp.refs.push_back(ref);
    std::vector<int> next;
    for (int i = 0; i < r; ++i)
      if (i != la && i != lb) next.push_back(cp.lorder[i]);
    next.push_back(ref.pa);  // out_a occupies in_a's physical axis
    next.push_back(ref.pb);
    cp.lorder.swap(next);
  }
  std::vector<int64_t> phys(r), fin(r);
  for (int a = 0; a < r; ++a) phys[a] = static_cast<int64_t>(1) << (r - 1 - a);
  for (int i = 0; i < r; ++i) fin[cp.lorder[i]] = static_cast<int64_t>(1) << (r - 1 - i);
  TNC_TRY(plan_passes(r, cp.refs, phys, fin, cp.passes));
  const int P = static_cast<int>(cp.passes.size());
  cp.in_st.assign(P, {});
  cp.out_st.assign(P, {});
  cp.in_st[0] = phys;
  cp.out_st[P - 1] = fin;
  for (int k = 0; k + 1 < P; ++k) {
    // link axes of the handover: the next pass's 3 fastest... chosen as the
    // axes both tiles share, in the order the planner picked them
    std::vector<int> link;
    for (int a : cp.passes[k + 1].tile)
      if (has(cp.passes[k].tile, a) && static_cast<int>(link.size()) < kLink) link.push_back(a);
    // pad both tiles to 13 axes first so the handover can use them
    cp.out_st[k] = handover_layout(r, cp.passes[k + 1], link);
    cp.in_st[k + 1] = cp.out_st[k];
  }
  // pad tiles to 13 axes: fastest input axes first (longer contiguous runs)
  for (int k = 0; k < P; ++k) {
    std::vector<int> order(r);
    for (int a = 0; a < r; ++a) order[a] = a;
    const auto& st = cp.in_st[k].empty() ? phys : cp.in_st[k];
    std::sort(order.begin(), order.end(), [&](int x, int y) { return st[x] < st[y]; });
    for (int a : order)
      if (static_cast<int>(cp.passes[k].tile.size()) < kTB) add(cp.passes[k].tile, a);
  }
  cp.total_groups = 0;
  for (auto& ps : cp.passes) cp.total_groups += static_cast<int>(ps.groups.size());
  if (cp.total_groups > kMaxAllGroups) TNC_RET(TNC_ERR_UNSUPPORTED, "absorb: too many gate groups");
  return TNC_OK;
}

// fragment table: 32 u32 per lane per group
size_t frag_bytes(const ChainPlan& cp) {
  return (std::max<size_t>(static_cast<size_t>(cp.total_groups) * kGroupWords * 32, 1) * 4 + 255) & ~size_t(255);
}

}  // namespace

int absorb_chain_workspace(int t_rank, int n_gates, const int32_t* axes, size_t* bytes) {
  ChainPlan cp;
  TNC_TRY(plan_chain(t_rank, n_gates, axes, cp));
  const size_t tensor = cp.passes.size() > 1 ? (static_cast<size_t>(1) << t_rank) * sizeof(float2) : 0;
  *bytes = tensor + frag_bytes(cp);
  return TNC_OK;
}

int absorb_chain_launch(int t_rank, const void* t_in, void* t_out, int n_gates, const void* const* gates,
                        const int64_t* gate_strides, const int32_t* axes, void* workspace,
                        size_t workspace_bytes, cudaStream_t stream) {
  const int r = t_rank;
  ChainPlan cp;
  TNC_TRY(plan_chain(r, n_gates, axes, cp));
  const int P = static_cast<int>(cp.passes.size());
  const size_t tensor = P > 1 ? (static_cast<size_t>(1) << r) * sizeof(float2) : 0;
  if (workspace_bytes < tensor + frag_bytes(cp) || workspace == nullptr)
    TNC_RET(TNC_ERR_WORKSPACE, "absorb: workspace too small (see tnc_absorb_chain_workspace)");
  for (int g = 0; g < n_gates; ++g)
    if (gates[g] == nullptr) TNC_RET(TNC_ERR_INVALID, "absorb: null gate pointer");
  float2* ws = static_cast<float2*>(workspace);
  uint32_t* table = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(workspace) + tensor);

  // per-pass parameters (bit placement needs both layouts)
  std::vector<AbsorbParams> params(P);
  FragParams fp;
  std::memset(&fp, 0, sizeof(fp));
  int gbase = 0, gidx = 0, foff = 0;
  for (int k = 0; k < P; ++k) {
    const Pass& ps = cp.passes[k];
    const std::vector<int> bit_axis = place_bits(ps.tile, cp.in_st[k], cp.out_st[k]);
    std::vector<std::vector<int>> colbits;
    TNC_TRY(build_pass_params(r, ps, bit_axis, cp.in_st[k], cp.out_st[k], foff, params[k], colbits));
    std::vector<int> pos(r, -1);
    for (int b = 0; b < kTB; ++b) pos[bit_axis[b]] = b;
    for (size_t g = 0; g < ps.groups.size(); ++g) {
      fp.grp_first[gbase + g] = gidx;
      fp.grp_off[gbase + g] = params[k].g[g].frag_off;
      fp.grp_w[gbase + g] = static_cast<signed char>(colbits[g].size());
      foff += kGroupWords;
      for (int gi : ps.groups[g]) {
        const GateRef& gr = cp.refs[gi];
        auto col = [&](int axis) {
          const int b = pos[axis];
          for (size_t c = 0; c < colbits[g].size(); ++c)
            if (colbits[g][c] == b) return static_cast<int>(c);
          return -1;
        };
        fp.grp_gate[gidx] = static_cast<short>(gi);
        fp.grp_ca[gidx] = static_cast<signed char>(col(gr.pa));
        fp.grp_cb[gidx] = static_cast<signed char>(col(gr.pb));
        ++gidx;
      }
    }
    gbase += static_cast<int>(ps.groups.size());
  }
  fp.grp_first[gbase] = gidx;
  fp.n_groups = gbase;
  for (int g = 0; g < n_gates; ++g) {
    fp.gate[g] = static_cast<const float2*>(gates[g]);
    for (int k = 0; k < 4; ++k) fp.gstride[g][k] = gate_strides[4 * g + k];
  }
  if (fp.n_groups > 0) {
    absorb_frag_kernel<<<fp.n_groups, 32, 0, stream>>>(fp, table);
    TNC_CHECK_LAUNCH();
  }
  int max_groups = 0;
  for (const auto& prm : params) max_groups = std::max(max_groups, prm.n_groups);
  const size_t smem = static_cast<size_t>(kBufs) * kTile * sizeof(float2) +
                      static_cast<size_t>(max_groups) * kGroupWords * 32 * 4;
  TNC_CUDA_TRY(cudaFuncSetAttribute(absorb_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  const float2* cur = static_cast<const float2*>(t_in);
  for (int k = 0; k < P; ++k) {
    float2* dst = ((P - 1 - k) % 2 == 0) ? static_cast<float2*>(t_out) : ws;
    const AbsorbParams& p = params[k];
    const int64_t blocks = std::min<int64_t>(p.n_tiles, static_cast<int64_t>(num_sms()));
    {
      ProfScope prof(PROF_ABSORB, 768.0 * p.n_groups * static_cast<double>(int64_t(1) << r),
                     16.0 * static_cast<double>(int64_t(1) << r), stream);
      absorb_mma_kernel<<<static_cast<unsigned>(blocks), kThreads, smem, stream>>>(cur, dst, table, p);
      TNC_CHECK_LAUNCH();
    }
    cur = dst;
  }
  return TNC_OK;
}

int absorb_chain_passes(int t_rank, int n_gates, const int32_t* axes, int* passes, int* groups) {
  ChainPlan cp;
  TNC_TRY(plan_chain(t_rank, n_gates, axes, cp));
  *passes = static_cast<int>(cp.passes.size());
  *groups = cp.total_groups;
  if (std::getenv("TNC_ABSORB_DEBUG")) {  // print the bit placement of every pass
    AbsorbParams* prm = new AbsorbParams;
    for (size_t k = 0; k < cp.passes.size(); ++k) {
      std::vector<std::vector<int>> colbits;
      build_pass_params(t_rank, cp.passes[k], place_bits(cp.passes[k].tile, cp.in_st[k], cp.out_st[k]), cp.in_st[k],
                        cp.out_st[k], 0, *prm, colbits);
    }
    delete prm;
  }
  return TNC_OK;
}

}  // namespace tnc
