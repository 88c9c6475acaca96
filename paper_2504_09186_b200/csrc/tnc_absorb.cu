// K4: step fusion -- a chain of two-leg gate absorptions into one resident
// tensor in the fewest HBM passes, the gate math overlapped with the HBM
// streams.
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
//    C2 (16 random gates on a rank-30 tensor): 2 passes (3 with in-order
//    sections of 12-bit tiles).
//  * Pipeline.  One persistent CTA per SM (640 threads), warp-specialised over
//    a ring of 3 tile buffers: 4 memory warps gather tile k (cp.async,
//    mbarrier-tracked) and store tile k-2, and TWO math teams of 8 warps
//    each own every other tile, so one team's shared-memory regrouping
//    (cube loads / stores, team barrier) overlaps the other team's FP32 math.
//    A pure copy pass runs at 6.4 TB/s (99 % of the measured HBM peak), so
//    the pass time is max(HBM, gate math, tile regrouping).
//  * Math.  Gates are grouped on <= 5 tile axes; each math thread holds a
//    32-element register cube of the group's axes (256 threads x 32 = the
//    tile) and applies the group's 4x4 gates with packed FP32 FMAs (FFMA2:
//    2 per complex MAC).  The pass's gate coefficients sit in the constant
//    bank (copied device-to-device from the table the table kernel builds
//    from the caller's device gate tensors: no host round trip), so the
//    FFMA2s take them as uniform-register operands and a math thread needs
//    96 registers.  FFMA2 issues at 0.46 / clk / SM sub-partition
//    (tools/ffma2_rate.cu): the same 118 FMA lanes / clk / SM as scalar
//    FFMA in half the issue slots, which sets the FP32 floor of a pass.
//    (A tensor-core variant -- 16x16 group unitaries on mma.sync with a
//    3xFP16 split -- was correct but issue-bound at ~2 ms per group: commit
//    d9b05fc.)
//  * Banks.  8-byte smem slots are XOR-swizzled (swz); a tile bit's bank class
//    is (bit mod 4).  The host places tile axes so that the 4 fastest load
//    axes and the 4 fastest store axes each cover the 4 classes, and picks a
//    cube's lane bits with distinct classes.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "tnc_common.cuh"
#include "tnc_tcgen05.cuh"

namespace tnc {

namespace {

using namespace tc5;

constexpr int kTB = 13;                       // tile bits
constexpr int kTile = 1 << kTB;               // 8192 complex64 = 64 KB
constexpr int kTeams = 2;                     // math teams, one tile each
constexpr int kTeamThreads = 256;             // 8 math warps: one 32-element cube per thread
constexpr int kMathThreads = kTeams * kTeamThreads;
constexpr int kMemThreads = 128;              // 4 memory warps (HBM <-> smem)
constexpr int kThreads = kMathThreads + kMemThreads;
constexpr int kBufs = 3;                      // tile ring: loading or storing / team 0 / team 1
constexpr int kMemPer = kTile / kMemThreads;  // 64 elements per memory thread per tile
constexpr int kMemThrBits = 7;
constexpr int kCubeBits = 5;
constexpr int kCube = 1 << kCubeBits;
constexpr int kMaxGroups = 24;                // groups per pass
constexpr int kMaxPassGates = 64;             // gates per pass (constant bank: 192 B each)
constexpr int kMaxChainGates = 512;

// The running pass's gate coefficients, 48 floats per gate: 16 aligned pairs
// (-im, im) of U[o][i], then the 16 real parts (an FFMA2 takes the pair as a
// 64-bit uniform-register operand and the real part as a broadcast scalar).
constexpr int kGateFloats = 48;
__constant__ float c_gates[kMaxPassGates * kGateFloats];

struct GroupParams {
  int cube_slot[kCubeBits];  // slot vectors of the cube (register-index) bits
  int lane_slot[5];          // lane bits
  int warp_slot[3];          // math warp id bits
  int g_first, g_last;       // the group's gates in the pass's gate list
};

struct AbsorbParams {
  int n_outer;
  int n_groups;
  int n_gates;               // gates of this pass
  int table_base;            // the pass's first gate in the device table
  int teams;                 // math teams in use (2; 1 = A/B switch TNC_ABSORB_TEAMS)
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
  int gate_local[kMaxPassGates];    // 8 * (cube bit of in_a) + cube bit of in_b, a < b
  int64_t outer_in[TNC_MAX_RANK];   // outer bit k of the tile index: input / output stride
  int64_t outer_out[TNC_MAX_RANK];
};

// Device gate tables: entry j = the 48 floats (see c_gates) of chain gate
// src[j], oriented so that its in_a axis is the lower cube bit.
struct TableParams {
  int n;
  short src[kMaxChainGates];
  signed char swap[kMaxChainGates];
  const float2* gate[kMaxChainGates];
  int64_t gstride[kMaxChainGates][4];  // element strides of the (out_a, out_b, in_a, in_b) legs
};

// lowest set bit of n in [1, 31] (compile-time under full unrolling)
__host__ __device__ constexpr int ctz5(int n) { return (n & 1) ? 0 : (n & 2) ? 1 : (n & 4) ? 2 : (n & 8) ? 3 : 4; }

__host__ __device__ __forceinline__ int swz(int e) { return e ^ (((e >> 4) ^ (e >> 8) ^ (e >> 12)) & 15); }

__device__ __forceinline__ void cp_async8(uint32_t smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_dst), "l"(gmem_src) : "memory");
}

__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

typedef unsigned long long u64;
__device__ __forceinline__ u64 as_u64(float2 v) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y));
  return r;
}
__device__ __forceinline__ float2 as_f2(u64 r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ u64 bcast(float x) {
  u64 r;
  asm("mov.b64 %0, {%1, %1};" : "=l"(r) : "f"(x));
  return r;
}
// packed fp32x2 FMA (sm_100 FFMA2): one issue slot for both halves
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

// 4x4 gate on cube bits (LA = in_a < LB = in_b) of a 32-element register
// cube.  acc += u * x is two FFMA2 whose coefficient operands come from
// uniform registers (the constant bank, warp-uniform gate index) and whose
// half swaps are operand modifiers -- no moves, no negations:
//   acc += (u.re, u.re) * (x.re, x.im) + (-u.im, u.im) * (x.im, x.re)
template <int LA, int LB>
__device__ __forceinline__ void apply_local(float2 (&v)[kCube], const float* u) {
#pragma unroll
  for (int s = 0; s < kCube; ++s) {
    if ((s >> LA) & 1) continue;
    if ((s >> LB) & 1) continue;
    const int idx[4] = {s, s | (1 << LB), s | (1 << LA), s | (1 << LA) | (1 << LB)};
    u64 x[4], xs[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      x[i] = as_u64(v[idx[i]]);
      xs[i] = as_u64(make_float2(v[idx[i]].y, v[idx[i]].x));
    }
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      u64 acc = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float2 ci = reinterpret_cast<const float2*>(u)[o * 4 + i];
        acc = ffma2(bcast(u[32 + o * 4 + i]), x[i], acc);
        acc = ffma2(as_u64(ci), xs[i], acc);
      }
      v[idx[o]] = as_f2(acc);
    }
  }
}

__device__ __forceinline__ void apply_gate(float2 (&v)[kCube], int local, const float* u) {
  switch (local) {
    case 8 * 0 + 1: apply_local<0, 1>(v, u); break;
    case 8 * 0 + 2: apply_local<0, 2>(v, u); break;
    case 8 * 0 + 3: apply_local<0, 3>(v, u); break;
    case 8 * 0 + 4: apply_local<0, 4>(v, u); break;
    case 8 * 1 + 2: apply_local<1, 2>(v, u); break;
    case 8 * 1 + 3: apply_local<1, 3>(v, u); break;
    case 8 * 1 + 4: apply_local<1, 4>(v, u); break;
    case 8 * 2 + 3: apply_local<2, 3>(v, u); break;
    case 8 * 2 + 4: apply_local<2, 4>(v, u); break;
    case 8 * 3 + 4: apply_local<3, 4>(v, u); break;
    default: break;
  }
}

// Gate tables from the caller's device gate tensors (one thread per entry).
__global__ void absorb_table_kernel(const TableParams p, float* __restrict__ table) {
  const int j = blockIdx.x;
  const int e = threadIdx.x;  // 16 entries
  if (j >= p.n || e >= 16) return;
  const int g = p.src[j];
  const int o = e >> 2, i = e & 3;
  auto q = [&](int x) { return p.swap[j] ? (((x & 1) << 1) | (x >> 1)) : x; };
  const int oo = q(o), ii = q(i);
  const int64_t* st = p.gstride[g];
  const float2 u = p.gate[g][(oo >> 1) * st[0] + (oo & 1) * st[1] + (ii >> 1) * st[2] + (ii & 1) * st[3]];
  float* g_out = table + kGateFloats * j;
  g_out[2 * e] = -u.y;
  g_out[2 * e + 1] = u.y;
  g_out[32 + e] = u.x;
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
// ring of 3 tile buffers (192 KB of smem); tile k of the CTA lives in buffer
// k % 3 and belongs to math team k % 2:
//   memory warps (4):  step k = cp.async gather of tile k (HBM -> smem, 8-byte
//                      elements, completion tracked by mbarrier full[b]), then
//                      the store of tile k-2 (smem -> HBM in the output layout)
//                      once its team released it (computed[b]), then empty[b];
//   math teams (2 x 8 warps): the pass's gate groups on 32-element register
//                      cubes, one team barrier per group.
// While one team regroups its tile through shared memory the other team's
// FFMA2s have the FP32 pipe, and the loads / stores of two more tiles overlap.
__global__ void __launch_bounds__(kThreads, 1) absorb_pass_kernel(const float2* __restrict__ in,
                                                                   float2* __restrict__ out,
                                                                   const AbsorbParams p) {
  extern __shared__ __align__(16) float2 tiles[];  // kBufs x kTile
  __shared__ __align__(8) uint64_t full[kBufs], computed[kBufs], empty[kBufs], stagger;
  __shared__ int64_t s_oin[TNC_MAX_RANK], s_oout[TNC_MAX_RANK];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  // warp-uniform by construction, and visibly so to the compiler: the role
  // branches are then convergent and the gate coefficients can ride the
  // uniform datapath
  const int warp = __shfl_sync(0xffffffffu, tid >> 5, 0);
  if (tid < p.n_outer) {
    s_oin[tid] = p.outer_in[tid];
    s_oout[tid] = p.outer_out[tid];
  }
  if (tid == 0) {
    for (int b = 0; b < kBufs; ++b) {
      mbar_init(&full[b], kMemThreads);
      mbar_init(&computed[b], 1);
      mbar_init(&empty[b], kMemThreads);
    }
    mbar_init(&stagger, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (warp >= kMathThreads / 32) {
    // ---- memory warps (one warpgroup): hand registers to the math warpgroups
    asm volatile("setmaxnreg.dec.sync.aligned.u32 32;");
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
      if (t < p.n_tiles) {
        const int b = static_cast<int>(k % kBufs);
        if (k >= kBufs) mbar_wait(&empty[b], static_cast<uint32_t>((k / kBufs - 1) & 1));
        const float2* src = in + tile_base(t, s_oin, p.n_outer, lane) + my_in;
        const uint32_t dst = tiles_s + b * kTile * 8;
#pragma unroll 16
        for (int i = 0; i < kMemPer; ++i) cp_async8(dst + ((my_in_slot ^ p.in_slot_i[i]) << 3), src + p.in_i[i]);
        cp_async_arrive(&full[b]);
      }
      if (k >= p.teams) {
        const int64_t kp = k - p.teams;
        const int64_t tp = blockIdx.x + kp * gridDim.x;
        if (tp >= p.n_tiles) break;
        const int bp = static_cast<int>(kp % kBufs);
        mbar_wait(&computed[bp], static_cast<uint32_t>((kp / kBufs) & 1));
        const float2* tile = tiles + bp * kTile;
        float2* dst = out + tile_base(tp, s_oout, p.n_outer, lane) + my_out;
#pragma unroll 16
        for (int i = 0; i < kMemPer; ++i) __stcs(dst + p.out_i[i], tile[my_out_slot ^ p.out_slot_i[i]]);
        mbar_arrive(&empty[bp]);
      }
    }
  } else {
    // ---- math teams (warpgroups 0-3): 640 x 96 registers at launch, 512 x 112 + 128 x 40 now
    asm volatile("setmaxnreg.inc.sync.aligned.u32 112;");
    const int team = warp >> 3;
    const int tw = warp & 7;
    // Team 1 starts half a tile behind team 0 (released when team 0 is half
    // way through the groups of its first tile) and the teams stay in
    // anti-phase from there: nothing else would separate them, and two teams
    // in phase regroup at the same time and do their math at the same time.
    if (team >= p.teams) return;
    if (team == 1) mbar_wait(&stagger, 0);
    for (int64_t k = team;; k += p.teams) {
      const int64_t t = blockIdx.x + k * gridDim.x;
      if (t >= p.n_tiles) break;
      const int b = static_cast<int>(k % kBufs);
      mbar_wait(&full[b], static_cast<uint32_t>((k / kBufs) & 1));
      // the buffer's byte offset (a multiple of 64 KB) rides in the running XOR
      // with the in-tile offsets, so an element address is one LOP3
      char* tile_b = reinterpret_cast<char*>(tiles);
      const uint32_t buf_off = static_cast<uint32_t>(b) * (kTile * 8u);
      for (int g = 0; g < p.n_groups; ++g) {
        const GroupParams& gp = p.g[g];
        // byte offsets inside the tile buffer: the running XOR is the whole
        // per-element address arithmetic (the buffer base is uniform)
        uint32_t base = buf_off;
#pragma unroll
        for (int j = 0; j < 5; ++j)
          if ((lane >> j) & 1) base ^= static_cast<uint32_t>(gp.lane_slot[j]) << 3;
#pragma unroll
        for (int j = 0; j < 3; ++j)
          if ((tw >> j) & 1) base ^= static_cast<uint32_t>(gp.warp_slot[j]) << 3;
        uint32_t sb[kCubeBits];
#pragma unroll
        for (int j = 0; j < kCubeBits; ++j) sb[j] = static_cast<uint32_t>(gp.cube_slot[j]) << 3;
        // cube elements in Gray-code order: one running offset, one XOR with a
        // uniform slot vector per element (no table of 32 addresses kept live)
        float2 c[kCube];
        uint32_t a = base;
#pragma unroll
        for (int n = 0; n < kCube; ++n) {
          if (n > 0) a ^= sb[ctz5(n)];
          c[n ^ (n >> 1)] = *reinterpret_cast<const float2*>(tile_b + a);
        }
        for (int k2 = gp.g_first; k2 < gp.g_last; ++k2) apply_gate(c, p.gate_local[k2], c_gates + kGateFloats * k2);
        asm volatile("mov.b32 %0, %1;" : "=r"(a) : "r"(base));  // recompute, do not keep, the addresses
#pragma unroll
        for (int n = 0; n < kCube; ++n) {
          if (n > 0) a ^= sb[ctz5(n)];
          *reinterpret_cast<float2*>(tile_b + a) = c[n ^ (n >> 1)];
        }
        // team barrier (ids 1, 2): the next group's cubes cross the team's warps
        if (team == 0) asm volatile("bar.sync 1, %0;" ::"n"(kTeamThreads) : "memory");
        else asm volatile("bar.sync 2, %0;" ::"n"(kTeamThreads) : "memory");
        if (k == 0 && tid == 0 && g == (p.n_groups - 1) / 2) mbar_arrive(&stagger);
      }
      if (k == 0 && tid == 0 && p.n_groups == 0) mbar_arrive(&stagger);
      if ((tid & (kTeamThreads - 1)) == 0) mbar_arrive(&computed[b]);
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
    // groups of <= 5 axes (same deferral rule); groups beyond kMaxGroups
    // (or gates beyond kMaxPassGates) go back to the remaining gates (the
    // first k groups are a dependency-closed prefix of the pass's gates)
    {
      std::vector<int> todo2 = ps.gates;
      int n_in = 0;
      while (!todo2.empty()) {
        std::vector<int> axes, rest2;
        std::vector<int> grp = pack(gates, todo2, axes, kCubeBits, rest2);
        if (static_cast<int>(ps.groups.size()) == kMaxGroups ||
            n_in + static_cast<int>(grp.size()) > kMaxPassGates) {
          rest.insert(rest.end(), todo2.begin(), todo2.end());
          std::sort(rest.begin(), rest.end());
          break;
        }
        n_in += static_cast<int>(grp.size());
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

// group_local: (chain gate index, swap) of the pass's gates in table order
int build_pass_params(int r, const Pass& ps, const std::vector<GateRef>& gates_of_pass, const std::vector<int>& bit_axis,
                      const std::vector<int64_t>& in_st, const std::vector<int64_t>& out_st, int table_base,
                      AbsorbParams& p, std::vector<std::pair<int, int>>& group_local) {
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
  p.table_base = table_base;
  {
    const char* e = std::getenv("TNC_ABSORB_TEAMS");
    p.teams = (e && std::atoi(e) == 1) ? 1 : kTeams;
  }
  // each group: 5 cube bits (its axes + padding), 5 lane bits (the first 4
  // of distinct bank classes), 3 warp bits; gates oriented so in_a is the
  // lower cube bit
  group_local.clear();
  p.n_gates = 0;
  for (int g = 0; g < p.n_groups; ++g) {
    auto cl = [](int b) { return b & 3; };
    std::vector<int> cube;
    for (int a : ps.gaxes[g]) cube.push_back(pos[a]);
    std::vector<int> rest_bits;
    for (int b = 0; b < kTB; ++b)
      if (!has(cube, b)) rest_bits.push_back(b);
    // lane bits 0..3 of distinct classes from the non-cube bits, chosen first so
    // the padding cube bits do not take them
    std::vector<int> lanes;
    for (int c = 0; c < 4; ++c)
      for (int b : rest_bits)
        if (cl(b) == c && !has(lanes, b)) {
          lanes.push_back(b);
          break;
        }
    std::vector<int> free_bits;
    for (int b : rest_bits)
      if (!has(lanes, b)) free_bits.push_back(b);
    size_t fi = 0;
    while (static_cast<int>(cube.size()) < kCubeBits) cube.push_back(free_bits[fi++]);
    while (lanes.size() < 5) lanes.push_back(free_bits[fi++]);
    std::vector<int> warps(free_bits.begin() + fi, free_bits.end());
    GroupParams& gp = p.g[g];
    for (int j = 0; j < kCubeBits; ++j) gp.cube_slot[j] = swz(1 << cube[j]);
    for (int j = 0; j < 5; ++j) gp.lane_slot[j] = swz(1 << lanes[j]);
    for (int j = 0; j < 3; ++j) gp.warp_slot[j] = swz(1 << warps[j]);
    gp.g_first = p.n_gates;
    for (int gi : ps.groups[g]) {
      auto ci = [&](int axis) {
        return static_cast<int>(std::find(cube.begin(), cube.end(), pos[axis]) - cube.begin());
      };
      int la = ci(gates_of_pass[gi].pa), lb = ci(gates_of_pass[gi].pb);
      const bool swap = la > lb;
      if (swap) std::swap(la, lb);
      p.gate_local[p.n_gates++] = 8 * la + lb;
      group_local.push_back({gi, swap ? 1 : 0});
    }
    gp.g_last = p.n_gates;
    if (std::getenv("TNC_ABSORB_DEBUG"))
      std::fprintf(stderr, "  group %d: %zu gates, %zu axes, lane classes %d %d %d %d\n", g, ps.groups[g].size(),
                   ps.gaxes[g].size(), cl(lanes[0]), cl(lanes[1]), cl(lanes[2]), cl(lanes[3]));
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
  return TNC_OK;
}

// gate tables: 48 floats per gate
size_t table_bytes(int n_gates) {
  return (static_cast<size_t>(std::max(n_gates, 1)) * kGateFloats * sizeof(float) + 255) & ~size_t(255);
}

// c_gates is one per device: chains launched on different streams take turns
// (the later stream waits for the earlier chain's last pass).
struct ConstOwner {
  cudaStream_t stream = nullptr;
  cudaEvent_t done = nullptr;
  bool used = false;
};
std::mutex g_const_mu;
ConstOwner g_const_owner[64];

}  // namespace

int absorb_chain_workspace(int t_rank, int n_gates, const int32_t* axes, size_t* bytes) {
  ChainPlan cp;
  TNC_TRY(plan_chain(t_rank, n_gates, axes, cp));
  const size_t tensor = cp.passes.size() > 1 ? (static_cast<size_t>(1) << t_rank) * sizeof(float2) : 0;
  *bytes = tensor + table_bytes(n_gates);
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
  if (workspace_bytes < tensor + table_bytes(n_gates) || workspace == nullptr)
    TNC_RET(TNC_ERR_WORKSPACE, "absorb: workspace too small (see tnc_absorb_chain_workspace)");
  for (int g = 0; g < n_gates; ++g)
    if (gates[g] == nullptr) TNC_RET(TNC_ERR_INVALID, "absorb: null gate pointer");
  float2* ws = static_cast<float2*>(workspace);
  float* table = reinterpret_cast<float*>(static_cast<uint8_t*>(workspace) + tensor);

  std::vector<AbsorbParams> params(P);
  TableParams tp;
  std::memset(&tp, 0, sizeof(tp));
  int base = 0;
  for (int k = 0; k < P; ++k) {
    const Pass& ps = cp.passes[k];
    std::vector<std::pair<int, int>> gl;
    TNC_TRY(build_pass_params(r, ps, cp.refs, place_bits(ps.tile, cp.in_st[k], cp.out_st[k]), cp.in_st[k],
                              cp.out_st[k], base, params[k], gl));
    for (const auto& e : gl) {
      tp.src[base] = static_cast<short>(e.first);
      tp.swap[base] = static_cast<signed char>(e.second);
      ++base;
    }
  }
  tp.n = base;
  for (int g = 0; g < n_gates; ++g) {
    tp.gate[g] = static_cast<const float2*>(gates[g]);
    for (int k = 0; k < 4; ++k) tp.gstride[g][k] = gate_strides[4 * g + k];
  }
  if (tp.n > 0) {
    absorb_table_kernel<<<tp.n, 16, 0, stream>>>(tp, table);
    TNC_CHECK_LAUNCH();
  }
  const size_t smem = static_cast<size_t>(kBufs) * kTile * sizeof(float2);
  TNC_CUDA_TRY(cudaFuncSetAttribute(absorb_pass_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(smem)));
  int dev = 0;
  TNC_CUDA_TRY(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) TNC_RET(TNC_ERR_UNSUPPORTED, "absorb: device index out of range");
  std::lock_guard<std::mutex> lock(g_const_mu);
  ConstOwner& owner = g_const_owner[dev];
  if (!owner.done) TNC_CUDA_TRY(cudaEventCreateWithFlags(&owner.done, cudaEventDisableTiming));
  if (owner.used && owner.stream != stream) TNC_CUDA_TRY(cudaStreamWaitEvent(stream, owner.done, 0));
  const float2* cur = static_cast<const float2*>(t_in);
  for (int k = 0; k < P; ++k) {
    float2* dst = ((P - 1 - k) % 2 == 0) ? static_cast<float2*>(t_out) : ws;
    const AbsorbParams& p = params[k];
    const int64_t blocks = std::min<int64_t>(p.n_tiles, static_cast<int64_t>(num_sms()));
    if (p.n_gates > 0)
      TNC_CUDA_TRY(cudaMemcpyToSymbolAsync(c_gates, table + kGateFloats * p.table_base,
                                           static_cast<size_t>(p.n_gates) * kGateFloats * sizeof(float), 0,
                                           cudaMemcpyDeviceToDevice, stream));
    {
      // algorithmic work: 16 complex MACs (64 real flops) per 4 elements per gate
      ProfScope prof(PROF_ABSORB, 32.0 * p.n_gates * static_cast<double>(int64_t(1) << r),
                     16.0 * static_cast<double>(int64_t(1) << r), stream);
      absorb_pass_kernel<<<static_cast<unsigned>(blocks), kThreads, smem, stream>>>(cur, dst, p);
      TNC_CHECK_LAUNCH();
    }
    cur = dst;
  }
  TNC_CUDA_TRY(cudaEventRecord(owner.done, stream));
  owner.stream = stream;
  owner.used = true;
  return TNC_OK;
}

// tnc_shutdown: drop the events that order streams on the constant table
void absorb_shutdown() {
  std::lock_guard<std::mutex> lock(g_const_mu);
  for (ConstOwner& o : g_const_owner) {
    if (o.done) cudaEventDestroy(o.done);
    o = ConstOwner{};
  }
}

int absorb_chain_passes(int t_rank, int n_gates, const int32_t* axes, int* passes, int* groups) {
  ChainPlan cp;
  TNC_TRY(plan_chain(t_rank, n_gates, axes, cp));
  *passes = static_cast<int>(cp.passes.size());
  *groups = cp.total_groups;
  if (std::getenv("TNC_ABSORB_DEBUG")) {  // print the bit placement of every pass
    AbsorbParams* prm = new AbsorbParams;
    for (size_t k = 0; k < cp.passes.size(); ++k) {
      std::vector<std::pair<int, int>> gl;
      build_pass_params(t_rank, cp.passes[k], cp.refs, place_bits(cp.passes[k].tile, cp.in_st[k], cp.out_st[k]),
                        cp.in_st[k], cp.out_st[k], 0, *prm, gl);
    }
    delete prm;
  }
  return TNC_OK;
}

}  // namespace tnc
