// K4: step fusion -- a chain of two-leg gate absorptions into one resident
// tensor in as few HBM passes as the on-chip tile allows.
//
// Reference semantics: successive contract_pair(T, G) along a stem
// (execute.py:150-173 over tree.py:278-384 stems; contract.py:149-165):
// gate g = (out_a, out_b, in_a, in_b) contracts T's legs at logical
// positions axes[2g] (in_a) and axes[2g+1] (in_b); the two legs leave the
// order and (out_a, out_b) are appended at the end.
//
// B200 design.  The data never moves between gates: logical legs map onto
// fixed physical axes (out_a lands on in_a's axis).  Gates are grouped into
// sections whose touched axes, plus the 3 input-fastest axes (coalescing), fit
// one shared-memory tile of 2^12 elements; each section is one pass
//   HBM -> smem tile (coalesced) -> apply the section's 4x4 unitaries in smem
//   -> HBM (same layout; the LAST pass stores in the final logical order)
// so a 16-gate chain on a rank-30 tensor costs ~4 passes instead of 16
// permute+GEMM round trips.  Index maps are 2-level bit tables (all dims 2).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "tnc_common.cuh"

namespace tnc {

namespace {

constexpr int kTileBits = 12;              // 4096 complex64 = 32 KB tile
constexpr int kTile = 1 << kTileBits;
constexpr int kMaxSectionGates = 16;
constexpr int kCubeBits = 5;               // register cube: 32 complex per thread
constexpr int kCube = 1 << kCubeBits;
constexpr int kThreadBits = kTileBits - kCubeBits;
constexpr int kThreadsAbs = 1 << kThreadBits;  // one cube per thread in the gate phase

// Gates of a section are applied in groups whose legs span <= 5 tile bits: a
// thread keeps the 32-element sub-cube in registers and applies every gate of
// the group before writing it back (2 shared-memory round trips per group
// instead of 2 per gate).
struct AbsorbParams {
  int n_outer;
  int n_groups;
  int64_t n_tiles;
  // 2-level tables over the tile index (low 6 bits / high 6 bits)
  int64_t in_lo[64], in_hi[64];    // input element offset of load index e
  int64_t out_lo[64], out_hi[64];  // output element offset of store index f
  int src_lo[64], src_hi[64];      // swizzled smem slot of store index f (XOR halves)
  // swizzled smem slot of each sub-cube bit (register index bit j) and of each
  // thread-index bit (cube base) of a group; all other slots are XORs of these
  int group_cube[kMaxSectionGates][kCubeBits];
  int group_lane[kMaxSectionGates][kThreadBits];
  int group_gates[kMaxSectionGates][2];         // [first gate, last gate) of the group
  int gate_local[kMaxSectionGates];             // 8 * (local bit of in_a) + local bit of in_b, a < b
  float4 u[kMaxSectionGates][16];  // U[(oa,ob),(ia,ib)] row-major as (re, im, -im, re)
  int outer_shift[TNC_MAX_RANK];   // outer axis digit = (t >> shift) & 1
  int64_t outer_in[TNC_MAX_RANK];
  int64_t outer_out[TNC_MAX_RANK];
};

// XOR swizzle of the smem tile: 8-byte elements, 16 per 128-byte bank row.
// Gate-group accesses step the tile index by powers of two; folding bits
// 4..11 into the low nibble spreads those strides over the 16 bank slots
// (ncu: ~75% of shared wavefronts were bank conflicts without it).  swz is
// linear over GF(2): swz(x ^ y) = swz(x) ^ swz(y), so a cube's 32 slots are
// one per-thread base XOR a per-group pattern.
__host__ __device__ __forceinline__ int swz(int e) { return e ^ (((e >> 4) ^ (e >> 8)) & 15); }

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

// acc += u * x as two FFMA2: (x.re, x.re) * (u.re, u.im) + (x.im, x.im) * (-u.im, u.re)
__device__ __forceinline__ u64 cmac(u64 acc, float4 u, float2 x) {
  acc = ffma2(bcast(x.x), as_u64(make_float2(u.x, u.y)), acc);
  return ffma2(bcast(x.y), as_u64(make_float2(u.z, u.w)), acc);
}

// 4x4 gate on local bits (LA = in_a < LB = in_b) of a 32-element register cube
template <int LA, int LB>
__device__ __forceinline__ void apply_local(float2 (&v)[kCube], const float4* __restrict__ u) {
#pragma unroll
  for (int s = 0; s < kCube; ++s) {
    if ((s >> LA) & 1) continue;
    if ((s >> LB) & 1) continue;
    const int i1 = s | (1 << LB), i2 = s | (1 << LA), i3 = s | (1 << LA) | (1 << LB);
    const float2 x0 = v[s], x1 = v[i1], x2 = v[i2], x3 = v[i3];
    u64 y[4];
#pragma unroll
    for (int o = 0; o < 4; ++o) {
      u64 acc = 0;
      acc = cmac(acc, u[o * 4 + 0], x0);
      acc = cmac(acc, u[o * 4 + 1], x1);
      acc = cmac(acc, u[o * 4 + 2], x2);
      acc = cmac(acc, u[o * 4 + 3], x3);
      y[o] = acc;
    }
    v[s] = as_f2(y[0]);
    v[i1] = as_f2(y[1]);
    v[i2] = as_f2(y[2]);
    v[i3] = as_f2(y[3]);
  }
}

// The host orients every gate so that its in_a bit is the lower local bit
// (U transposed accordingly), leaving 10 (a < b) cases.
__device__ __forceinline__ void apply_gate(float2 (&v)[kCube], int local, const float4* __restrict__ u) {
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

__device__ __forceinline__ void cp_async8(uint32_t smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_dst), "l"(gmem_src) : "memory");
}

// One pass: tiles of 2^12 elements stream HBM -> smem (cp.async, coalesced
// along the input-fastest axes), the section's gates run on 32-element
// register cubes (one per thread, FFMA2), and the tile leaves smem in the
// output order.  NBUF = 2 overlaps the next tile's loads with this tile's
// gates inside the block (3 blocks/SM: slower); NBUF = 1 relies on
// co-resident blocks for that; NBUF = 3 (default) is NBUF = 1 with the next
// tile's loads issued as soon as the tile sits in registers, before its
// stores (C2 16.7 -> 16.4 ms).
template <int NBUF>
__global__ void __launch_bounds__(kThreadsAbs) absorb_pass_kernel(const float2* __restrict__ in,
                                                                  float2* __restrict__ out,
                                                                  const AbsorbParams p) {
  extern __shared__ __align__(16) float2 tiles[];  // NBUF x kTile
  // tile bases ring-indexed by iteration: a fast warp decoding tile i+1 can
  // never overwrite a base a slow warp still reads (it passed iteration i's barrier)
  __shared__ int64_t s_base[4][2];
  // per-element table lookups must not hit the (serialising) param/constant
  // bank with divergent addresses: stage the tables in shared memory
  __shared__ int64_t s_oin[TNC_MAX_RANK], s_oout[TNC_MAX_RANK];
  __shared__ int s_oshift[TNC_MAX_RANK];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  if (tid < p.n_outer) {
    s_oin[tid] = p.outer_in[tid];
    s_oout[tid] = p.outer_out[tid];
    s_oshift[tid] = p.outer_shift[tid];
  }
  // element e = tid + kThreadsAbs * i: its low 6 bits are the thread's own
  // (kThreadsAbs is a multiple of 64), its high 6 bits are (tid >> 6) + 2 i
  // high-table entry (tid >> 6) + 2 i splits into a per-thread part (bit 0)
  // and a uniform part (bits 1-5) read as constant-bank operands: the maps are
  // sums (offsets) / XORs (swizzled slots) of per-bit terms
  const int64_t my_in_lo = p.in_lo[tid & 63] + p.in_hi[tid >> 6];
  const int my_swz = swz(tid);
  const int64_t my_out_lo = p.out_lo[tid & 63] + p.out_hi[tid >> 6];
  const int my_src_lo = p.src_lo[tid & 63] ^ p.src_hi[tid >> 6];
  const uint32_t tiles_s = static_cast<uint32_t>(__cvta_generic_to_shared(tiles));
  __syncthreads();
  constexpr int kPer = kTile / kThreadsAbs;
  static_assert(kPer == kCube, "one cube per thread");
  auto decode = [&](int64_t t, int slot) {
    if (tid < 32) {
      int64_t bi = 0, bo = 0;
      for (int a = lane; a < p.n_outer; a += 32) {
        const int64_t d = (t >> s_oshift[a]) & 1;
        bi += d * s_oin[a];
        bo += d * s_oout[a];
      }
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        bi += __shfl_xor_sync(0xffffffffu, bi, s);
        bo += __shfl_xor_sync(0xffffffffu, bo, s);
      }
      if (lane == 0) {
        s_base[slot][0] = bi;
        s_base[slot][1] = bo;
      }
    }
  };
  auto issue_loads = [&](int slot, int bslot) {
    const float2* src = in + s_base[bslot][0] + my_in_lo;
    const uint32_t dst = tiles_s + slot * kTile * 8;
#pragma unroll
    for (int i = 0; i < kPer; ++i)
      cp_async8(dst + ((my_swz ^ swz(kThreadsAbs * i)) << 3), src + p.in_hi[2 * i]);
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  int slot = 0, it = 0;
  if (NBUF >= 2 && blockIdx.x < p.n_tiles) {
    decode(blockIdx.x, 0);
    __syncthreads();
    issue_loads(0, 0);
  }
  for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it) {
    if (NBUF == 2) {
      const int64_t tn = t + gridDim.x;
      if (tn < p.n_tiles) decode(tn, (it + 1) & 3);
      __syncthreads();  // next base visible; previous store phase done with slot ^ 1
      if (tn < p.n_tiles) {
        issue_loads(slot ^ 1, (it + 1) & 3);
        asm volatile("cp.async.wait_group 1;" ::: "memory");
      } else {
        asm volatile("cp.async.wait_group 0;" ::: "memory");
      }
    } else if (NBUF == 3) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");  // issued at the end of the previous tile
    } else {
      decode(t, it & 3);
      __syncthreads();  // base visible; previous store phase done with the tile
      issue_loads(0, it & 3);
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // tile t resident
    float2* tile = tiles + slot * kTile;
    float2* dst = out + s_base[it & 3][1] + my_out_lo;
    float2 c[kCube];
    for (int g = 0; g < p.n_groups; ++g) {
      int sb[kCubeBits];
#pragma unroll
      for (int j = 0; j < kCubeBits; ++j) sb[j] = p.group_cube[g][j];
      int b0 = 0;
#pragma unroll
      for (int j = 0; j < kThreadBits; ++j)
        if ((tid >> j) & 1) b0 ^= p.group_lane[g][j];
#pragma unroll
      for (int s = 0; s < kCube; ++s) {
        int a = b0;
#pragma unroll
        for (int j = 0; j < kCubeBits; ++j)
          if ((s >> j) & 1) a ^= sb[j];
        c[s] = tile[a];
      }
      for (int k = p.group_gates[g][0]; k < p.group_gates[g][1]; ++k) apply_gate(c, p.gate_local[k], p.u[k]);
#pragma unroll
      for (int s = 0; s < kCube; ++s) {
        int a = b0;
#pragma unroll
        for (int j = 0; j < kCubeBits; ++j)
          if ((s >> j) & 1) a ^= sb[j];
        tile[a] = c[s];
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) c[i] = tile[my_src_lo ^ p.src_hi[2 * i]];
    if (NBUF == 3) {
      // the tile is in registers: start the next tile's loads before the stores
      const int64_t tn = t + gridDim.x;
      if (tn < p.n_tiles) decode(tn, (it + 1) & 3);
      __syncthreads();  // every thread has read the tile; next base visible
      if (tn < p.n_tiles) issue_loads(0, (it + 1) & 3);
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) dst[p.out_hi[2 * i]] = c[i];
    if (NBUF == 2) slot ^= 1;
  }
  if (NBUF == 2) asm volatile("cp.async.wait_group 0;" ::: "memory");
}

struct GateRef {
  int pa, pb;  // physical axes of in_a, in_b
  const void* u;
};

// Host plan: physical axis i (0 = most significant) has stride 2^(r-1-i).
struct Section {
  std::vector<int> gates;  // indices into the gate list
  std::vector<int> axes;   // physical tile axes
};

int plan_sections(int r, const std::vector<GateRef>& gates, const std::vector<int>& final_lorder,
                  std::vector<Section>& out) {
  const int reserve_in = std::min(3, r);
  auto fast_in = [&](std::vector<int>& s) {
    for (int i = 0; i < reserve_in; ++i) s.push_back(r - 1 - i);
  };
  out.clear();
  Section cur;
  fast_in(cur.axes);
  auto add_axes = [](std::vector<int> s, int a, int b) {
    if (std::find(s.begin(), s.end(), a) == s.end()) s.push_back(a);
    if (std::find(s.begin(), s.end(), b) == s.end()) s.push_back(b);
    return s;
  };
  for (size_t g = 0; g < gates.size(); ++g) {
    std::vector<int> trial = add_axes(cur.axes, gates[g].pa, gates[g].pb);
    if (static_cast<int>(trial.size()) > kTileBits ||
        static_cast<int>(cur.gates.size()) >= kMaxSectionGates) {
      out.push_back(cur);
      cur = Section();
      fast_in(cur.axes);
      trial = add_axes(cur.axes, gates[g].pa, gates[g].pb);
    }
    cur.axes = trial;
    cur.gates.push_back(static_cast<int>(g));
  }
  out.push_back(cur);
  // the last pass stores in the final order: its tile also needs the 3
  // output-fastest axes; split its gates off into a new pass if they do not fit
  std::vector<int> fast_out;
  for (int i = 0; i < std::min(3, r); ++i) fast_out.push_back(final_lorder[r - 1 - i]);
  Section& last = out.back();
  std::vector<int> with_out = last.axes;
  for (int a : fast_out)
    if (std::find(with_out.begin(), with_out.end(), a) == with_out.end()) with_out.push_back(a);
  if (static_cast<int>(with_out.size()) <= kTileBits) {
    last.axes = with_out;
  } else {
    Section fin;
    fin.axes = std::vector<int>();
    fast_in(fin.axes);
    for (int a : fast_out)
      if (std::find(fin.axes.begin(), fin.axes.end(), a) == fin.axes.end()) fin.axes.push_back(a);
    out.push_back(fin);  // pure permutation pass
  }
  // pad every tile to kTileBits axes (more work per block, coalescing)
  for (auto& sec : out) {
    for (int a = r - 1; a >= 0 && static_cast<int>(sec.axes.size()) < std::min(kTileBits, r); --a)
      if (std::find(sec.axes.begin(), sec.axes.end(), a) == sec.axes.end()) sec.axes.push_back(a);
  }
  return TNC_OK;
}

int launch_pass(int r, const Section& sec, const std::vector<GateRef>& gates, const float2* in,
                float2* out, const std::vector<int64_t>& out_stride, cudaStream_t stream) {
  const int nt = static_cast<int>(sec.axes.size());
  if (nt != kTileBits) TNC_RET(TNC_ERR_UNSUPPORTED, "absorb: tensor rank below tile size");
  AbsorbParams p{};
  // load enumeration: tile axes sorted by input stride ascending (physical axis descending)
  std::vector<int> ax_in = sec.axes;
  std::sort(ax_in.begin(), ax_in.end(), [](int x, int y) { return x > y; });
  std::vector<int> ax_out = sec.axes;
  std::sort(ax_out.begin(), ax_out.end(),
            [&](int x, int y) { return out_stride[x] < out_stride[y]; });
  auto in_stride = [&](int a) { return static_cast<int64_t>(1) << (r - 1 - a); };
  std::vector<int> bit_of(r, -1);
  for (int b = 0; b < nt; ++b) bit_of[ax_in[b]] = b;
  for (int i = 0; i < 64; ++i) {
    int64_t lo = 0, hi = 0, olo = 0, ohi = 0;
    int slo = 0, shi = 0;
    for (int b = 0; b < 6; ++b) {
      if (i & (1 << b)) {
        lo += in_stride(ax_in[b]);
        hi += in_stride(ax_in[b + 6]);
        olo += out_stride[ax_out[b]];
        ohi += out_stride[ax_out[b + 6]];
        slo |= 1 << bit_of[ax_out[b]];
        shi |= 1 << bit_of[ax_out[b + 6]];
      }
    }
    p.in_lo[i] = lo;
    p.in_hi[i] = hi;
    p.out_lo[i] = olo;
    p.out_hi[i] = ohi;
    p.src_lo[i] = swz(slo);  // swz is XOR-linear: swz(lo | hi) = swz(lo) ^ swz(hi)
    p.src_hi[i] = swz(shi);
  }
  // group consecutive gates whose legs span <= kCubeBits tile bits
  const int n_gates = static_cast<int>(sec.gates.size());
  std::vector<int> cur_bits;
  p.n_groups = 0;
  auto close_group = [&](int end) {
    if (cur_bits.empty()) return;
    // Bank conflicts: a 64-bit smem access is served per 16 lanes, and the
    // bank slot of tile bit t is (t mod 4) under swz; lanes 0..15 (thread bits
    // 0..3) must therefore sit on four tile bits of distinct t mod 4.  Pick
    // the cube's filler bits so that the remaining bits keep every class.
    std::vector<int> bits = cur_bits;
    auto in = [](const std::vector<int>& v, int x) { return std::find(v.begin(), v.end(), x) != v.end(); };
    while (static_cast<int>(bits.size()) < kCubeBits) {
      int best = -1, best_left = -1;
      for (int t = 0; t < kTileBits; ++t) {
        if (in(bits, t)) continue;
        int left = 0;  // free bits of t's class after taking t
        for (int u = 0; u < kTileBits; ++u)
          if (u != t && !in(bits, u) && (u & 3) == (t & 3)) ++left;
        if (left > best_left) best = t, best_left = left;
      }
      bits.push_back(best);
    }
    std::sort(bits.begin(), bits.end());
    std::vector<int> lanes;
    for (int cls = 0; cls < 4; ++cls)
      for (int t = 0; t < kTileBits; ++t)
        if (!in(bits, t) && !in(lanes, t) && (t & 3) == cls) {
          lanes.push_back(t);
          break;
        }
    for (int t = 0; t < kTileBits; ++t)
      if (!in(bits, t) && !in(lanes, t)) lanes.push_back(t);
    const int g = p.n_groups;
    for (int i = 0; i < kCubeBits; ++i) p.group_cube[g][i] = swz(1 << bits[i]);
    for (int i = 0; i < kThreadBits; ++i) p.group_lane[g][i] = swz(1 << lanes[i]);
    p.group_gates[g][1] = end;
    for (int k = p.group_gates[g][0]; k < end; ++k) {
      const GateRef& gr = gates[sec.gates[k]];
      int la = static_cast<int>(std::find(bits.begin(), bits.end(), bit_of[gr.pa]) - bits.begin());
      int lb = static_cast<int>(std::find(bits.begin(), bits.end(), bit_of[gr.pb]) - bits.begin());
      float2 u[16];
      std::memcpy(u, gr.u, sizeof(u));  // host gate data baked into the launch
      // orient the gate so in_a is the lower local bit: swapping the roles of
      // (a, b) transposes both the output and the input index pair of U
      const bool swap = la > lb;
      if (swap) std::swap(la, lb);
      auto q = [&](int x) { return swap ? (((x & 1) << 1) | (x >> 1)) : x; };
      for (int o = 0; o < 4; ++o)
        for (int i = 0; i < 4; ++i) {
          const float2 e = u[q(o) * 4 + q(i)];
          p.u[k][o * 4 + i] = make_float4(e.x, e.y, -e.y, e.x);
        }
      p.gate_local[k] = 8 * la + lb;
    }
    ++p.n_groups;
    cur_bits.clear();
  };
  for (int k = 0; k < n_gates; ++k) {
    const GateRef& gr = gates[sec.gates[k]];
    std::vector<int> trial = cur_bits;
    for (int b : {bit_of[gr.pa], bit_of[gr.pb]})
      if (std::find(trial.begin(), trial.end(), b) == trial.end()) trial.push_back(b);
    if (static_cast<int>(trial.size()) > kCubeBits) {
      close_group(k);
      trial = {bit_of[gr.pa], bit_of[gr.pb]};
    }
    if (cur_bits.empty()) p.group_gates[p.n_groups][0] = k;
    cur_bits = trial;
  }
  close_group(n_gates);
  // outer axes: physical axes not in the tile, enumerated least significant first
  std::vector<int> outer;
  for (int a = r - 1; a >= 0; --a)
    if (bit_of[a] < 0) outer.push_back(a);
  p.n_outer = static_cast<int>(outer.size());
  for (int i = 0; i < p.n_outer; ++i) {
    p.outer_shift[i] = i;
    p.outer_in[i] = in_stride(outer[i]);
    p.outer_out[i] = out_stride[outer[i]];
  }
  p.n_tiles = static_cast<int64_t>(1) << p.n_outer;
  ProfScope prof(PROF_ABSORB, 32.0 * n_gates * (static_cast<double>(1) * (int64_t(1) << r)),
                 16.0 * static_cast<double>(int64_t(1) << r), stream);
  static const int nbuf = [] {
    const char* e = std::getenv("TNC_ABSORB_NBUF");
    return e ? std::atoi(e) : 3;  // 3: one buffer, next tile's loads issued before the stores
  }();
  const size_t smem = static_cast<size_t>(nbuf == 2 ? 2 : 1) * kTile * sizeof(float2);
  const int per_sm = nbuf == 2 ? 3 : 4;  // smem (NBUF 2) or register (NBUF 1) limited residency
  const int64_t blocks = std::min<int64_t>(p.n_tiles, static_cast<int64_t>(num_sms()) * per_sm);
  if (nbuf == 2) {
    TNC_CUDA_TRY(cudaFuncSetAttribute(absorb_pass_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    absorb_pass_kernel<2><<<static_cast<unsigned>(blocks), kThreadsAbs, smem, stream>>>(in, out, p);
  } else if (nbuf == 3) {
    TNC_CUDA_TRY(cudaFuncSetAttribute(absorb_pass_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    absorb_pass_kernel<3><<<static_cast<unsigned>(blocks), kThreadsAbs, smem, stream>>>(in, out, p);
  } else {
    TNC_CUDA_TRY(cudaFuncSetAttribute(absorb_pass_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(smem)));
    absorb_pass_kernel<1><<<static_cast<unsigned>(blocks), kThreadsAbs, smem, stream>>>(in, out, p);
  }
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

}  // namespace

// Follow the reference's leg bookkeeping to physical axes; returns the final
// logical order (lorder[pos] = physical axis) and the pass sections.
int plan_chain(int r, int n_gates, const void* const* gates, const int32_t* axes,
               std::vector<GateRef>& refs, std::vector<int>& lorder, std::vector<Section>& secs) {
  if (r < kTileBits || r > TNC_MAX_RANK - 2)
    TNC_RET(TNC_ERR_UNSUPPORTED, "absorb: rank must be in [12, 62]");
  if (n_gates < 0) TNC_RET(TNC_ERR_INVALID, "absorb: negative gate count");
  lorder.resize(r);
  for (int i = 0; i < r; ++i) lorder[i] = i;
  refs.clear();
  for (int g = 0; g < n_gates; ++g) {
    const int pa = axes[2 * g], pb = axes[2 * g + 1];
    if (pa < 0 || pa >= r || pb < 0 || pb >= r || pa == pb)
      TNC_RET(TNC_ERR_CONTRACTION, "absorb: gate axes out of range");
    GateRef ref{lorder[pa], lorder[pb], gates ? gates[g] : nullptr};
    refs.push_back(ref);
    std::vector<int> next;
    for (int i = 0; i < r; ++i)
      if (i != pa && i != pb) next.push_back(lorder[i]);
    next.push_back(ref.pa);  // out_a occupies in_a's physical axis
    next.push_back(ref.pb);
    lorder.swap(next);
  }
  return plan_sections(r, refs, lorder, secs);
}

int absorb_chain_workspace(int t_rank, int n_gates, const int32_t* axes, size_t* bytes) {
  std::vector<GateRef> refs;
  std::vector<int> lorder;
  std::vector<Section> secs;
  TNC_TRY(plan_chain(t_rank, n_gates, nullptr, axes, refs, lorder, secs));
  *bytes = secs.size() > 1 ? (static_cast<size_t>(1) << t_rank) * sizeof(float2) : 0;
  return TNC_OK;
}

int absorb_chain_launch(int t_rank, const void* t_in, void* t_out, int n_gates,
                        const void* const* gates, const int32_t* axes, void* workspace,
                        size_t workspace_bytes, cudaStream_t stream) {
  const int r = t_rank;
  std::vector<GateRef> refs;
  std::vector<int> lorder;
  std::vector<Section> secs;
  TNC_TRY(plan_chain(r, n_gates, gates, axes, refs, lorder, secs));
  std::vector<int64_t> phys_stride(r), final_stride(r);
  for (int a = 0; a < r; ++a) phys_stride[a] = static_cast<int64_t>(1) << (r - 1 - a);
  for (int pos = 0; pos < r; ++pos) final_stride[lorder[pos]] = static_cast<int64_t>(1) << (r - 1 - pos);
  const size_t bytes = (static_cast<size_t>(1) << r) * sizeof(float2);
  if (secs.size() > 1 && workspace_bytes < bytes)
    TNC_RET(TNC_ERR_WORKSPACE, "absorb: workspace smaller than the tensor");
  const float2* cur = static_cast<const float2*>(t_in);
  float2* ws = static_cast<float2*>(workspace);
  for (size_t i = 0; i < secs.size(); ++i) {
    const bool last = i + 1 == secs.size();
    float2* dst = last ? static_cast<float2*>(t_out) : ws;
    TNC_TRY(launch_pass(r, secs[i], refs, cur, dst, last ? final_stride : phys_stride, stream));
    cur = ws;  // later passes read the workspace (in place for middle passes)
  }
  return TNC_OK;
}

}  // namespace tnc
