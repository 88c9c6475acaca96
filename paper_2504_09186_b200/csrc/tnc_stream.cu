// K5: narrow-step streaming contraction.  One pass over the large operand X
// in its own memory layout, the small operand Y resident on chip, and the
// result written straight into the requested output order -- the
// permute -> GEMM -> permute sequence of contract_pair (contract.py:131-165,
// tensor.py:252-274) for a step like C1a (M = 2^22, K = 2^6, N = 2^4), which
// is HBM-bound: 8 B in and 8*N/2^K B out per multiply-row.
//
// All legs have extent 2 (quantum-circuit networks), so every index map is a
// sum of per-bit strides and the tables below are 2-level (low 6 / high 6
// bits) like the absorb kernel's.
//
// A CTA owns a tile of R = 2^t rows of X (t X-free bits chosen to contain X's
// and the output's fastest free axes) times all K = 2^kb common bits:
//   load   R*K elements HBM -> smem, enumerated in X's stride order (coalesced)
//   math   thread (j, row group, k-slice): y = Y[j, slice] lives in registers,
//          X rows are broadcast 16-byte smem loads, FFMA2 complex MACs
//   reduce k-slice partials through smem
//   store  R*N outputs enumerated in the OUTPUT's stride order (coalesced)
#include <algorithm>
#include <cstring>
#include <vector>

#include "tnc_common.cuh"

namespace tnc {

namespace {

constexpr int kThreadsSt = 256;
constexpr int kMaxSlice = 16;  // complex K per thread slice (y kept in registers)
constexpr int kMaxRowsPer = 16;

struct StreamParams {
  int kb, t, g;            // log2 K, log2 R, log2 N
  int slices, groups;      // S k-slices, G row groups (N * S * G == kThreadsSt)
  int kpad;                // smem row pitch of the X tile (complex)
  int part_alias;          // k-slice partials reuse the X tile buffer
  int npitch;              // row pitch of the partials (N + 1: bank spread)
  int n_outer;
  int64_t n_tiles;
  int64_t in_lo[64], in_hi[64];    // X offset of load index e
  int pos_lo[64], pos_hi[64];      // smem slot (r * kpad + k) of load index e
  int64_t out_lo[64], out_hi[64];  // output offset of store index f
  int src_lo[64], src_hi[64];      // (r * npitch + j) of store index f
  int64_t yj[64];                  // Y offset of column j
  int64_t yk_lo[32], yk_hi[32];    // Y offset of common index k
  int64_t outer_x[TNC_MAX_RANK], outer_out[TNC_MAX_RANK];
};

typedef unsigned long long u64;

__device__ __forceinline__ u64 pack2(float a, float b) {
  u64 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 unpack2(u64 r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
__device__ __forceinline__ u64 ffma2(u64 a, u64 b, u64 c) {
  u64 r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
  return r;
}

__device__ __forceinline__ void cp_async8(uint32_t smem_dst, const void* gmem_src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_dst), "l"(gmem_src) : "memory");
}

// 128 registers (2 CTAs / SM); a 3-CTA register cap spills and measured 2x slower
template <int KS, int RP>
__global__ void __launch_bounds__(kThreadsSt, 2) stream_kernel(const float2* __restrict__ X,
                                                            const float2* __restrict__ Y,
                                                            float2* __restrict__ C,
                                                            const StreamParams p) {
  // smem: two X tile buffers [R][kpad] (cp.async double buffering) and the
  // k-slice partials [S][R][N], which alias the current X buffer once the
  // math is done when they fit (p.part_alias), else a third region.
  extern __shared__ __align__(16) float2 sm[];
  const int R = 1 << p.t, K = 1 << p.kb, N = 1 << p.g;
  const int buf_elems = R * p.kpad;
  // tile bases ring-indexed by iteration (see absorb_pass_kernel)
  __shared__ int64_t s_base[4][2];
  __shared__ int64_t s_ox[TNC_MAX_RANK], s_oo[TNC_MAX_RANK];
  const int tid = threadIdx.x;
  if (tid < p.n_outer) {
    s_ox[tid] = p.outer_x[tid];
    s_oo[tid] = p.outer_out[tid];
  }
  // thread roles: j fastest, then row group, then k-slice
  const int j = tid & (N - 1);
  const int grp = (tid >> p.g) % p.groups;
  const int slc = (tid >> p.g) / p.groups;
  // this thread's Y column slice, pre-arranged for FFMA2: (re) and (-im, im)
  float yre[KS];
  u64 yim[KS];
#pragma unroll
  for (int q = 0; q < KS; ++q) {
    const int k = slc * KS + q;
    float2 v = make_float2(0.f, 0.f);
    if (k < K) v = Y[p.yj[j] + p.yk_lo[k & 31] + p.yk_hi[k >> 5]];
    yre[q] = v.x;
    yim[q] = pack2(-v.y, v.y);
  }
  // element e = tid + 256 i: low 6 bits tid & 63, high 6 bits (tid >> 6) + 4 i.
  // The maps are sums of per-bit strides, so the high-table entry splits into
  // a per-thread part (bits 0-1) and a uniform part (bits 2-5) that the
  // unrolled loops read as constant-bank operands.
  const int hi0 = tid >> 6;
  const int64_t my_in = p.in_lo[tid & 63] + p.in_hi[hi0];
  const int my_pos = p.pos_lo[tid & 63] + p.pos_hi[hi0];
  const int64_t my_out = p.out_lo[tid & 63] + p.out_hi[hi0];
  const int my_src = p.src_lo[tid & 63] + p.src_hi[hi0];
  const int tile_elems = R * K, out_elems = R * N;
  const uint32_t sm_s = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
  auto decode = [&](int64_t t, int slot) {
    if (tid < 32) {
      int64_t bx = 0, bo = 0;
      for (int a = tid; a < p.n_outer; a += 32) {
        const int64_t d = (t >> a) & 1;
        bx += d * s_ox[a];
        bo += d * s_oo[a];
      }
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        bx += __shfl_xor_sync(0xffffffffu, bx, s);
        bo += __shfl_xor_sync(0xffffffffu, bo, s);
      }
      if (tid == 0) {
        s_base[slot][0] = bx;
        s_base[slot][1] = bo;
      }
    }
  };
  auto issue_loads = [&](int buf, int slot) {
    const float2* src = X + s_base[slot][0] + my_in;
    const uint32_t dst = sm_s + 8u * static_cast<uint32_t>(buf * buf_elems + my_pos);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (tid + i * kThreadsSt >= tile_elems) break;
      cp_async8(dst + 8u * static_cast<uint32_t>(p.pos_hi[4 * i]), src + p.in_hi[4 * i]);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  __syncthreads();
  int buf = 0, it = 0;
  if (blockIdx.x < p.n_tiles) {
    decode(blockIdx.x, 0);
    __syncthreads();
    issue_loads(0, 0);
  }
  for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x, ++it, buf ^= 1) {
    const int64_t tn = t + gridDim.x;
    if (tn < p.n_tiles) decode(tn, (it + 1) & 3);
    __syncthreads();  // next base visible; last iteration's store phase is done with buf ^ 1
    if (tn < p.n_tiles) {
      issue_loads(buf ^ 1, (it + 1) & 3);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();  // tile t resident
    const int64_t obase = s_base[it & 3][1];
    float2* xs = sm + buf * buf_elems;
    float2* part = p.part_alias ? xs : sm + 2 * buf_elems;
    // math: rows grp, grp + G, ... ; k in this thread's slice
    // RP rows per thread, compile-time: the whole block of row loads and
    // FFMA2 chains is straight-line code the scheduler can overlap
    float2 res[RP];
#pragma unroll
    for (int rr = 0; rr < RP; ++rr) {
      const int r = grp + rr * p.groups;
      const float4* xr = reinterpret_cast<const float4*>(xs + r * p.kpad + slc * KS);
      u64 acc0 = 0, acc1 = 0;
#pragma unroll
      for (int q = 0; q < KS; q += 2) {
        const float4 x2 = xr[q >> 1];
        // (x.re, x.im) * y.re + (x.im, x.re) * (-y.im, y.im)
        acc0 = ffma2(pack2(x2.x, x2.y), pack2(yre[q], yre[q]), acc0);
        acc1 = ffma2(pack2(x2.y, x2.x), yim[q], acc1);
        if (q + 1 < KS) {
          acc0 = ffma2(pack2(x2.z, x2.w), pack2(yre[q + 1], yre[q + 1]), acc0);
          acc1 = ffma2(pack2(x2.w, x2.z), yim[q + 1], acc1);
        }
      }
      const float2 a0 = unpack2(acc0), a1 = unpack2(acc1);
      res[rr] = make_float2(a0.x + a1.x, a0.y + a1.y);
    }
    if (p.part_alias) __syncthreads();  // every thread is done reading the X tile
#pragma unroll
    for (int rr = 0; rr < RP; ++rr) {
      part[(slc * R + grp + rr * p.groups) * p.npitch + j] = res[rr];
    }
    __syncthreads();
    // store in output order; sum the k-slice partials in fixed order
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (tid + i * kThreadsSt >= out_elems) break;
      const int sidx = my_src + p.src_hi[4 * i];
      float2 v = part[sidx];
      for (int s = 1; s < p.slices; ++s) {
        const float2 w = part[s * R * p.npitch + sidx];
        v.x += w.x;
        v.y += w.y;
      }
      C[obase + my_out + p.out_hi[4 * i]] = v;
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

}  // namespace

struct StreamPlan {
  StreamParams p;
  size_t smem;
  int ks;
};

// legs: kind 0 = X-free (x_stride, out_stride), 1 = common (x_stride,
// y_stride), 2 = Y-free (y_stride, out_stride).  Extents are all 2.
int stream_prepare(int n_legs, const StreamLeg* legs, StreamPlan** out) {
  *out = nullptr;
  std::vector<StreamLeg> xf, cm, yf;
  for (int i = 0; i < n_legs; ++i) {
    if (legs[i].kind == 0) xf.push_back(legs[i]);
    else if (legs[i].kind == 1) cm.push_back(legs[i]);
    else yf.push_back(legs[i]);
  }
  const int kb = static_cast<int>(cm.size()), g = static_cast<int>(yf.size()), fx = static_cast<int>(xf.size());
  if (kb > 10 || g > 6 || (1 << (kb + g)) > 4096) TNC_RET(TNC_ERR_UNSUPPORTED, "stream: Y too large");
  const int K = 1 << kb, N = 1 << g;
  const int ks = std::min(K, kMaxSlice);
  const int S = K / ks;
  if (N * S > kThreadsSt) TNC_RET(TNC_ERR_UNSUPPORTED, "stream: N * K too large");
  const int G = kThreadsSt / (N * S);
  // largest tile that fits the smem / register budget
  int t = -1;
  for (int c = std::min(fx, 12); c >= 0; --c) {
    const int R = 1 << c;
    if (R * K > 4096 || R * N > 4096 || S * R * N > 4096 || R < G || R / G > kMaxRowsPer) continue;
    t = c;
    break;
  }
  if (t < 0) TNC_RET(TNC_ERR_UNSUPPORTED, "stream: no tile shape fits");
  auto* sp = new StreamPlan();
  std::memset(&sp->p, 0, sizeof(sp->p));
  StreamParams& p = sp->p;
  p.kb = kb;
  p.t = t;
  p.g = g;
  p.slices = S;
  p.groups = G;
  p.kpad = K >= 16 ? K + 2 : std::max(K, 2);  // even: 16-byte row loads
  // tile rows: alternate X's fastest and the output's fastest free legs
  std::vector<int> by_x(fx), by_o(fx), tile;
  for (int i = 0; i < fx; ++i) by_x[i] = by_o[i] = i;
  std::sort(by_x.begin(), by_x.end(), [&](int a, int b) { return xf[a].x_stride < xf[b].x_stride; });
  std::sort(by_o.begin(), by_o.end(), [&](int a, int b) { return xf[a].out_stride < xf[b].out_stride; });
  auto take = [&](int c) {
    if (static_cast<int>(tile.size()) < t && std::find(tile.begin(), tile.end(), c) == tile.end()) tile.push_back(c);
  };
  // X's free legs among its 4 fastest axes first (DRAM reads come in >= 64-byte
  // runs), then alternate output-fastest / X-fastest
  {
    std::vector<int64_t> all;
    for (auto& l : xf) all.push_back(l.x_stride);
    for (auto& l : cm) all.push_back(l.x_stride);
    std::sort(all.begin(), all.end());
    const int64_t cut = all[std::min<size_t>(3, all.size() - 1)];
    for (int c : by_x)
      if (xf[c].x_stride <= cut) take(c);
  }
  for (int i = 0; i < fx; ++i) {
    take(by_o[i]);
    take(by_x[i]);
  }
  // row index r: bit b <-> tile[b]; column k: bit b <-> cm[b] (Y's k order is
  // the same bit order); output column j: bit b <-> yf[b]
  // load enumeration: all tile bits (rows + commons) by X stride ascending
  struct Bit { int64_t xs; int pos; };
  std::vector<Bit> lb;
  for (int b = 0; b < t; ++b) lb.push_back({xf[tile[b]].x_stride, (1 << b) * p.kpad});
  for (int b = 0; b < kb; ++b) lb.push_back({cm[b].x_stride, 1 << b});
  std::stable_sort(lb.begin(), lb.end(), [](const Bit& a, const Bit& b) { return a.xs < b.xs; });
  // store enumeration: row bits + Y-free bits by output stride ascending
  struct OBit { int64_t os; int src; };
  std::vector<OBit> ob;
  const int np = N > 1 ? N + 1 : 1;  // odd partial pitch: output-ordered reads spread over banks
  p.npitch = np;
  for (int b = 0; b < t; ++b) ob.push_back({xf[tile[b]].out_stride, (1 << b) * np});
  for (int b = 0; b < g; ++b) ob.push_back({yf[b].out_stride, 1 << b});
  std::stable_sort(ob.begin(), ob.end(), [](const OBit& a, const OBit& b) { return a.os < b.os; });
  for (int i = 0; i < 64; ++i) {
    for (int b = 0; b < 6; ++b) {
      if (!(i & (1 << b))) continue;
      if (b < static_cast<int>(lb.size())) {
        p.in_lo[i] += lb[b].xs;
        p.pos_lo[i] += lb[b].pos;
      }
      if (b + 6 < static_cast<int>(lb.size())) {
        p.in_hi[i] += lb[b + 6].xs;
        p.pos_hi[i] += lb[b + 6].pos;
      }
      if (b < static_cast<int>(ob.size())) {
        p.out_lo[i] += ob[b].os;
        p.src_lo[i] += ob[b].src;
      }
      if (b + 6 < static_cast<int>(ob.size())) {
        p.out_hi[i] += ob[b + 6].os;
        p.src_hi[i] += ob[b + 6].src;
      }
    }
  }
  for (int jj = 0; jj < N; ++jj)
    for (int b = 0; b < g; ++b)
      if (jj & (1 << b)) p.yj[jj] += yf[b].y_stride;
  for (int i = 0; i < 32; ++i)
    for (int b = 0; b < 5; ++b)
      if (i & (1 << b)) {
        if (b < kb) p.yk_lo[i] += cm[b].y_stride;
        if (b + 5 < kb) p.yk_hi[i] += cm[b + 5].y_stride;
      }
  // outer bits: X-free legs outside the tile, X-fastest first, so tiles that
  // run concurrently (consecutive tile ids) share DRAM sectors in L2
  for (int i : by_x) {
    if (std::find(tile.begin(), tile.end(), i) != tile.end()) continue;
    p.outer_x[p.n_outer] = xf[i].x_stride;
    p.outer_out[p.n_outer] = xf[i].out_stride;
    ++p.n_outer;
  }
  p.n_tiles = static_cast<int64_t>(1) << p.n_outer;
  const int R = 1 << t;
  p.part_alias = S * R * np <= R * p.kpad ? 1 : 0;
  sp->smem = static_cast<size_t>(2 * R * p.kpad + (p.part_alias ? 0 : S * R * np)) * sizeof(float2);
  sp->ks = ks;
  *out = sp;
  return TNC_OK;
}

void stream_destroy(StreamPlan* sp) { delete sp; }

int stream_launch(const StreamPlan* sp, const void* x, const void* y, void* c, cudaStream_t stream) {
  const StreamParams& p = sp->p;
  const int64_t rows = (static_cast<int64_t>(1) << (p.t + p.n_outer));
  ProfScope prof(PROF_STREAM, 8.0 * rows * (1 << p.kb) * (1 << p.g),
                 8.0 * (rows * (1 << p.kb) + (1 << (p.kb + p.g)) + rows * (1 << p.g)), stream);
  auto go = [&](auto kern) -> int {
    TNC_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>(sp->smem)));
    int per_sm = 1;
    TNC_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreadsSt, sp->smem));
    const int64_t blocks = std::min<int64_t>(p.n_tiles, static_cast<int64_t>(num_sms()) * std::max(1, per_sm));
    kern<<<static_cast<unsigned>(blocks), kThreadsSt, sp->smem, stream>>>(
        static_cast<const float2*>(x), static_cast<const float2*>(y), static_cast<float2*>(c), p);
    TNC_CHECK_LAUNCH();
    return TNC_OK;
  };
  const int rp = (1 << p.t) / p.groups;
#define TNC_STREAM_RP(KS_)                           \
  switch (rp) {                                      \
    case 1: return go(stream_kernel<KS_, 1>);        \
    case 2: return go(stream_kernel<KS_, 2>);        \
    case 4: return go(stream_kernel<KS_, 4>);        \
    case 8: return go(stream_kernel<KS_, 8>);        \
    default: return go(stream_kernel<KS_, 16>);      \
  }
  switch (sp->ks) {
    case 1: TNC_STREAM_RP(1)
    case 2: TNC_STREAM_RP(2)
    case 4: TNC_STREAM_RP(4)
    case 8: TNC_STREAM_RP(8)
    default: TNC_STREAM_RP(16)
  }
#undef TNC_STREAM_RP
}

}  // namespace tnc
