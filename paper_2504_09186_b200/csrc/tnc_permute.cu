// K1: general strided permutation (reference tensor.py:252-274, `permute`).
//
// The reference builds an int64 offset table of |T| entries and gathers
// element by element.  Here the permutation is first normalised on the host
// (unit legs dropped, legs adjacent in both orders merged, long legs split),
// then one of two HBM-streaming kernels runs:
//   * row copy  - the innermost output leg is also unit-stride in the input:
//                 every output row is one contiguous input run (coalesced both
//                 ways, vectorised);
//   * tile      - a tile spanning the input-fastest legs (coalesced reads)
//                 and the output-fastest legs (coalesced writes) is staged in
//                 shared memory; per-block offset tables are built once and the
//                 block strides over all tiles (persistent, grid = k*148).
// Pure copies: results are bit-exact.
#include <algorithm>
#include <vector>

#include "tnc_common.cuh"
#include "tnc_permute.cuh"

namespace tnc {

namespace {

constexpr int kMaxTile = 2048;  // elements per smem tile
constexpr int kMaxAxes = 2 * TNC_MAX_RANK;

// Outer (non-tile) axes of a permutation: digit a of a linear outer index id
// is (id / div[a]) % dim[a]; it moves the input by sin[a], the output by sout[a].
struct OuterAxes {
  int n;
  int64_t dim[kMaxAxes];
  int64_t div[kMaxAxes];
  int64_t sin[kMaxAxes];
  int64_t sout[kMaxAxes];
};

struct PermParams {
  int n_tile;              // tile axes, ordered by input stride ascending
  int tile_elems;
  int64_t n_tiles;
  int64_t tile_dim[16];
  int64_t tile_in[16];
  int64_t tile_out[16];
  int tile_out_rank[16];   // position of tile axis in output-fastest order
  OuterAxes outer;
};

struct RowParams {
  int64_t row_len;
  int64_t n_rows;
  OuterAxes outer;
};

// Warp-parallel decode of an outer index: lane l handles axes l, l+32, ...,
// contributions are summed with shuffles.  All lanes return the result.
__device__ __forceinline__ void warp_decode(int64_t id, const OuterAxes& o, int lane, int64_t& bin,
                                            int64_t& bout) {
  int64_t si = 0, so = 0;
  for (int a = lane; a < o.n; a += 32) {
    const int64_t digit = (id / o.div[a]) % o.dim[a];
    si += digit * o.sin[a];
    so += digit * o.sout[a];
  }
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    si += __shfl_xor_sync(0xffffffffu, si, s);
    so += __shfl_xor_sync(0xffffffffu, so, s);
  }
  bin = si;
  bout = so;
}

// The decode indexes the axis tables per lane; from the kernel-parameter bank
// those divergent loads serialise, so each block stages them in smem first.
__device__ __forceinline__ void stage_outer(const OuterAxes& src, OuterAxes& dst) {
  if (threadIdx.x == 0) dst.n = src.n;
  for (int a = threadIdx.x; a < src.n; a += blockDim.x) {
    dst.dim[a] = src.dim[a];
    dst.div[a] = src.div[a];
    dst.sin[a] = src.sin[a];
    dst.sout[a] = src.sout[a];
  }
  __syncthreads();
}

__device__ __forceinline__ int pad_idx(int e) { return e + (e >> 4); }

constexpr int kTileThreads = 256;
constexpr int kItems = kMaxTile / kTileThreads;  // elements per thread per tile (<= 8)

// Epilogue of the tile kernel: a plain copy, or the 3xFP16 operand split of a
// GEMM operand gathered to [R rows, K] (K = 2^log_k, row pitch K): pass 1
// (ROWMAX) folds each row's max |component| into rowmax[], pass 2 (SPLIT0 /
// SPLIT1) writes the scaled hi / lo fp16 planes (SPLIT1: the expanded rows
// 2r = (re, -im), 2r+1 = (im, re)) -- the same planes f16_split_launch makes
// from the permuted copy, without writing or re-reading that copy.
enum PermMode { PERM_COPY = 0, PERM_ROWMAX = 1, PERM_SPLIT0 = 2, PERM_SPLIT1 = 3 };

struct SplitOut {
  int log_k;
  unsigned* rowmax;   // ROWMAX: float bits of max |component| per row (atomicMax)
  const float* scale; // SPLIT: per-row 2^-e
  __half2* hi;
  __half2* lo;
};

// Off: element offsets inside one tile, int32 when every tile offset fits
// (smaller tables: 4 instead of 3 blocks per SM for complex64 tiles)
template <typename T, int MODE, typename Off>
__global__ void __launch_bounds__(kTileThreads) permute_tile_kernel(const T* __restrict__ in,
                                                                    T* __restrict__ out,
                                                                    const PermParams p, const SplitOut so_) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);
  const int tiles_pad = pad_idx(p.tile_elems) + 1;
  Off* in_off = reinterpret_cast<Off*>(tile + tiles_pad);
  Off* out_off = in_off + p.tile_elems;
  int* src_of = reinterpret_cast<int*>(out_off + p.tile_elems);
  // ROWMAX only: row slot of each input-order element, per-slot maxima
  int16_t* slot_of = reinterpret_cast<int16_t*>(src_of + p.tile_elems);
  unsigned* rmax = reinterpret_cast<unsigned*>(slot_of + p.tile_elems + (p.tile_elems & 1));
  __shared__ int64_t s_base[2];
  __shared__ int s_nslots;

  // Build tables once per block.
  // Input-order enumeration e: digits over tile axes, axis 0 fastest.
  // Output-order enumeration f: digits ordered by tile_out_rank (0 fastest).
  for (int e = threadIdx.x; e < p.tile_elems; e += blockDim.x) {
    int64_t rem = e, oin = 0;
    int slot = 0, cm = 1;
    for (int a = 0; a < p.n_tile; ++a) {
      int64_t d = p.tile_dim[a];
      int64_t q = rem / d;
      oin += (rem - q * d) * p.tile_in[a];
      if (MODE == PERM_ROWMAX && p.tile_out[a] >= (int64_t{1} << so_.log_k)) {  // a row axis
        slot += static_cast<int>(rem - q * d) * cm;
        cm *= static_cast<int>(d);
      }
      rem = q;
    }
    in_off[e] = static_cast<Off>(oin);
    if (MODE == PERM_ROWMAX) {
      slot_of[e] = static_cast<int16_t>(slot);
      if (e == 0) s_nslots = cm;
    }
  }
  for (int f = threadIdx.x; f < p.tile_elems; f += blockDim.x) {
    // decode f over axes sorted by output stride (rank 0 fastest)
    int64_t rem = f, oout = 0;
    int e = 0;
    // digit of each tile axis
    int64_t digit[16];
    for (int r = 0; r < p.n_tile; ++r) {
      // find axis with out rank r
      int a = 0;
      for (int b = 0; b < p.n_tile; ++b)
        if (p.tile_out_rank[b] == r) a = b;
      int64_t d = p.tile_dim[a];
      int64_t q = rem / d;
      digit[a] = rem - q * d;
      rem = q;
      oout += digit[a] * p.tile_out[a];
    }
    int64_t mul = 1;
    for (int a = 0; a < p.n_tile; ++a) {
      e += static_cast<int>(digit[a] * mul);
      mul *= p.tile_dim[a];
    }
    out_off[f] = static_cast<Off>(oout);
    src_of[f] = pad_idx(e);
  }
  __syncthreads();

  const int tid = threadIdx.x;
  const int lane = tid & 31;
  __shared__ OuterAxes so;
  stage_outer(p.outer, so);
  for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
    if (tid < 32) {
      int64_t bin, bout;
      warp_decode(t, so, lane, bin, bout);
      if (lane == 0) {
        s_base[0] = bin;
        s_base[1] = bout;
      }
    }
    __syncthreads();
    const T* src = in + s_base[0];
    T* dst = out + s_base[1];
    // batched loads: all of this thread's elements in flight before any store
    T v[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int e = tid + i * kTileThreads;
      if (e < p.tile_elems) v[i] = src[in_off[e]];
    }
    if constexpr (MODE == PERM_ROWMAX) {
      // per-tile row maxima in smem (no transpose needed), then one global
      // atomic per row of the tile; non-negative floats order like their bits
      for (int q = tid; q < s_nslots; q += kTileThreads) rmax[q] = 0u;
      __syncthreads();
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const int e = tid + i * kTileThreads;
        if (e < p.tile_elems) {
          // a tile can hold few rows: read first, so only increases hit the
          // (contended) smem atomic
          const unsigned b = __float_as_uint(fmaxf(fabsf(v[i].re), fabsf(v[i].im)));
          volatile unsigned* a = rmax + slot_of[e];
          if (b > *a) atomicMax(const_cast<unsigned*>(a), b);
        }
      }
      __syncthreads();
      for (int q = tid; q < s_nslots; q += kTileThreads) {
        int64_t off = 0;
        int rest = q;
        for (int a = 0; a < p.n_tile; ++a)
          if (p.tile_out[a] >= (int64_t{1} << so_.log_k)) {
            off += static_cast<int64_t>(rest % p.tile_dim[a]) * p.tile_out[a];
            rest /= static_cast<int>(p.tile_dim[a]);
          }
        atomicMax(so_.rowmax + ((s_base[1] + off) >> so_.log_k), rmax[q]);
      }
      __syncthreads();
    } else {
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int e = tid + i * kTileThreads;
      if (e < p.tile_elems) tile[pad_idx(e)] = v[i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int f = tid + i * kTileThreads;
      if (f < p.tile_elems) v[i] = tile[src_of[f]];
    }
    if constexpr (MODE == PERM_COPY) {
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const int f = tid + i * kTileThreads;
        if (f < p.tile_elems) dst[out_off[f]] = v[i];
      }
    } else {
#pragma unroll
      for (int i = 0; i < kItems; ++i) {
        const int f = tid + i * kTileThreads;
        if (f < p.tile_elems) {
          const int64_t o = s_base[1] + out_off[f];
          const int64_t r = o >> so_.log_k;
          const int64_t k = o & ((int64_t{1} << so_.log_k) - 1);
          const float sc = __ldg(so_.scale + r);
          const float re = v[i].re * sc, im = v[i].im * sc;
          const __half hre = __float2half_rn(re), him = __float2half_rn(im);
          const __half lre = __float2half_rn(re - __half2float(hre));
          const __half lim = __float2half_rn(im - __half2float(him));
          if constexpr (MODE == PERM_SPLIT0) {
            so_.hi[o] = __halves2half2(hre, him);
            so_.lo[o] = __halves2half2(lre, lim);
          } else {
            const int64_t o0 = ((2 * r) << so_.log_k) + k;
            const int64_t o1 = o0 + (int64_t{1} << so_.log_k);
            so_.hi[o0] = __halves2half2(hre, __hneg(him));
            so_.lo[o0] = __halves2half2(lre, __hneg(lim));
            so_.hi[o1] = __halves2half2(him, hre);
            so_.lo[o1] = __halves2half2(lim, lre);
          }
        }
      }
    }
    __syncthreads();
    }  // MODE != PERM_ROWMAX
  }
}

// Row maxima of a permuted view without permuting it.  The operand's legs are
// all powers of two, so the view splits into binary axes; each is a row axis
// (output stride >= 2^log_k) or a K axis.  The five smallest-input-stride axes
// are the lane bits (one coalesced 256-byte load per warp instruction); the
// other K axes are walked by a carry-delta counter; the other row axes pick
// the warp's task.  A task keeps its rows' maxima in registers, folds the lanes
// that differ only in K bits with shuffles, and does one global atomicMax per
// row -- the tile kernel's ROWMAX mode paid per-tile smem atomics plus one
// global atomic per tile row (~2 TB/s on C3's operands).
constexpr int kRmAxes = 40;
struct RowmaxParams {
  int64_t lane_in[5];
  int64_t lane_row[5];
  unsigned lane_kmask;      // lane bits that are K axes
  int n_ro;                 // row axes outside the lanes
  int kc_log;               // K-walk length per task: 2^kc_log
  int chunk_bits;           // (n K axes outside the lanes) - kc_log
  int64_t tasks;
  int64_t ro_in[kRmAxes];
  int64_t ro_row[kRmAxes];
  int64_t ko_in[kRmAxes];     // K axes outside the lanes, fastest first
  int64_t ko_delta[kRmAxes + 1];  // off(j + 1) - off(j) when ctz(j + 1) = t
};

__global__ void __launch_bounds__(256) rowmax_warp_kernel(const c64* __restrict__ in, const RowmaxParams p,
                                                          unsigned* __restrict__ rowmax) {
  const int lane = threadIdx.x & 31;
  int64_t lane_off = 0, lane_row = 0;
#pragma unroll
  for (int b = 0; b < 5; ++b)
    if ((lane >> b) & 1) {
      lane_off += p.lane_in[b];
      lane_row += p.lane_row[b];
    }
  const int64_t nw = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
  const int64_t steps = int64_t{1} << p.kc_log;
  for (int64_t task = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); task < p.tasks;
       task += nw) {
    const int64_t ro = task >> p.chunk_bits;
    int64_t base = lane_off, row = lane_row;
    for (int b = 0; b < p.n_ro; ++b)
      if ((ro >> b) & 1) {
        base += p.ro_in[b];
        row += p.ro_row[b];
      }
    const int64_t kc = task & ((int64_t{1} << p.chunk_bits) - 1);
    for (int b = 0; b < p.chunk_bits; ++b)
      if ((kc >> b) & 1) base += p.ko_in[p.kc_log + b];
    const float2* src = reinterpret_cast<const float2*>(in) + base;
    float m = 0.f;
    int64_t off = 0;
    for (int64_t j = 0; j < steps; j += 8) {
      int64_t o[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        o[u] = off;
        off += p.ko_delta[__ffsll(j + u + 1) - 1];
      }
      float2 v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u < steps) v[u] = __ldg(src + o[u]);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u < steps) m = fmaxf(m, fmaxf(fabsf(v[u].x), fabsf(v[u].y)));
    }
#pragma unroll
    for (int b = 0; b < 5; ++b)
      if ((p.lane_kmask >> b) & 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1 << b));
    // non-negative floats order like their bit patterns (NaN sorts above all)
    if ((lane & p.lane_kmask) == 0) atomicMax(rowmax + row, __float_as_uint(m));
  }
}

// false when the view does not fit the binary-axis scheme (the tile kernel's
// ROWMAX mode then runs)
bool plan_rowmax(int rank, const int64_t* dims, const int64_t* in_strides, const int32_t* perm, int log_k,
                 int sms, RowmaxParams& p, int64_t& blocks) {
  struct Bit {
    int64_t in, out;
  };
  std::vector<Bit> bits;
  int64_t os = 1;
  for (int t = rank - 1; t >= 0; --t) {
    const int s = perm[t];
    const int64_t d = dims[s];
    if (d < 1 || (d & (d - 1)) != 0) return false;
    for (int64_t f = 1; f < d; f *= 2) bits.push_back({in_strides[s] * f, os * f});
    os *= d;
  }
  if (bits.size() < 5 || bits.size() > static_cast<size_t>(kRmAxes)) return false;
  std::stable_sort(bits.begin(), bits.end(), [](const Bit& a, const Bit& b) { return a.in < b.in; });
  const int64_t K = int64_t{1} << log_k;
  p = RowmaxParams{};
  std::vector<int64_t> ko;
  for (size_t i = 0; i < bits.size(); ++i) {
    const bool is_row = bits[i].out >= K;
    if (i < 5) {
      p.lane_in[i] = bits[i].in;
      p.lane_row[i] = is_row ? bits[i].out >> log_k : 0;
      if (!is_row) p.lane_kmask |= 1u << i;
    } else if (is_row) {
      p.ro_in[p.n_ro] = bits[i].in;
      p.ro_row[p.n_ro] = bits[i].out >> log_k;
      ++p.n_ro;
    } else {
      ko.push_back(bits[i].in);
    }
  }
  const int n_ko = static_cast<int>(ko.size());
  int64_t sum = 0;
  for (int t = 0; t < n_ko; ++t) {
    p.ko_in[t] = ko[t];
    p.ko_delta[t] = ko[t] - sum;
    sum += ko[t];
  }
  // enough tasks to fill every SM several times over, >= 8 steps per task
  const int64_t warps = static_cast<int64_t>(sms) * 64;
  p.kc_log = n_ko;
  while (p.kc_log > 3 && (int64_t{1} << (p.n_ro + n_ko - p.kc_log)) < 8 * warps) --p.kc_log;
  p.chunk_bits = n_ko - p.kc_log;
  p.tasks = int64_t{1} << (p.n_ro + p.chunk_bits);
  blocks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.tasks, 8), static_cast<int64_t>(sms) * 8));
  return true;
}

// row maxima -> exponents (for the GEMM epilogue) and 2^-e scales (written
// over the maxima: the split pass reads them as floats)
__global__ void rowmax_to_exp_kernel(int64_t R, unsigned* __restrict__ rowmax, int* __restrict__ exps) {
  for (int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; r < R;
       r += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float mx = __uint_as_float(rowmax[r]);
    const int e = f16_row_exponent(mx);  // same rule as f16_split_kernel
    exps[r] = e;
    rowmax[r] = __float_as_uint(ldexpf(1.f, -e));
  }
}

template <typename T>
__global__ void __launch_bounds__(256) permute_rows_kernel(const T* __restrict__ in,
                                                           T* __restrict__ out,
                                                           const RowParams p) {
  // one warp per row (grid-stride); rows are row_len contiguous elements
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  __shared__ OuterAxes so;
  stage_outer(p.outer, so);
  for (int64_t r = warp; r < p.n_rows; r += n_warps) {
    int64_t bin, bout;
    warp_decode(r, so, lane, bin, bout);
    const T* src = in + bin;
    T* dst = out + bout;
    int64_t i = lane;
    for (; i + 96 < p.row_len; i += 128) {
      T v0 = src[i], v1 = src[i + 32], v2 = src[i + 64], v3 = src[i + 96];
      dst[i] = v0;
      dst[i + 32] = v1;
      dst[i + 64] = v2;
      dst[i + 96] = v3;
    }
    for (; i < p.row_len; i += 32) dst[i] = src[i];
  }
}

struct NormAxis {
  int64_t dim, in_stride, out_stride;
};

// outer axes listed most significant first
int fill_outer(const std::vector<NormAxis>& axes, OuterAxes& o) {
  if (axes.size() > static_cast<size_t>(kMaxAxes)) TNC_RET(TNC_ERR_TENSOR, "permute: too many legs");
  o.n = static_cast<int>(axes.size());
  int64_t div = 1;
  for (int a = o.n - 1; a >= 0; --a) {
    o.dim[a] = axes[a].dim;
    o.div[a] = div;
    o.sin[a] = axes[a].in_stride;
    o.sout[a] = axes[a].out_stride;
    div *= axes[a].dim;
  }
  return TNC_OK;
}

}  // namespace

namespace {

// How a permutation runs: a plain copy, one contiguous run per output row, or
// smem tiles (see the file header).
struct PermPlan {
  enum Kind { EMPTY, MEMCPY, ROWS, TILE } kind = EMPTY;
  int64_t total = 0;
  RowParams rp{};
  PermParams tp{};
  int64_t blocks = 0;
  size_t smem = 0;
  bool off32 = false;  // tile offset tables fit int32
};

int plan_permute(size_t eb, int rank, const int64_t* dims, const int64_t* in_strides, const int32_t* perm,
                 PermPlan& pl) {
  if (rank < 0 || rank > TNC_MAX_RANK) TNC_RET(TNC_ERR_TENSOR, "permute: rank out of range");
  std::vector<int> seen(rank, 0);
  int64_t total = 1;
  for (int t = 0; t < rank; ++t) {
    if (perm[t] < 0 || perm[t] >= rank || seen[perm[t]])
      TNC_RET(TNC_ERR_PERMUTATION, "permute: perm is not a permutation of the legs");
    seen[perm[t]] = 1;
  }
  for (int s = 0; s < rank; ++s) {
    if (dims[s] < 1) TNC_RET(TNC_ERR_TENSOR, "permute: dim < 1");
    total *= dims[s];
  }
  pl.total = total;
  // target-order axes with output strides (contiguous output)
  std::vector<NormAxis> ax;
  {
    int64_t os = 1;
    std::vector<NormAxis> rev;
    for (int t = rank - 1; t >= 0; --t) {
      int s = perm[t];
      rev.push_back({dims[s], in_strides[s], os});
      os *= dims[s];
    }
    std::reverse(rev.begin(), rev.end());
    for (auto& a : rev)
      if (a.dim != 1) ax.push_back(a);
  }
  // merge target-adjacent legs that are also adjacent (same order) in the input
  {
    std::vector<NormAxis> merged;
    for (auto& a : ax) {
      if (!merged.empty()) {
        NormAxis& b = merged.back();
        if (b.in_stride == a.dim * a.in_stride && b.out_stride == a.dim * a.out_stride) {
          b.dim *= a.dim;
          b.in_stride = a.in_stride;
          b.out_stride = a.out_stride;
          continue;
        }
      }
      merged.push_back(a);
    }
    ax.swap(merged);
  }
  if (total == 0) {
    pl.kind = PermPlan::EMPTY;
    return TNC_OK;
  }
  // full contiguous copy
  if (ax.empty() || (ax.size() == 1 && ax[0].in_stride == 1)) {
    pl.kind = PermPlan::MEMCPY;
    return TNC_OK;
  }
  const int sms = num_sms();
  // row copy when the innermost output leg is unit stride in the input and long
  const NormAxis& inner = ax.back();
  if (inner.in_stride == 1 && inner.dim >= 16) {
    RowParams& p = pl.rp;
    p.row_len = inner.dim;
    p.n_rows = total / inner.dim;
    std::vector<NormAxis> outer(ax.begin(), ax.end() - 1);
    TNC_TRY(fill_outer(outer, p.outer));
    pl.blocks = std::max<int64_t>(std::min<int64_t>(ceil_div(p.n_rows, 8), static_cast<int64_t>(sms) * 16), 1);
    pl.kind = PermPlan::ROWS;
    return TNC_OK;
  }
  // tile path: split long legs.  Power-of-two legs (every quantum-circuit
  // leg, and runs of them merged above) split into factors of 2, so the tile
  // below can always grow one bit at a time to kMaxTile (with factors of 32 a
  // merged run could stall the growth at a small tile, measured 2 TB/s on a
  // C4 operand gather); other legs split into factors of 32 (a 32x32
  // transpose tile still fits twice in kMaxTile)
  {
    std::vector<NormAxis> split;
    for (auto& a : ax) {
      NormAxis cur = a;
      std::vector<NormAxis> parts;  // least significant first
      const bool pow2 = (cur.dim & (cur.dim - 1)) == 0;
      const int64_t f = pow2 ? 2 : 32;
      while (cur.dim > f && cur.dim % f == 0) {
        parts.push_back({f, cur.in_stride, cur.out_stride});
        cur.in_stride *= f;
        cur.out_stride *= f;
        cur.dim /= f;
      }
      parts.push_back(cur);
      for (auto it = parts.rbegin(); it != parts.rend(); ++it) split.push_back(*it);
    }
    ax.swap(split);
  }
  const int n = static_cast<int>(ax.size());
  std::vector<int> by_in(n), by_out(n);
  for (int i = 0; i < n; ++i) by_in[i] = by_out[i] = i;
  std::stable_sort(by_in.begin(), by_in.end(),
                   [&](int x, int y) { return ax[x].in_stride < ax[y].in_stride; });
  std::stable_sort(by_out.begin(), by_out.end(),
                   [&](int x, int y) { return ax[x].out_stride < ax[y].out_stride; });
  std::vector<char> in_tile(n, 0);
  int64_t tile = 1;
  auto try_add = [&](int a) {
    if (in_tile[a]) return true;
    if (tile * ax[a].dim > kMaxTile) return false;
    in_tile[a] = 1;
    tile *= ax[a].dim;
    return true;
  };
  // alternate: input-fastest and output-fastest legs until both sides have >= 32
  int64_t prod_in = 1, prod_out = 1;
  size_t pi = 0, po = 0;
  while ((prod_in < 32 && pi < by_in.size()) || (prod_out < 32 && po < by_out.size())) {
    bool progressed = false;
    if (prod_in < 32 && pi < by_in.size()) {
      int a = by_in[pi];
      if (try_add(a)) {
        prod_in *= ax[a].dim;
        ++pi;
        progressed = true;
      } else {
        pi = by_in.size();
      }
    }
    if (prod_out < 32 && po < by_out.size()) {
      int a = by_out[po];
      if (try_add(a)) {
        prod_out *= ax[a].dim;
        ++po;
        progressed = true;
      } else {
        po = by_out.size();
      }
    }
    if (!progressed) break;
  }
  // then grow the tile (alternating input- / output-fastest legs) up to
  // kMaxTile elements: more bytes per block barrier, more loads in flight
  {
    size_t qi = 0, qo = 0;
    bool grew = true;
    while (grew) {
      grew = false;
      while (qi < by_in.size() && in_tile[by_in[qi]]) ++qi;
      if (qi < by_in.size() && tile * ax[by_in[qi]].dim <= kMaxTile) {
        try_add(by_in[qi]);
        grew = true;
      }
      while (qo < by_out.size() && in_tile[by_out[qo]]) ++qo;
      if (qo < by_out.size() && tile * ax[by_out[qo]].dim <= kMaxTile) {
        try_add(by_out[qo]);
        grew = true;
      }
    }
  }
  if (tile == 1) {
    // every leg is huge and unsplittable: degenerate to one-element tiles
    in_tile[by_out[0]] = 1;
    tile = ax[by_out[0]].dim;
    if (tile > kMaxTile) TNC_RET(TNC_ERR_UNSUPPORTED, "permute: unsplittable leg too long");
  }
  PermParams& p = pl.tp;
  p.tile_elems = static_cast<int>(tile);
  int nt = 0;
  for (int a : by_in)
    if (in_tile[a]) {
      if (nt >= 16) TNC_RET(TNC_ERR_UNSUPPORTED, "permute: tile too fragmented");
      p.tile_dim[nt] = ax[a].dim;
      p.tile_in[nt] = ax[a].in_stride;
      p.tile_out[nt] = ax[a].out_stride;
      int r = 0;
      for (int b : by_out) {
        if (b == a) break;
        if (in_tile[b]) ++r;
      }
      p.tile_out_rank[nt] = r;
      ++nt;
    }
  p.n_tile = nt;
  {
    std::vector<NormAxis> outer;
    for (int a = 0; a < n; ++a)
      if (!in_tile[a]) outer.push_back(ax[a]);
    TNC_TRY(fill_outer(outer, p.outer));
  }
  p.n_tiles = total / tile;
  const int tiles_pad = (p.tile_elems + (p.tile_elems >> 4)) + 1;
  {
    int64_t max_in = 0, max_out = 0;
    for (int a = 0; a < p.n_tile; ++a) {
      max_in += (p.tile_dim[a] - 1) * p.tile_in[a];
      max_out += (p.tile_dim[a] - 1) * p.tile_out[a];
    }
    pl.off32 = max_in <= INT32_MAX && max_out <= INT32_MAX;
  }
  size_t smem = static_cast<size_t>(tiles_pad) * eb + static_cast<size_t>(p.tile_elems) * (pl.off32 ? 12 : 20);
  smem = (smem + 15) & ~size_t(15);
  // residency by smem (+ ~4.5 KB of static tables per block)
  const int by_smem = static_cast<int>((200 * 1024) / (smem + 4608));
  const int blocks_per_sm = std::max(1, std::min(tile >= 1024 ? 4 : 6, by_smem));
  pl.blocks = std::min<int64_t>(p.n_tiles, static_cast<int64_t>(sms) * blocks_per_sm);
  pl.smem = smem;
  pl.kind = PermPlan::TILE;
  return TNC_OK;
}

}  // namespace

// launch the tile kernel with the offset width the plan allows
template <typename T, int MODE>
int launch_tile(const PermPlan& pl, const void* in, void* out, const SplitOut& so, size_t smem,
                cudaStream_t stream) {
  auto k = pl.off32 ? permute_tile_kernel<T, MODE, int32_t> : permute_tile_kernel<T, MODE, int64_t>;
  TNC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
  k<<<static_cast<unsigned>(pl.blocks), 256, smem, stream>>>(static_cast<const T*>(in), static_cast<T*>(out),
                                                             pl.tp, so);
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

// Small tensors (the hundreds of leaf-sized steps of a slice): one thread per
// output element decodes its index.  The tile kernel's per-block table setup
// costs tens of microseconds, more than moving a megabyte.
constexpr int64_t kSmallPermute = int64_t{1} << 17;
struct SmallPermParams {
  int rank;
  int64_t total;
  int pow2;
  int64_t odim[TNC_MAX_RANK];     // output order, last fastest
  int64_t istride[TNC_MAX_RANK];  // input stride of the same leg
  int olog[TNC_MAX_RANK];         // log2 of the extent when pow2
};

template <typename T>
__global__ void __launch_bounds__(256) permute_small_kernel(const T* __restrict__ in, T* __restrict__ out,
                                                            const SmallPermParams p) {
  const int64_t o = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (o >= p.total) return;
  int64_t rem = o, off = 0;
  if (p.pow2) {  // every extent a power of two (qubit networks): shifts instead of divisions
    for (int a = p.rank - 1; a >= 0; --a) {
      off += (rem & (p.odim[a] - 1)) * p.istride[a];
      rem >>= p.olog[a];
    }
  } else {
    for (int a = p.rank - 1; a >= 0; --a) {
      const int64_t d = p.odim[a];
      const int64_t q = rem / d;
      off += (rem - q * d) * p.istride[a];
      rem = q;
    }
  }
  out[o] = in[off];
}

int permute_launch(int dtype, int rank, const int64_t* dims, const int64_t* in_strides,
                   const int32_t* perm, const void* in, void* out, cudaStream_t stream) {
  const size_t eb = elem_bytes(dtype);
  PermPlan pl;
  TNC_TRY(plan_permute(eb, rank, dims, in_strides, perm, pl));
  if (pl.kind == PermPlan::EMPTY) return TNC_OK;
  ProfScope prof(PROF_PERMUTE, 0.0, 2.0 * static_cast<double>(pl.total) * eb, stream);
  if (pl.kind == PermPlan::TILE && pl.total <= kSmallPermute && std::getenv("TNC_NO_SMALL_PERMUTE") == nullptr) {
    SmallPermParams sp;
    sp.rank = rank;
    sp.total = pl.total;
    sp.pow2 = 1;
    for (int t = 0; t < rank; ++t) {
      const int64_t d = dims[perm[t]];
      sp.odim[t] = d;
      sp.istride[t] = in_strides[perm[t]];
      sp.olog[t] = 0;
      while ((int64_t{1} << sp.olog[t]) < d) ++sp.olog[t];
      if ((int64_t{1} << sp.olog[t]) != d) sp.pow2 = 0;
    }
    const unsigned blocks = static_cast<unsigned>(ceil_div(pl.total, 256));
    if (dtype == TNC_C128)
      permute_small_kernel<c128><<<blocks, 256, 0, stream>>>(static_cast<const c128*>(in), static_cast<c128*>(out), sp);
    else
      permute_small_kernel<c64><<<blocks, 256, 0, stream>>>(static_cast<const c64*>(in), static_cast<c64*>(out), sp);
    TNC_CHECK_LAUNCH();
    return TNC_OK;
  }
  if (pl.kind == PermPlan::MEMCPY) {
    TNC_CUDA_TRY(cudaMemcpyAsync(out, in, static_cast<size_t>(pl.total) * eb, cudaMemcpyDeviceToDevice, stream));
    return TNC_OK;
  }
  if (pl.kind == PermPlan::ROWS) {
    if (dtype == TNC_C128)
      permute_rows_kernel<c128><<<static_cast<unsigned>(pl.blocks), 256, 0, stream>>>(
          static_cast<const c128*>(in), static_cast<c128*>(out), pl.rp);
    else
      permute_rows_kernel<c64><<<static_cast<unsigned>(pl.blocks), 256, 0, stream>>>(
          static_cast<const c64*>(in), static_cast<c64*>(out), pl.rp);
    TNC_CHECK_LAUNCH();
    return TNC_OK;
  }
  const SplitOut none{};
  if (dtype == TNC_C128) return launch_tile<c128, PERM_COPY>(pl, in, out, none, pl.smem, stream);
  return launch_tile<c64, PERM_COPY>(pl, in, out, none, pl.smem, stream);
}

int permute_split_f16_launch(int rank, const int64_t* dims, const int64_t* in_strides, const int32_t* perm,
                             const void* in, int mode, int64_t R, int log_k, void* hi, void* lo, int* exps,
                             unsigned* rowmax, cudaStream_t stream) {
  PermPlan pl;
  TNC_TRY(plan_permute(sizeof(c64), rank, dims, in_strides, perm, pl));
  if (pl.kind != PermPlan::TILE) TNC_RET(TNC_ERR_UNSUPPORTED, "permute+split: not a tiled permutation");
  if (pl.total != (R << log_k)) TNC_RET(TNC_ERR_INVALID, "permute+split: R * 2^log_k != elements");
  // one read for the row maxima, one read + the plane writes for the split
  ProfScope prof(PROF_SPLIT_PREP, 0.0, 16.0 * pl.total + (mode ? 16.0 : 8.0) * pl.total, stream);
  TNC_CUDA_TRY(cudaMemsetAsync(rowmax, 0, static_cast<size_t>(R) * sizeof(unsigned), stream));
  SplitOut so{log_k, rowmax, reinterpret_cast<const float*>(rowmax), static_cast<__half2*>(hi),
              static_cast<__half2*>(lo)};
  RowmaxParams rp;
  int64_t rblocks = 0;
  if (std::getenv("TNC_TILE_ROWMAX") == nullptr &&
      plan_rowmax(rank, dims, in_strides, perm, log_k, num_sms(), rp, rblocks)) {
    rowmax_warp_kernel<<<static_cast<unsigned>(rblocks), 256, 0, stream>>>(static_cast<const c64*>(in), rp, rowmax);
    TNC_CHECK_LAUNCH();
  } else {
    const size_t smem = pl.smem + static_cast<size_t>(pl.tp.tile_elems) * (2 + 4) + 16;
    TNC_TRY((launch_tile<c64, PERM_ROWMAX>(pl, in, nullptr, so, smem, stream)));
  }
  rowmax_to_exp_kernel<<<static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(ceil_div(R, 256), 4096))), 256,
                         0, stream>>>(R, rowmax, exps);
  TNC_CHECK_LAUNCH();
  if (mode == 0) return launch_tile<c64, PERM_SPLIT0>(pl, in, nullptr, so, pl.smem, stream);
  return launch_tile<c64, PERM_SPLIT1>(pl, in, nullptr, so, pl.smem, stream);
}

}  // namespace tnc
