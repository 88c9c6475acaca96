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

template <typename T>
__global__ void __launch_bounds__(kTileThreads) permute_tile_kernel(const T* __restrict__ in,
                                                                    T* __restrict__ out,
                                                                    const PermParams p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* tile = reinterpret_cast<T*>(smem_raw);
  const int tiles_pad = pad_idx(p.tile_elems) + 1;
  int64_t* in_off = reinterpret_cast<int64_t*>(tile + tiles_pad);
  int64_t* out_off = in_off + p.tile_elems;
  int* src_of = reinterpret_cast<int*>(out_off + p.tile_elems);
  __shared__ int64_t s_base[2];

  // Build tables once per block.
  // Input-order enumeration e: digits over tile axes, axis 0 fastest.
  // Output-order enumeration f: digits ordered by tile_out_rank (0 fastest).
  for (int e = threadIdx.x; e < p.tile_elems; e += blockDim.x) {
    int64_t rem = e, oin = 0;
    for (int a = 0; a < p.n_tile; ++a) {
      int64_t d = p.tile_dim[a];
      int64_t q = rem / d;
      oin += (rem - q * d) * p.tile_in[a];
      rem = q;
    }
    in_off[e] = oin;
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
    out_off[f] = oout;
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
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int f = tid + i * kTileThreads;
      if (f < p.tile_elems) dst[out_off[f]] = v[i];
    }
    __syncthreads();
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

int permute_launch(int dtype, int rank, const int64_t* dims, const int64_t* in_strides,
                   const int32_t* perm, const void* in, void* out, cudaStream_t stream) {
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
  const size_t eb = elem_bytes(dtype);
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
  if (total == 0) return TNC_OK;
  ProfScope prof(PROF_PERMUTE, 0.0, 2.0 * static_cast<double>(total) * eb, stream);
  // full contiguous copy
  if (ax.empty() || (ax.size() == 1 && ax[0].in_stride == 1)) {
    TNC_CUDA_TRY(cudaMemcpyAsync(out, in, static_cast<size_t>(total) * eb,
                                 cudaMemcpyDeviceToDevice, stream));
    return TNC_OK;
  }
  const int sms = num_sms();
  // row copy when the innermost output leg is unit stride in the input and long
  const NormAxis& inner = ax.back();
  if (inner.in_stride == 1 && inner.dim >= 16) {
    RowParams p{};
    p.row_len = inner.dim;
    p.n_rows = total / inner.dim;
    std::vector<NormAxis> outer(ax.begin(), ax.end() - 1);
    TNC_TRY(fill_outer(outer, p.outer));
    int64_t warps_needed = p.n_rows;
    int64_t blocks = std::min<int64_t>(ceil_div(warps_needed, 8), static_cast<int64_t>(sms) * 16);
    blocks = std::max<int64_t>(blocks, 1);
    if (dtype == TNC_C128)
      permute_rows_kernel<c128><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
          static_cast<const c128*>(in), static_cast<c128*>(out), p);
    else
      permute_rows_kernel<c64><<<static_cast<unsigned>(blocks), 256, 0, stream>>>(
          static_cast<const c64*>(in), static_cast<c64*>(out), p);
    TNC_CHECK_LAUNCH();
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
  PermParams p{};
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
  size_t smem = static_cast<size_t>(tiles_pad) * eb + static_cast<size_t>(p.tile_elems) * 20;
  smem = (smem + 15) & ~size_t(15);
  int blocks_per_sm = tile >= 1024 ? 3 : 6;
  int64_t blocks = std::min<int64_t>(p.n_tiles, static_cast<int64_t>(sms) * blocks_per_sm);
  if (dtype == TNC_C128) {
    auto k = permute_tile_kernel<c128>;
    TNC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    k<<<static_cast<unsigned>(blocks), 256, smem, stream>>>(static_cast<const c128*>(in),
                                                            static_cast<c128*>(out), p);
  } else {
    auto k = permute_tile_kernel<c64>;
    TNC_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
    k<<<static_cast<unsigned>(blocks), 256, smem, stream>>>(static_cast<const c64*>(in),
                                                            static_cast<c64*>(out), p);
  }
  TNC_CHECK_LAUNCH();
  return TNC_OK;
}

}  // namespace tnc
