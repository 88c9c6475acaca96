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
#include <cstring>
#include <vector>

#include "tnc_common.cuh"

namespace tnc {

namespace {

constexpr int kTileBits = 12;              // 4096 complex64 = 32 KB tile
constexpr int kTile = 1 << kTileBits;
constexpr int kMaxSectionGates = 16;
constexpr int kThreadsAbs = 512;

struct AbsorbParams {
  int n_outer;
  int n_gates;
  int64_t n_tiles;
  // 2-level tables over the tile index (low 6 bits / high 6 bits)
  int64_t in_lo[64], in_hi[64];    // input element offset of load index e
  int64_t out_lo[64], out_hi[64];  // output element offset of store index f
  int src_lo[64], src_hi[64];      // load index e holding store index f
  int gate_bits[kMaxSectionGates][2];  // tile bit of in_a, in_b (load enumeration)
  float2 u[kMaxSectionGates][16];      // U[(oa,ob),(ia,ib)] row-major
  int outer_shift[TNC_MAX_RANK];       // outer axis digit = (t >> shift) & 1
  int64_t outer_in[TNC_MAX_RANK];
  int64_t outer_out[TNC_MAX_RANK];
};

__device__ __forceinline__ float2 cmul_add(float2 acc, float2 a, float2 b) {
  acc.x = fmaf(a.x, b.x, acc.x);
  acc.x = fmaf(-a.y, b.y, acc.x);
  acc.y = fmaf(a.x, b.y, acc.y);
  acc.y = fmaf(a.y, b.x, acc.y);
  return acc;
}

__global__ void __launch_bounds__(kThreadsAbs) absorb_pass_kernel(const float2* __restrict__ in,
                                                                  float2* __restrict__ out,
                                                                  const AbsorbParams p) {
  __shared__ float2 tile[kTile];
  __shared__ int64_t s_base[2];
  const int tid = threadIdx.x;
  const int lane = tid & 31;
  for (int64_t t = blockIdx.x; t < p.n_tiles; t += gridDim.x) {
    if (tid < 32) {
      int64_t bi = 0, bo = 0;
      for (int a = lane; a < p.n_outer; a += 32) {
        const int64_t d = (t >> p.outer_shift[a]) & 1;
        bi += d * p.outer_in[a];
        bo += d * p.outer_out[a];
      }
#pragma unroll
      for (int s = 16; s > 0; s >>= 1) {
        bi += __shfl_xor_sync(0xffffffffu, bi, s);
        bo += __shfl_xor_sync(0xffffffffu, bo, s);
      }
      if (lane == 0) {
        s_base[0] = bi;
        s_base[1] = bo;
      }
    }
    __syncthreads();
    const float2* src = in + s_base[0];
    float2* dst = out + s_base[1];
    constexpr int kPer = kTile / kThreadsAbs;
    float2 v[kPer];
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int e = tid + i * kThreadsAbs;
      v[i] = src[p.in_lo[e & 63] + p.in_hi[e >> 6]];
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) tile[tid + i * kThreadsAbs] = v[i];
    __syncthreads();
    for (int g = 0; g < p.n_gates; ++g) {
      const int ba = p.gate_bits[g][0], bb = p.gate_bits[g][1];
      const int lo = min(ba, bb), hi = max(ba, bb);
      // quartets: insert zero bits at positions lo and hi into q
      for (int q = tid; q < kTile / 4; q += kThreadsAbs) {
        int base = q;
        base = ((base >> lo) << (lo + 1)) | (base & ((1 << lo) - 1));
        base = ((base >> hi) << (hi + 1)) | (base & ((1 << hi) - 1));
        const int ia[4] = {base, base | (1 << bb), base | (1 << ba), base | (1 << ba) | (1 << bb)};
        float2 x[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = tile[ia[j]];
#pragma unroll
        for (int o = 0; o < 4; ++o) {
          float2 acc = make_float2(0.f, 0.f);
#pragma unroll
          for (int j = 0; j < 4; ++j) acc = cmul_add(acc, p.u[g][o * 4 + j], x[j]);
          tile[ia[o]] = acc;
        }
      }
      __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int f = tid + i * kThreadsAbs;
      v[i] = tile[p.src_lo[f & 63] | p.src_hi[f >> 6]];
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int f = tid + i * kThreadsAbs;
      dst[p.out_lo[f & 63] + p.out_hi[f >> 6]] = v[i];
    }
    __syncthreads();
  }
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
    p.src_lo[i] = slo;
    p.src_hi[i] = shi;
  }
  p.n_gates = static_cast<int>(sec.gates.size());
  for (int g = 0; g < p.n_gates; ++g) {
    const GateRef& gr = gates[sec.gates[g]];
    p.gate_bits[g][0] = bit_of[gr.pa];
    p.gate_bits[g][1] = bit_of[gr.pb];
    std::memcpy(p.u[g], gr.u, 16 * sizeof(float2));  // host gate data baked into the launch
  }
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
  const int64_t blocks = std::min<int64_t>(p.n_tiles, static_cast<int64_t>(num_sms()) * 4);
  ProfScope prof(PROF_ABSORB, 32.0 * p.n_gates * (static_cast<double>(1) * (int64_t(1) << r)),
                 16.0 * static_cast<double>(int64_t(1) << r), stream);
  absorb_pass_kernel<<<static_cast<unsigned>(blocks), kThreadsAbs, 0, stream>>>(in, out, p);
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
