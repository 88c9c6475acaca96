// C-ABI entry points (include/tnc_b200.h) and the contraction planner.
//
// tnc_plan_contract realises the reference's contract_pair index map
// (contract.py:58-117): free_A (A order), common (A order), free_B (B order),
// result legs free_A ++ free_B (or a caller-given permutation of them).  The
// device execution differs from the reference's permute-both-then-GEMM:
//   * the larger operand X goes on the GEMM row side and keeps its own order
//     of the common legs, so it is consumed in place whenever its legs are
//     already [free..., common...] (true for most stem tensors);
//   * the smaller operand Y is gathered to [free_Y, common(X order)];
//   * the GEMM epilogue writes C straight into the output layout
//     (free_A ++ free_B, row- or column-oriented), no trailing transpose.
#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "tnc_common.cuh"
#include "tnc_gather_tc.cuh"
#include "tnc_permute.cuh"

namespace tnc {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
const char* last_error() { return g_last_error.c_str(); }

// ---- launch counter and optional per-kernel event timing ----
static std::atomic<int64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

namespace {
struct ProfRec {
  int kind;
  double flops, bytes;
  cudaEvent_t start, stop;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;
std::atomic<bool> g_prof_on{false};
}  // namespace

ProfScope::ProfScope(int kind, double flops, double bytes, cudaStream_t stream)
    : kind_(kind), flops_(flops), bytes_(bytes), stream_(stream) {
  if (!g_prof_on.load(std::memory_order_relaxed)) return;
  if (cudaEventCreate(&start_) != cudaSuccess) {
    start_ = nullptr;
    return;
  }
  cudaEventRecord(start_, stream_);
}

ProfScope::~ProfScope() {
  if (!start_) return;
  cudaEvent_t stop = nullptr;
  if (cudaEventCreate(&stop) != cudaSuccess) {
    cudaEventDestroy(start_);
    return;
  }
  cudaEventRecord(stop, stream_);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back({kind_, flops_, bytes_, start_, stop});
}

namespace {

struct Leg {
  int32_t label;
  int64_t dim;
  int64_t stride;
};

struct Operand {
  std::vector<Leg> free;    // operand's own order
  std::vector<Leg> common;  // in X's common order
  bool in_place = false;    // consumable as a [rows, K] matrix without a gather
  int64_t ld = 0;           // row stride when in place
  // gather (permute) description when not in place
  std::vector<int64_t> dims, strides;
  std::vector<int32_t> perm;
  int64_t rows = 1;
};

}  // namespace
}  // namespace tnc

struct tnc_plan {
  int32_t dtype;
  int32_t variant;
  int32_t b_is_multiplier;
  int32_t x_is_a;  // row-side operand is A
  int64_t m, k, n;        // reference TTGT shape (free_A, common, free_B)
  int64_t rows_x, rows_y; // GEMM rows of X and Y
  int64_t kp;             // padded K for the tensor-core planes
  int32_t n_common;
  tnc::Operand x, y;
  // split_common_contract panels cut K in A's common order (reference
  // contract.py:58-75, 168-208); when B is the row side, x / y list the
  // commons in B's order (in-place friendly), so the split path uses these
  tnc::Operand sx, sy;
  bool split_alt = false;
  int64_t ldcm, ldcn;      // C[x, y] strides in the (default-order) result
  bool custom_out;         // result order is a different permutation
  std::vector<int64_t> out_perm_dims, out_perm_strides;
  std::vector<int32_t> out_perm;
  int32_t out_rank;
  std::vector<int32_t> out_labels;
  std::vector<int64_t> out_dims;
  // workspace layout (bytes)
  size_t off_x, off_y, off_planes, off_partials, off_tmp, ws_bytes;
  size_t ws_layout;  // bytes of the staged-operand layout (split path); == ws_bytes unless streaming
  tnc::StreamPlan* stream = nullptr;  // TNC_VARIANT_STREAM
  tnc::GatherTcPlan* gt = nullptr;    // TNC_VARIANT_TCGATHER
  int32_t k_splits;
  __int128 multiplies;
  // split-K with in-kernel gather (no operand permutation): packed offset
  // tables [rowx | rowy | tx0 tx1 tx2 | ty0 ty1 ty2], uploaded once per plan
  bool gather_splitk = false;
  int32_t g_levels = 0;
  int64_t g_size[3] = {1, 1, 1};
  int32_t g_x_kfast = 1, g_y_kfast = 1;
  int64_t g_chunks = 1;
  std::vector<int64_t> g_host;
  mutable int64_t* g_dev = nullptr;
  // tensor-core GEMM writing the caller's leg order itself: offset of C[x, y] =
  // out_tab[x] + out_tab[rows_x + y] (the order permutes row legs and column
  // legs, so the offset separates); uploaded once per plan
  bool fuse_out = false;
  std::vector<int64_t> out_tab_host;
  mutable int64_t* out_tab_dev = nullptr;
  ~tnc_plan() {
    if (g_dev) cudaFree(g_dev);
    if (out_tab_dev) cudaFree(out_tab_dev);
    if (stream) tnc::stream_destroy(stream);
    if (gt) tnc::gather_tc_destroy(gt);
  }
};

namespace tnc {
namespace {

constexpr size_t kAlign = 256;
size_t align_up(size_t v) { return (v + kAlign - 1) & ~(kAlign - 1); }

bool checked_mul(int64_t a, int64_t b, int64_t* out) {
  __int128 r = static_cast<__int128>(a) * b;
  if (r > static_cast<__int128>(INT64_MAX)) return false;
  *out = static_cast<int64_t>(r);
  return true;
}

int read_desc(const tnc_tensor_desc* d, std::vector<Leg>& legs) {
  if (!d) TNC_RET(TNC_ERR_INVALID, "null tensor descriptor");
  if (d->rank < 0 || d->rank > TNC_MAX_RANK) TNC_RET(TNC_ERR_TENSOR, "rank out of range");
  legs.clear();
  for (int i = 0; i < d->rank; ++i) {
    if (d->dims[i] < 1) TNC_RET(TNC_ERR_TENSOR, "dim < 1");
    for (auto& l : legs)
      if (l.label == d->labels[i]) TNC_RET(TNC_ERR_TENSOR, "duplicate label in tensor");
    legs.push_back({d->labels[i], d->dims[i], d->strides[i]});
  }
  return TNC_OK;
}

// Is `legs` (in memory order given by strides) a [free..., common...] matrix
// with unit-stride K?  free/common are in the order the GEMM enumerates them.
bool matrix_view(const std::vector<Leg>& free, const std::vector<Leg>& common, int64_t* ld) {
  int64_t expect = 1;
  for (int i = static_cast<int>(common.size()) - 1; i >= 0; --i) {
    if (common[i].dim == 1) continue;
    if (common[i].stride != expect) return false;
    expect *= common[i].dim;
  }
  const int64_t kk = expect;
  // free legs: innermost free stride defines ld, then row-major above it
  int64_t row_stride = -1;
  int64_t fexpect = -1;
  for (int i = static_cast<int>(free.size()) - 1; i >= 0; --i) {
    if (free[i].dim == 1) continue;
    if (fexpect < 0) {
      if (free[i].stride < kk) return false;
      row_stride = free[i].stride;
      fexpect = free[i].stride;
    }
    if (free[i].stride != fexpect) return false;
    fexpect *= free[i].dim;
  }
  *ld = row_stride < 0 ? kk : row_stride;
  return true;
}

void build_gather(Operand& op) {
  // source legs = free then common (each with its stride); output contiguous
  op.dims.clear();
  op.strides.clear();
  op.perm.clear();
  int idx = 0;
  for (auto& l : op.free) {
    op.dims.push_back(l.dim);
    op.strides.push_back(l.stride);
    op.perm.push_back(idx++);
  }
  for (auto& l : op.common) {
    op.dims.push_back(l.dim);
    op.strides.push_back(l.stride);
    op.perm.push_back(idx++);
  }
}

// Offsets of every row of a leg group (first leg most significant).
void group_offsets(const std::vector<Leg>& legs, std::vector<int64_t>& out) {
  out.assign(1, 0);
  for (const Leg& l : legs) {
    std::vector<int64_t> next;
    next.reserve(out.size() * l.dim);
    for (int64_t base : out)
      for (int64_t d = 0; d < l.dim; ++d) next.push_back(base + d * l.stride);
    out.swap(next);
  }
}

// Split-K with the operand gathers folded into the kernel: rows of X / Y are
// small tables, the common legs (X's memory order) are cut into <= 3 levels of
// <= 1024 entries so a K index decodes to 3 table lookups per operand.
bool build_gather_splitk(tnc_plan* p) {
  const Operand& X = p->x;
  const Operand& Y = p->y;
  if (p->rows_x > 64 || p->rows_y > 64 || X.common.empty()) return false;
  const int nc = static_cast<int>(X.common.size());
  std::vector<std::vector<int>> levels;
  int i = nc - 1;
  while (i >= 0 && levels.size() < 3) {
    std::vector<int> idx;
    int64_t prod = 1;
    while (i >= 0 && prod * X.common[i].dim <= 1024) {
      idx.insert(idx.begin(), i);
      prod *= X.common[i].dim;
      --i;
    }
    if (idx.empty()) return false;
    levels.push_back(idx);
  }
  if (i >= 0) return false;
  std::vector<int64_t> rowx, rowy;
  group_offsets(X.free, rowx);
  group_offsets(Y.free, rowy);
  std::vector<int64_t> tx[3], ty[3];
  for (size_t l = 0; l < levels.size(); ++l) {
    std::vector<Leg> lx, ly;
    for (int j : levels[l]) {
      lx.push_back(X.common[j]);
      ly.push_back(Y.common[j]);
    }
    group_offsets(lx, tx[l]);
    group_offsets(ly, ty[l]);
    p->g_size[l] = static_cast<int64_t>(tx[l].size());
  }
  p->g_levels = static_cast<int32_t>(levels.size());
  for (size_t l = levels.size(); l < 3; ++l) {
    tx[l].assign(1, 0);
    ty[l].assign(1, 0);
    p->g_size[l] = 1;
  }
  auto min_free = [](const Operand& o) {
    int64_t s = INT64_MAX;
    for (const Leg& l : o.free)
      if (l.dim > 1) s = std::min(s, l.stride);
    return s;
  };
  p->g_x_kfast = X.common.back().stride < min_free(X) ? 1 : 0;
  p->g_y_kfast = Y.common.back().stride < min_free(Y) ? 1 : 0;
  p->g_host.clear();
  for (auto* v : {&rowx, &rowy, &tx[0], &tx[1], &tx[2], &ty[0], &ty[1], &ty[2]})
    p->g_host.insert(p->g_host.end(), v->begin(), v->end());
  const int64_t target = static_cast<int64_t>(num_sms()) * 4;
  int64_t kc = ceil_div(p->k, target);
  kc = std::max<int64_t>(64, ceil_div(kc, 64) * 64);
  p->g_chunks = ceil_div(p->k, kc);
  if (upload_table(p->g_host.data(), p->g_host.size(), &p->g_dev) != TNC_OK) return false;
  p->gather_splitk = true;
  return true;
}

int env_flag(const char* name, int dflt) {
  const char* v = std::getenv(name);
  return v ? std::atoi(v) : dflt;
}

// 3xFP16 (2x-rate kind::f16, half the operand bytes) unless TNC_TC_TF32=1
int default_tc_variant() {
  const char* v = std::getenv("TNC_TC_TF32");
  return (v && std::atoi(v) != 0) ? TNC_VARIANT_TC3XTF32 : TNC_VARIANT_TC3XF16;
}

// K5 streaming path: every leg of extent 2 (extent-1 legs are dropped), a
// small Y (rows_y * K <= 4096) and a large X.  Builds the kernel tables with
// the FINAL output strides, so the result needs no separate permutation.
int try_stream(tnc_plan* p, const std::vector<Leg>& free_a, const std::vector<Leg>& free_b) {
  if (p->dtype != TNC_C64) return TNC_ERR_UNSUPPORTED;
  const Operand& X = p->x;
  const Operand& Y = p->y;
  for (const auto* v : {&X.free, &X.common, &Y.free, &Y.common})
    for (const Leg& l : *v)
      if (l.dim != 1 && l.dim != 2) return TNC_ERR_UNSUPPORTED;
  if (p->rows_y * p->k > 4096) return TNC_ERR_UNSUPPORTED;
  // final output strides by label
  std::vector<Leg> order;
  if (p->custom_out) {
    std::vector<Leg> def_out = free_a;
    def_out.insert(def_out.end(), free_b.begin(), free_b.end());
    for (int32_t i : p->out_perm) order.push_back(def_out[i]);
  } else {
    order = free_a;
    order.insert(order.end(), free_b.begin(), free_b.end());
  }
  auto out_stride = [&](int32_t label) {
    int64_t s = 1;
    for (int i = static_cast<int>(order.size()) - 1; i >= 0; --i) {
      if (order[i].label == label) return s;
      s *= order[i].dim;
    }
    return static_cast<int64_t>(-1);
  };
  std::vector<StreamLeg> legs;
  for (const Leg& l : X.free)
    if (l.dim == 2) legs.push_back({0, l.stride, 0, out_stride(l.label)});
  for (size_t i = 0; i < X.common.size(); ++i)
    if (X.common[i].dim == 2) legs.push_back({1, X.common[i].stride, Y.common[i].stride, 0});
  for (const Leg& l : Y.free)
    if (l.dim == 2) legs.push_back({2, 0, l.stride, out_stride(l.label)});
  return stream_prepare(static_cast<int>(legs.size()), legs.data(), &p->stream);
}

// Final output stride of every free leg (the caller's order when given).
std::vector<std::pair<int32_t, int64_t>> final_out_strides(const tnc_plan* p, const std::vector<Leg>& free_a,
                                                           const std::vector<Leg>& free_b) {
  std::vector<Leg> order;
  if (p->custom_out) {
    std::vector<Leg> def_out = free_a;
    def_out.insert(def_out.end(), free_b.begin(), free_b.end());
    for (int32_t i : p->out_perm) order.push_back(def_out[i]);
  } else {
    order = free_a;
    order.insert(order.end(), free_b.begin(), free_b.end());
  }
  std::vector<std::pair<int32_t, int64_t>> out;
  int64_t s = 1;
  for (int i = static_cast<int>(order.size()) - 1; i >= 0; --i) {
    out.push_back({order[i].label, s});
    s *= order[i].dim;
  }
  return out;
}

// K6 gather-fed tensor-core path: c64, every leg of extent <= 2, rows_y <= 128,
// rows_x >= 64, K >= one k-block.  Both operands are read in place.
int try_gather_tc(tnc_plan* p, const std::vector<Leg>& free_a, const std::vector<Leg>& free_b) {
  if (p->dtype != TNC_C64) return TNC_ERR_UNSUPPORTED;
  const Operand& X = p->x;
  const Operand& Y = p->y;
  for (const auto* v : {&X.free, &X.common, &Y.free, &Y.common})
    for (const Leg& l : *v)
      if (l.dim != 1 && l.dim != 2) return TNC_ERR_UNSUPPORTED;
  const auto outs = final_out_strides(p, free_a, free_b);
  auto out_stride = [&](int32_t label) {
    for (auto& o : outs)
      if (o.first == label) return o.second;
    return static_cast<int64_t>(-1);
  };
  std::vector<GatherTcLeg> legs;
  int64_t canon = 1;  // Y-free legs: canonical column index, last leg fastest
  for (int i = static_cast<int>(Y.free.size()) - 1; i >= 0; --i) {
    const Leg& l = Y.free[i];
    if (l.dim == 2) legs.push_back({2, 0, l.stride, out_stride(l.label), canon});
    canon *= l.dim;
  }
  canon = p->rows_y;  // X-free legs: canonical row index times rows_y
  for (int i = static_cast<int>(X.free.size()) - 1; i >= 0; --i) {
    const Leg& l = X.free[i];
    if (l.dim == 2) legs.push_back({0, l.stride, 0, out_stride(l.label), canon});
    canon *= l.dim;
  }
  for (size_t i = 0; i < X.common.size(); ++i)
    if (X.common[i].dim == 2) legs.push_back({1, X.common[i].stride, Y.common[i].stride, 0, 0});
  return gather_tc_prepare(static_cast<int>(legs.size()), legs.data(), &p->gt);
}

bool tc_eligible(const tnc_plan* p) {
  return p->dtype == TNC_C64 && p->rows_x >= 128 && p->rows_y >= 32 && p->k >= 8 &&
         static_cast<__int128>(p->rows_x) * p->rows_y * p->k >= (static_cast<__int128>(1) << 26);
}

}  // namespace
}  // namespace tnc

using namespace tnc;

extern "C" {

int tnc_abi_version(void) { return TNC_ABI_VERSION; }

int64_t tnc_launch_count(void) { return g_launches.load(); }

int tnc_profile_enable(int on) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventDestroy(r.start);
    cudaEventDestroy(r.stop);
  }
  g_prof.clear();
  g_prof_on.store(on != 0);
  return TNC_OK;
}

int tnc_profile_read(int32_t kind, int64_t* launches, double* total_ms, double* flops,
                     double* bytes) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  int64_t n = 0;
  double ms = 0, fl = 0, by = 0;
  for (auto& r : g_prof) {
    if (r.kind != kind) continue;
    TNC_CUDA_TRY(cudaEventSynchronize(r.stop));
    float t = 0.f;
    TNC_CUDA_TRY(cudaEventElapsedTime(&t, r.start, r.stop));
    ++n;
    ms += t;
    fl += r.flops;
    by += r.bytes;
  }
  if (launches) *launches = n;
  if (total_ms) *total_ms = ms;
  if (flops) *flops = fl;
  if (bytes) *bytes = by;
  return TNC_OK;
}

const char* tnc_last_error(void) { return tnc::last_error(); }

int tnc_init(int device) {
  TNC_CUDA_TRY(cudaSetDevice(device));
  TNC_CUDA_TRY(cudaFree(nullptr));
  return TNC_OK;
}

// Releases the library's process-wide state (profiling events); device
// buffers owned by plans are released by tnc_plan_destroy.  Safe to call
// more than once; the library stays usable (tnc_init again).
void tnc_shutdown(void) {
  tnc_profile_enable(0);
  tnc::absorb_shutdown();
  cudaGetLastError();  // clear a sticky launch error from a failed call
}

int tnc_device_info(int* sm_count, int* cc_major, int* cc_minor, size_t* smem_optin) {
  int dev = 0;
  TNC_CUDA_TRY(cudaGetDevice(&dev));
  cudaDeviceProp prop;
  TNC_CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
  if (sm_count) *sm_count = prop.multiProcessorCount;
  if (cc_major) *cc_major = prop.major;
  if (cc_minor) *cc_minor = prop.minor;
  if (smem_optin) *smem_optin = prop.sharedMemPerBlockOptin;
  return TNC_OK;
}

int tnc_permute(int32_t dtype, int32_t rank, const int64_t* dims, const int64_t* in_strides,
                const int32_t* perm, const void* in, void* out, void* stream) {
  if (dtype != TNC_C64 && dtype != TNC_C128) TNC_RET(TNC_ERR_INVALID, "permute: bad dtype");
  return permute_launch(dtype, rank, dims, in_strides, perm, in, out,
                        static_cast<cudaStream_t>(stream));
}

int tnc_axpy(int32_t dtype, int64_t n, const void* x, void* y, void* stream) {
  return axpy_launch(dtype, n, x, y, static_cast<cudaStream_t>(stream));
}

int tnc_plan_contract(const tnc_tensor_desc* a, const tnc_tensor_desc* b, int32_t out_rank,
                      const int32_t* out_labels, int32_t variant, tnc_plan** plan_out) {
  if (!plan_out) TNC_RET(TNC_ERR_INVALID, "null plan pointer");
  *plan_out = nullptr;
  std::vector<Leg> la, lb;
  TNC_TRY(read_desc(a, la));
  TNC_TRY(read_desc(b, lb));
  if (a->dtype != b->dtype) TNC_RET(TNC_ERR_INVALID, "operand dtypes differ");
  if (a->dtype != TNC_C64 && a->dtype != TNC_C128) TNC_RET(TNC_ERR_INVALID, "bad dtype");
  std::vector<Leg> free_a, common_a, free_b, common_b;
  for (auto& l : la) {
    const Leg* twin = nullptr;
    for (auto& r : lb)
      if (r.label == l.label) twin = &r;
    if (!twin) {
      free_a.push_back(l);
    } else {
      if (twin->dim != l.dim) TNC_RET(TNC_ERR_CONTRACTION, "shared label has mismatched dims");
      common_a.push_back(l);
      common_b.push_back(*twin);
    }
  }
  for (auto& r : lb) {
    bool shared = false;
    for (auto& l : la) shared |= (l.label == r.label);
    if (!shared) free_b.push_back(r);
  }
  auto* p = new tnc_plan();
  p->dtype = a->dtype;
  p->n_common = static_cast<int32_t>(common_a.size());
  int64_t m = 1, k = 1, n = 1;
  bool ok = true;
  for (auto& l : free_a) ok &= checked_mul(m, l.dim, &m);
  for (auto& l : common_a) ok &= checked_mul(k, l.dim, &k);
  for (auto& l : free_b) ok &= checked_mul(n, l.dim, &n);
  int64_t tmp;
  ok &= checked_mul(m, n, &tmp);
  if (!ok) {
    delete p;
    TNC_RET(TNC_ERR_TENSOR, "contraction extent overflows int64");
  }
  p->m = m;
  p->k = k;
  p->n = n;
  p->multiplies = static_cast<__int128>(m) * k * n;
  // reference multiplier choice (ties resolved by the caller's label strings)
  p->b_is_multiplier = (k * n > m * k) ? 1 : 0;
  // row side X = larger operand (ties: A)
  p->x_is_a = (k * n > m * k) ? 0 : 1;
  Operand& X = p->x;
  Operand& Y = p->y;
  if (p->x_is_a) {
    X.free = free_a;
    X.common = common_a;
    Y.free = free_b;
    Y.common = common_b;  // already listed in A's common order
  } else {
    // common order = B's own order; reorder A's commons accordingly
    X.free = free_b;
    Y.free = free_a;
    for (auto& r : lb)
      for (size_t i = 0; i < common_b.size(); ++i)
        if (common_b[i].label == r.label) {
          X.common.push_back(common_b[i]);
          Y.common.push_back(common_a[i]);
        }
  }
  p->rows_x = p->x_is_a ? m : n;
  p->rows_y = p->x_is_a ? n : m;
  if (!p->x_is_a && common_a.size() > 1) {
    p->split_alt = true;
    p->sx.free = free_b;
    p->sy.free = free_a;
    p->sx.common = common_b;  // listed in A's common order
    p->sy.common = common_a;
    for (Operand* op : {&p->sx, &p->sy}) {
      int64_t rows = 1;
      for (auto& l : op->free) rows *= l.dim;
      op->rows = rows;
      op->in_place = matrix_view(op->free, op->common, &op->ld);
      if (!op->in_place) {
        build_gather(*op);
        op->ld = k;
      }
    }
  }
  for (Operand* op : {&X, &Y}) {
    int64_t rows = 1;
    for (auto& l : op->free) rows *= l.dim;
    op->rows = rows;
    op->in_place = matrix_view(op->free, op->common, &op->ld);
    if (!op->in_place) {
      build_gather(*op);
      op->ld = k;
    }
  }
  // output order
  std::vector<Leg> def_out;  // default order free_A ++ free_B with contiguous strides
  for (auto& l : free_a) def_out.push_back(l);
  for (auto& l : free_b) def_out.push_back(l);
  p->custom_out = false;
  if (out_rank >= 0) {
    if (out_rank != static_cast<int32_t>(def_out.size())) {
      delete p;
      TNC_RET(TNC_ERR_PERMUTATION, "output labels are not a permutation of the free legs");
    }
    std::vector<int> used(def_out.size(), 0);
    for (int t = 0; t < out_rank; ++t) {
      int found = -1;
      for (size_t i = 0; i < def_out.size(); ++i)
        if (def_out[i].label == out_labels[t] && !used[i]) found = static_cast<int>(i);
      if (found < 0) {
        delete p;
        TNC_RET(TNC_ERR_PERMUTATION, "output labels are not a permutation of the free legs");
      }
      used[found] = 1;
      p->out_perm.push_back(found);
      if (found != t) p->custom_out = true;
    }
  }
  p->out_rank = static_cast<int32_t>(def_out.size());
  if (p->custom_out) {
    for (int t = 0; t < p->out_rank; ++t) {
      p->out_labels.push_back(def_out[p->out_perm[t]].label);
      p->out_dims.push_back(def_out[p->out_perm[t]].dim);
    }
    int64_t s = 1;
    std::vector<int64_t> st(def_out.size());
    for (int i = static_cast<int>(def_out.size()) - 1; i >= 0; --i) {
      st[i] = s;
      s *= def_out[i].dim;
    }
    for (auto& l : def_out) p->out_perm_dims.push_back(l.dim);
    p->out_perm_strides = st;
  } else {
    for (auto& l : def_out) {
      p->out_labels.push_back(l.label);
      p->out_dims.push_back(l.dim);
    }
  }
  // default-order C strides for C[x_row, y_row]
  if (p->x_is_a) {
    p->ldcm = n;
    p->ldcn = 1;
  } else {
    p->ldcm = 1;  // x enumerates free_B (fastest in free_A ++ free_B)
    p->ldcn = n;
  }
  // variant
  int want = variant;
  if (want == TNC_VARIANT_AUTO) {
    if (p->rows_x * p->rows_y <= 1024 && k >= 4096)
      want = TNC_VARIANT_SPLITK;  // tiny output, huge K: CUDA-core split-K reduction
    else
      want = tc_eligible(p) ? default_tc_variant() : TNC_VARIANT_SIMT;
    // short K: 3xFP16 pads K to 32 (64 fp16 per 128B row); 3xTF32 pads to 16
    if (want == TNC_VARIANT_TC3XF16 && k <= 16) want = TNC_VARIANT_TC3XTF32;
  }
  const bool tc = want == TNC_VARIANT_TC3XTF32 || want == TNC_VARIANT_TC3XF16;
  if (tc && p->dtype != TNC_C64) {
    delete p;
    TNC_RET(TNC_ERR_UNSUPPORTED, "tensor-core variant needs complex64");
  }
  if (want == TNC_VARIANT_STREAM || (variant == TNC_VARIANT_AUTO && want != TNC_VARIANT_SPLITK &&
                                       p->rows_x >= 4096 && (p->rows_y <= 16 || !tc_eligible(p)))) {
    const int st = try_stream(p, free_a, free_b);
    if (st == TNC_OK) {
      want = TNC_VARIANT_STREAM;
    } else if (want == TNC_VARIANT_STREAM) {
      delete p;
      return st;
    }
  }
  // K6 (operands gathered in-kernel, tensor cores) takes over the CUDA-core
  // split-K, the streaming kernel and the tensor-core steps that are narrow
  // (<= 64 Y columns: the permute + split passes over X cost more than the
  // GEMM) or split-K shaped (one row of 128-row tiles per SM at most)
  // whenever the step fits its envelope.  TNC_TCGATHER=0 disables it.
  if (variant == TNC_VARIANT_AUTO && p->dtype == TNC_C64 && env_flag("TNC_TCGATHER", 1) &&
      (want == TNC_VARIANT_SPLITK || want == TNC_VARIANT_STREAM ||
       (tc && (p->rows_y <= 64 || p->rows_x <= 128 * static_cast<int64_t>(num_sms())))) &&
      p->rows_x >= 64 && p->rows_y <= 128 && k >= 16) {
    if (try_gather_tc(p, free_a, free_b) == TNC_OK) {
      if (p->stream) {
        stream_destroy(p->stream);
        p->stream = nullptr;
      }
      want = TNC_VARIANT_TCGATHER;
    }
  } else if (want == TNC_VARIANT_TCGATHER) {
    const int st = try_gather_tc(p, free_a, free_b);
    if (st != TNC_OK) {
      delete p;
      return st;
    }
  }
  p->variant = want;
  if (want == TNC_VARIANT_SPLITK && build_gather_splitk(p)) {
    X.in_place = Y.in_place = true;  // the kernel gathers from the original strides
  }
  p->kp = want == TNC_VARIANT_TC3XF16 ? ((k + 31) / 32) * 32 : ((k + 15) / 16) * 16;
  // split-K when the output tile grid cannot fill the machine
  p->k_splits = 1;
  if (tc) {
    const int64_t bn = (2 * p->rows_y >= 256) ? 256 : 128;
    const int64_t tiles = ceil_div(2 * p->rows_y, bn) * ceil_div(p->rows_x, 128);
    const int64_t kblocks = 2 * p->kp / 64;
    const int sms = num_sms();
    if (tiles < sms && kblocks >= 8) {
      int64_t want_splits = std::min<int64_t>(sms / tiles, kblocks / 4);
      p->k_splits = static_cast<int32_t>(std::max<int64_t>(1, want_splits));
    }
    if (const char* env = std::getenv("TNC_KSPLIT")) {  // experiment override
      const int64_t forced = std::atoll(env);
      if (forced >= 1) p->k_splits = static_cast<int32_t>(std::min<int64_t>(forced, kblocks));
    }
  }
  // K2 with one split writes a custom output order from its epilogue (no
  // temporary, no output permutation pass): per-row and per-column offsets
  if (p->custom_out && tc && p->k_splits == 1 && p->rows_x + p->rows_y <= (int64_t{1} << 22) &&
      env_flag("TNC_FUSE_OUT", 1) && !(std::getenv("TNC_TC_CFG") && std::atoi(std::getenv("TNC_TC_CFG")) == 2)) {
    const auto outs = final_out_strides(p, free_a, free_b);
    auto stride_of = [&](int32_t label) {
      for (const auto& e : outs)
        if (e.first == label) return e.second;
      return int64_t{0};
    };
    auto fill = [&](const std::vector<Leg>& legs, int64_t rows, int64_t* dst) {
      // row-major over the legs, last leg fastest
      for (int64_t r = 0; r < rows; ++r) {
        int64_t rem = r, off = 0;
        for (int i = static_cast<int>(legs.size()) - 1; i >= 0; --i) {
          off += (rem % legs[i].dim) * stride_of(legs[i].label);
          rem /= legs[i].dim;
        }
        dst[r] = off;
      }
    };
    p->out_tab_host.assign(static_cast<size_t>(p->rows_x + p->rows_y), 0);
    fill(X.free, p->rows_x, p->out_tab_host.data());
    fill(Y.free, p->rows_y, p->out_tab_host.data() + p->rows_x);
    if (upload_table(p->out_tab_host.data(), p->out_tab_host.size(), &p->out_tab_dev) != TNC_OK) {
      delete p;
      return TNC_ERR_CUDA;
    }
    p->fuse_out = true;
  }
  // workspace
  const size_t eb = elem_bytes(p->dtype);
  const bool kernel_gathers = want == TNC_VARIANT_TCGATHER;  // operands read in place
  size_t off = 0;
  p->off_x = off;
  if (!X.in_place && !kernel_gathers) off = align_up(off + static_cast<size_t>(p->rows_x) * k * eb);
  p->off_y = off;
  if (!Y.in_place && !kernel_gathers) off = align_up(off + static_cast<size_t>(p->rows_y) * k * eb);
  p->off_planes = off;
  if (tc) {
    const size_t pe = p->variant == TNC_VARIANT_TC3XF16 ? 2 : 4;
    const size_t a_plane = align_up(static_cast<size_t>(p->rows_x) * 2 * p->kp * pe);
    const size_t b_plane = align_up(static_cast<size_t>(2 * p->rows_y) * 2 * p->kp * pe);
    off = align_up(off + 2 * a_plane + 2 * b_plane + align_up(4 * p->rows_x) + align_up(4 * p->rows_y) +
                   4 * std::max(p->rows_x, p->rows_y));
  }
  p->off_partials = off;
  if (p->k_splits > 1) off = align_up(off + static_cast<size_t>(p->k_splits) * m * n * 8);
  if (kernel_gathers && gather_tc_splits(p->gt) > 1)
    off = align_up(off + static_cast<size_t>(gather_tc_splits(p->gt)) * m * n * 8);
  if (p->variant == TNC_VARIANT_SPLITK) {
    const int64_t chunks = p->gather_splitk ? p->g_chunks : splitk_chunks(p->rows_x, p->rows_y, k);
    off = align_up(off + static_cast<size_t>(chunks) * m * n * eb);
  }
  p->off_tmp = off;
  if (p->custom_out && !p->fuse_out && !(kernel_gathers && gather_tc_splits(p->gt) == 1))
    off = align_up(off + static_cast<size_t>(m) * n * eb);
  p->ws_bytes = off;
  p->ws_layout = off;
  if (want == TNC_VARIANT_STREAM) p->ws_bytes = 0;  // reads A/B in place, writes C in final order
  *plan_out = p;
  return TNC_OK;
}

int tnc_plan_get_info(const tnc_plan* p, tnc_plan_info* info) {
  if (!p || !info) TNC_RET(TNC_ERR_INVALID, "null argument");
  std::memset(info, 0, sizeof(*info));
  info->m = p->m;
  info->k = p->k;
  info->n = p->n;
  info->n_common = p->n_common;
  info->variant = p->variant;
  info->b_is_multiplier = p->b_is_multiplier;
  info->out_rank = p->out_rank;
  for (int i = 0; i < p->out_rank; ++i) {
    info->out_labels[i] = p->out_labels[i];
    info->out_dims[i] = p->out_dims[i];
  }
  info->workspace_bytes = p->ws_bytes;
  info->multiplies_lo = p->multiplies > static_cast<__int128>(INT64_MAX)
                            ? INT64_MAX
                            : static_cast<int64_t>(p->multiplies);
  return TNC_OK;
}

void tnc_plan_destroy(tnc_plan* p) { delete p; }

static int prep_operand(const tnc_plan* p, const Operand& op, const void* src, uint8_t* ws,
                        size_t off, const void** mat, int64_t* ld, cudaStream_t st) {
  if (op.in_place) {
    *mat = src;
    *ld = op.ld;
    return TNC_OK;
  }
  void* dst = ws + off;
  TNC_TRY(permute_launch(p->dtype, static_cast<int>(op.dims.size()), op.dims.data(),
                         op.strides.data(), op.perm.data(), src, dst, st));
  *mat = dst;
  *ld = p->k;
  return TNC_OK;
}

// 3xFP16 plane pointers inside a plan's workspace
struct F16Planes {
  uint8_t *ab, *as, *bb, *bs;
  int *ex, *ey;
  void* scratch;
};

static F16Planes f16_planes(const tnc_plan* p, uint8_t* ws) {
  const size_t a_plane = align_up(static_cast<size_t>(p->rows_x) * 2 * p->kp * 2);
  const size_t b_plane = align_up(static_cast<size_t>(2 * p->rows_y) * 2 * p->kp * 2);
  F16Planes f;
  f.ab = ws + p->off_planes;
  f.as = f.ab + a_plane;
  f.bb = f.as + a_plane;
  f.bs = f.bb + b_plane;
  f.ex = reinterpret_cast<int*>(f.bs + b_plane);
  f.ey = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(f.ex) + align_up(4 * p->rows_x));
  f.scratch = reinterpret_cast<uint8_t*>(f.ey) + align_up(4 * p->rows_y);
  return f;
}

// A gathered 3xFP16 operand goes straight from its own layout to the planes
// (one tiled pass pair, no permuted copy) when K is a power of two >= 32.
// Returns true when the planes were written.
static bool fused_gather_split(const tnc_plan* p, const Operand& op, const void* src, int mode, int64_t rows,
                               uint8_t* hi, uint8_t* lo, int* exps, void* scratch, cudaStream_t st) {
  if (op.in_place || p->variant != TNC_VARIANT_TC3XF16 || p->kp != p->k || p->dtype != TNC_C64) return false;
  if ((p->k & (p->k - 1)) != 0 || std::getenv("TNC_NO_FUSED_SPLIT")) return false;
  int log_k = 0;
  while ((int64_t{1} << log_k) < p->k) ++log_k;
  return permute_split_f16_launch(static_cast<int>(op.dims.size()), op.dims.data(), op.strides.data(),
                                  op.perm.data(), src, mode, rows, log_k, hi, lo, exps,
                                  static_cast<unsigned*>(scratch), st) == TNC_OK;
}

static int run_gemm(const tnc_plan* p, const void* xm, int64_t ldx, const void* ym, int64_t ldy,
                    void* c, int64_t ldcm, int64_t ldcn, uint8_t* ws, int k_splits,
                    cudaStream_t st, bool x_planes_done = false, bool y_planes_done = false,
                    const int64_t* row_off = nullptr, const int64_t* col_off = nullptr) {
  if (p->variant == TNC_VARIANT_TC3XTF32 || p->variant == TNC_VARIANT_TC3XF16) {
    const bool f16 = p->variant == TNC_VARIANT_TC3XF16;
    const size_t pe = f16 ? 2 : 4;
    const size_t a_plane = align_up(static_cast<size_t>(p->rows_x) * 2 * p->kp * pe);
    const size_t b_plane = align_up(static_cast<size_t>(2 * p->rows_y) * 2 * p->kp * pe);
    uint8_t* ab = ws + p->off_planes;
    uint8_t* as = ab + a_plane;
    uint8_t* bb = as + a_plane;
    uint8_t* bs = bb + b_plane;
    int* ex = reinterpret_cast<int*>(bs + b_plane);
    int* ey = reinterpret_cast<int*>(reinterpret_cast<uint8_t*>(ex) + align_up(4 * p->rows_x));
    if (f16) {
      void* scratch = reinterpret_cast<uint8_t*>(ey) + align_up(4 * p->rows_y);
      if (!x_planes_done) TNC_TRY(f16_split_launch(0, p->rows_x, p->k, p->kp, xm, ldx, ab, as, ex, scratch, st));
      if (!y_planes_done) TNC_TRY(f16_split_launch(1, p->rows_y, p->k, p->kp, ym, ldy, bb, bs, ey, scratch, st));
    } else {
      TNC_TRY(tf32_split_launch(0, p->rows_x, p->k, p->kp, xm, ldx, ab, as, st));
      TNC_TRY(tf32_split_launch(1, p->rows_y, p->k, p->kp, ym, ldy, bb, bs, st));
    }
    return tc_cgemm_launch(f16 ? 1 : 0, p->rows_x, p->rows_y, p->k, p->kp, ab, as, bb, bs,
                           f16 ? ex : nullptr, f16 ? ey : nullptr, c, ldcm, ldcn, k_splits,
                           reinterpret_cast<float*>(ws + p->off_partials), st, row_off, col_off);
  }
  if (p->variant == TNC_VARIANT_SPLITK && p->gather_splitk) {
    if (!p->g_dev) TNC_RET(TNC_ERR_INVALID, "split-K gather: plan tables missing");
    return splitk_gather_launch(p->dtype, p->rows_x, p->rows_y, p->k, xm, ym, p->g_dev, p->g_size,
                                p->g_x_kfast, p->g_y_kfast, p->g_chunks, c, ldcm, ldcn,
                                ws + p->off_partials, st);
  }
  if (p->variant == TNC_VARIANT_SPLITK)
    return simt_splitk_launch(p->dtype, p->rows_x, p->rows_y, p->k, xm, ldx, ym, ldy, c, ldcm, ldcn,
                              ws + p->off_partials, st);
  return simt_cgemm_launch(p->dtype, p->rows_x, p->rows_y, p->k, xm, ldx, ym, ldy, c, ldcm, ldcn,
                           0, st);
}

int tnc_contract(const tnc_plan* p, const void* a, const void* b, void* c, void* workspace,
                 size_t ws_bytes, void* stream) {
  if (!p) TNC_RET(TNC_ERR_INVALID, "null plan");
  if (ws_bytes < p->ws_bytes) TNC_RET(TNC_ERR_WORKSPACE, "workspace smaller than plan requires");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const void* xsrc = p->x_is_a ? a : b;
  const void* ysrc = p->x_is_a ? b : a;
  if (p->variant == TNC_VARIANT_STREAM) return stream_launch(p->stream, xsrc, ysrc, c, st);
  if (p->variant == TNC_VARIANT_TCGATHER) {
    const int splits = gather_tc_splits(p->gt);
    if (splits == 1) return gather_tc_launch(p->gt, xsrc, ysrc, c, nullptr, st);
    void* parts = ws + p->off_partials;
    TNC_TRY(gather_tc_launch(p->gt, xsrc, ysrc, nullptr, parts, st));
    void* dst = p->custom_out ? static_cast<void*>(ws + p->off_tmp) : c;
    TNC_TRY(tree_reduce_launch(TNC_C64, splits, p->rows_x * p->rows_y, parts, dst, p->rows_x, p->rows_y,
                               p->ldcm, p->ldcn, st));
    if (p->custom_out)
      TNC_TRY(permute_launch(p->dtype, static_cast<int>(p->out_perm.size()), p->out_perm_dims.data(),
                             p->out_perm_strides.data(), p->out_perm.data(), dst, c, st));
    return TNC_OK;
  }
  const void *xm = nullptr, *ym = nullptr;
  int64_t ldx = 0, ldy = 0;
  bool x_done = false, y_done = false;
  if (p->variant == TNC_VARIANT_TC3XF16) {
    const F16Planes f = f16_planes(p, ws);
    x_done = fused_gather_split(p, p->x, xsrc, 0, p->rows_x, f.ab, f.as, f.ex, f.scratch, st);
    y_done = fused_gather_split(p, p->y, ysrc, 1, p->rows_y, f.bb, f.bs, f.ey, f.scratch, st);
  }
  if (!x_done) TNC_TRY(prep_operand(p, p->x, xsrc, ws, p->off_x, &xm, &ldx, st));
  if (!y_done) TNC_TRY(prep_operand(p, p->y, ysrc, ws, p->off_y, &ym, &ldy, st));
  if (p->fuse_out) {
    if (!p->out_tab_dev) TNC_RET(TNC_ERR_INVALID, "contract: plan output tables missing");
    return run_gemm(p, xm, ldx, ym, ldy, c, p->ldcm, p->ldcn, ws, p->k_splits, st, x_done, y_done,
                    p->out_tab_dev, p->out_tab_dev + p->rows_x);
  }
  void* dst = p->custom_out ? static_cast<void*>(ws + p->off_tmp) : c;
  TNC_TRY(run_gemm(p, xm, ldx, ym, ldy, dst, p->ldcm, p->ldcn, ws, p->k_splits, st, x_done, y_done));
  if (p->custom_out) {
    TNC_TRY(permute_launch(p->dtype, static_cast<int>(p->out_perm.size()),
                           p->out_perm_dims.data(), p->out_perm_strides.data(),
                           p->out_perm.data(), dst, c, st));
  }
  return TNC_OK;
}

int tnc_contract_split_workspace(const tnc_plan* p, int32_t blocks, int32_t group,
                                 size_t* workspace_bytes) {
  if (!p || !workspace_bytes) TNC_RET(TNC_ERR_INVALID, "null argument");
  if (p->variant == TNC_VARIANT_TCGATHER)
    TNC_RET(TNC_ERR_UNSUPPORTED, "split contraction needs a staged (non-gather) plan");
  if (blocks < 1 || group < 1) TNC_RET(TNC_ERR_CONTRACTION, "blocks*group_size must be positive");
  const int64_t panels = std::min<int64_t>(static_cast<int64_t>(blocks) * group, p->k);
  const size_t eb = elem_bytes(p->dtype);
  size_t need = align_up(p->ws_layout) + align_up(static_cast<size_t>(panels) * p->m * p->n * eb);
  // operand gathers are always materialised for the split path
  need += align_up(static_cast<size_t>(p->rows_x) * p->k * eb) +
          align_up(static_cast<size_t>(p->rows_y) * p->k * eb);
  *workspace_bytes = need;
  return TNC_OK;
}

int tnc_contract_split(const tnc_plan* p, int32_t blocks, int32_t group, const void* a,
                       const void* b, void* c, void* workspace, size_t ws_bytes, void* stream) {
  size_t need = 0;
  TNC_TRY(tnc_contract_split_workspace(p, blocks, group, &need));
  if (ws_bytes < need) TNC_RET(TNC_ERR_WORKSPACE, "workspace smaller than split plan requires");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  const int64_t panels = std::min<int64_t>(static_cast<int64_t>(blocks) * group, p->k);
  const int64_t base = p->k / panels;
  const size_t eb = elem_bytes(p->dtype);
  uint8_t* parts = ws + align_up(p->ws_layout);
  const void* xsrc = p->x_is_a ? a : b;
  const void* ysrc = p->x_is_a ? b : a;
  const void *xm, *ym;
  int64_t ldx, ldy;
  // operands staged after the panel partials (K in A's common order)
  const size_t off_sx = align_up(p->ws_layout) + align_up(static_cast<size_t>(panels) * p->m * p->n * eb);
  const size_t off_sy = off_sx + align_up(static_cast<size_t>(p->rows_x) * p->k * eb);
  TNC_TRY(prep_operand(p, p->split_alt ? p->sx : p->x, xsrc, ws, off_sx, &xm, &ldx, st));
  TNC_TRY(prep_operand(p, p->split_alt ? p->sy : p->y, ysrc, ws, off_sy, &ym, &ldy, st));
  const int64_t mn = p->m * p->n;
  // each panel accumulates independently into its own [rows_x, rows_y] tile
  for (int64_t i = 0; i < panels; ++i) {
    const int64_t lo = i * base;
    const int64_t hi = (i == panels - 1) ? p->k : lo + base;
    const uint8_t* xp = static_cast<const uint8_t*>(xm) + static_cast<size_t>(lo) * eb;
    const uint8_t* yp = static_cast<const uint8_t*>(ym) + static_cast<size_t>(lo) * eb;
    void* dst = parts + static_cast<size_t>(i) * mn * eb;
    TNC_TRY(simt_cgemm_launch(p->dtype, p->rows_x, p->rows_y, hi - lo, xp, ldx, yp, ldy, dst,
                              p->rows_y, 1, 0, st));
  }
  // combine with the fixed pairwise tree, then place into the output layout
  void* dst = p->custom_out ? static_cast<void*>(ws + p->off_tmp) : c;
  TNC_TRY(tree_reduce_launch(p->dtype, panels, mn, parts, dst, p->rows_x, p->rows_y, p->ldcm,
                             p->ldcn, st));
  if (p->custom_out) {
    TNC_TRY(permute_launch(p->dtype, static_cast<int>(p->out_perm.size()),
                           p->out_perm_dims.data(), p->out_perm_strides.data(),
                           p->out_perm.data(), dst, c, st));
  }
  return TNC_OK;
}

int tnc_absorb_chain_workspace(int32_t t_rank, int32_t n_gates, const int32_t* axes,
                               size_t* workspace_bytes) {
  if (!workspace_bytes) TNC_RET(TNC_ERR_INVALID, "null argument");
  return absorb_chain_workspace(t_rank, n_gates, axes, workspace_bytes);
}

int tnc_absorb_chain(int32_t t_rank, const void* t_in, void* t_out, int32_t n_gates,
                     const void* const* gates, const int64_t* gate_strides, const int32_t* axes,
                     void* workspace, size_t workspace_bytes, void* stream) {
  if (n_gates > 0 && (!gates || !gate_strides || !axes)) TNC_RET(TNC_ERR_INVALID, "null argument");
  if (!t_in || !t_out || t_in == t_out) TNC_RET(TNC_ERR_INVALID, "absorb: t_in / t_out null or aliased");
  return absorb_chain_launch(t_rank, t_in, t_out, n_gates, gates, gate_strides, axes, workspace,
                             workspace_bytes, static_cast<cudaStream_t>(stream));
}

int tnc_absorb_chain_info(int32_t t_rank, int32_t n_gates, const int32_t* axes, int32_t* passes,
                          int32_t* groups) {
  if (!passes || !groups || (n_gates > 0 && !axes)) TNC_RET(TNC_ERR_INVALID, "null argument");
  int p = 0, g = 0;
  TNC_TRY(absorb_chain_passes(t_rank, n_gates, axes, &p, &g));
  *passes = p;
  *groups = g;
  return TNC_OK;
}

}  // extern "C"
