/*
 * tnc_b200.h -- C-ABI of the B200 tensor-network-contraction hot path.
 *
 * One shared library (paper_2504_09186_b200/libtnc_b200.so), extern "C",
 * plain pointers and sizes only.  The reference (tncsim, pure Python) has no
 * FFI; these entry points replace the numpy bodies of its L1 operator API
 * (SURVEY.md §8(b)):
 *
 *   tnc_permute         <- tncsim.tensor.permute          (pkg/src/tncsim/tensor.py:252-274)
 *   tnc_plan_contract   <- tncsim.contract.ttgt_plan       (pkg/src/tncsim/contract.py:98-117)
 *   tnc_contract        <- tncsim.contract.contract_pair   (pkg/src/tncsim/contract.py:149-165)
 *   tnc_contract_split  <- tncsim.contract.split_common_contract (pkg/src/tncsim/contract.py:168-208)
 *   tnc_absorb_chain    <- chain of contract_pair(T, gate) on a stem
 *                          (pkg/src/tncsim/execute.py:150-173 over tree.py:278-384 stems)
 *   tnc_axpy            <- slice-partial folds / MERGE sums
 *                          (pkg/src/tncsim/execute.py:97-112, 227, 288-305)
 *   tnc_project_view    <- tncsim.tensor.project           (pkg/src/tncsim/tensor.py:277-292),
 *                          realised as a zero-copy strided view.
 *
 * Conventions
 *  - Tensors are dense, complex, interleaved (re, im), element = 8 B
 *    (complex64, TNC_C64) or 16 B (complex128, TNC_C128).  A tensor is
 *    described by (rank, dims[], strides[]) in ELEMENTS, row-major when
 *    contiguous (last leg fastest), exactly the reference layout
 *    (tensor.py:3-9).  Arbitrary strides allow zero-copy projected views.
 *  - The caller owns every device buffer (inputs, outputs, workspace); the
 *    per-call entry points (tnc_contract, tnc_contract_split, tnc_permute,
 *    tnc_absorb_chain, tnc_axpy) never allocate and never synchronise: all
 *    launches are asynchronous on the caller's stream (a cudaStream_t passed
 *    as void*), so they can be captured in a CUDA graph.  tnc_plan_contract
 *    may allocate the plan's device index tables (uploaded and synchronised
 *    once, at plan creation); tnc_plan_destroy frees them.
 *  - Plans are immutable and may be shared across threads.
 *  - Return values are tnc_status codes; tnc_last_error() returns a
 *    thread-local message for the last failure on the calling thread.
 *    Status codes map one-to-one onto tncsim.errors classes in the Python
 *    wrapper (paper_2504_09186_b200/errors.py).
 */
#ifndef TNC_B200_H
#define TNC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TNC_MAX_RANK 64
#define TNC_ABI_VERSION 1

typedef enum tnc_status {
  TNC_OK = 0,
  TNC_ERR_INVALID = 1,       /* TncError: bad argument                         */
  TNC_ERR_TENSOR = 2,        /* TensorError: bad dims / strides / rank         */
  TNC_ERR_PERMUTATION = 3,   /* InvalidPermutationError                        */
  TNC_ERR_CONTRACTION = 4,   /* ContractionError: shared label dim mismatch... */
  TNC_ERR_WORKSPACE = 5,     /* MemoryBudgetError: workspace too small         */
  TNC_ERR_CUDA = 6,          /* DeviceError: CUDA runtime failure              */
  TNC_ERR_NCCL = 7,          /* DeviceError: NCCL failure                      */
  TNC_ERR_UNSUPPORTED = 8    /* TncError: variant not available for the input  */
} tnc_status;

typedef enum tnc_dtype { TNC_C64 = 0, TNC_C128 = 1 } tnc_dtype;

/* Kernel variants a contraction plan can select. */
typedef enum tnc_variant {
  TNC_VARIANT_AUTO = 0,
  TNC_VARIANT_SIMT = 1,        /* CUDA-core complex GEMM (fp32 / fp64 accumulate) */
  TNC_VARIANT_TC3XTF32 = 2,    /* tcgen05 kind::tf32, 3xTF32 split, TMEM accum    */
  TNC_VARIANT_SPLITK = 3,      /* CUDA-core split-K, fixed-order tree (tiny M*N)  */
  TNC_VARIANT_TC3XF16 = 4,     /* tcgen05 kind::f16, 2-piece FP16 split with
                                  per-row power-of-two scaling, TMEM accum        */
  TNC_VARIANT_STREAM = 5,      /* narrow step: X streamed once in place, small Y
                                  on chip, C written in the final order (c64,
                                  extent-2 legs, rows_y * K <= 4096)              */
  TNC_VARIANT_TCGATHER = 6     /* gather-fed tcgen05 GEMM: both operands gathered
                                  from their own layouts by the kernel, split to
                                  3xTF32 in shared memory, split-K over CTAs; C
                                  in the final order (c64, extent-2 legs,
                                  rows_y <= 128, K >= 16, rows_x >= 64)           */
} tnc_variant;

/* A labeled operand: leg i has label id labels[i], extent dims[i], element
 * stride strides[i].  Label ids are arbitrary integers, unique per tensor. */
typedef struct tnc_tensor_desc {
  int32_t rank;
  int32_t dtype; /* tnc_dtype */
  int32_t labels[TNC_MAX_RANK];
  int64_t dims[TNC_MAX_RANK];
  int64_t strides[TNC_MAX_RANK];
} tnc_tensor_desc;

typedef struct tnc_plan tnc_plan;

typedef struct tnc_plan_info {
  int64_t m, k, n;             /* TTGT shape: free_A, common, free_B extents      */
  int32_t n_common;
  int32_t variant;             /* tnc_variant actually selected                  */
  int32_t b_is_multiplier;     /* reference ttgt_plan multiplier choice           */
  int32_t out_rank;
  int32_t out_labels[TNC_MAX_RANK];
  int64_t out_dims[TNC_MAX_RANK];
  size_t workspace_bytes;      /* device scratch tnc_contract needs               */
  int64_t multiplies_lo;       /* M*K*N (low 63 bits; exact below 2^63)           */
} tnc_plan_info;

/* ---- library / device ---------------------------------------------------- */
int tnc_abi_version(void);
int tnc_init(int device);
/* Release process-wide library state (profiling events).  Plans own their
 * device tables and free them in tnc_plan_destroy.  Idempotent. */
void tnc_shutdown(void);
const char* tnc_last_error(void);
int tnc_device_info(int* sm_count, int* cc_major, int* cc_minor, size_t* smem_optin);

/* ---- K1: permutation (tensor.py:252-274) ----------------------------------
 * out (contiguous, target order) <- in (any strides).  perm[t] is the source
 * leg placed at target position t.  Bit-exact copy. */
int tnc_permute(int32_t dtype, int32_t rank, const int64_t* dims, const int64_t* in_strides,
                const int32_t* perm, const void* in, void* out, void* stream);

/* ---- K2/K3: pairwise contraction (contract.py:98-208) ---------------------
 * Plan C = sum over shared labels of A*B.  out_labels (out_rank legs) must be
 * a permutation of free_A ++ free_B; pass out_rank = -1 for the reference
 * order free_A ++ free_B.  `variant` forces a kernel (TNC_VARIANT_AUTO picks).
 * The descriptors' strides are baked into the plan (pointers are not). */
int tnc_plan_contract(const tnc_tensor_desc* a, const tnc_tensor_desc* b, int32_t out_rank,
                      const int32_t* out_labels, int32_t variant, tnc_plan** plan);
int tnc_plan_get_info(const tnc_plan* plan, tnc_plan_info* info);
void tnc_plan_destroy(tnc_plan* plan);
/* c is written densely in the plan's output order. */
int tnc_contract(const tnc_plan* plan, const void* a, const void* b, void* c, void* workspace,
                 size_t workspace_bytes, void* stream);
/* split_common_contract: K cut into min(blocks*group, K) panels (base K/panels,
 * remainder on the last), each accumulated independently, then combined by a
 * left-complete pairwise tree (contract.py:193-207). */
int tnc_contract_split_workspace(const tnc_plan* plan, int32_t blocks, int32_t group,
                                 size_t* workspace_bytes);
int tnc_contract_split(const tnc_plan* plan, int32_t blocks, int32_t group, const void* a,
                       const void* b, void* c, void* workspace, size_t workspace_bytes,
                       void* stream);

/* ---- K4: step fusion (absorb a chain of small gates into a big tensor) -----
 * T (rank t_rank in [13, 62], contiguous complex64, dims all 2) absorbs n_gates
 * two-leg gates sequentially.  gates[g] is a DEVICE pointer to the gate's 16
 * complex64 values; gate_strides[4g .. 4g+3] are the element strides of its
 * (out_a, out_b, in_a, in_b) legs, so any leg order / strided view of a
 * rank-4 gate tensor works without a copy.  The gate acts on T legs
 * (axes[2g] = in_a, axes[2g+1] = in_b) -- positions in the CURRENT leg order.
 * Reference semantics of contract_pair(T, G) (contract.py:149-165): the two
 * contracted legs are removed and the gate's out legs are appended at the end.
 * The output is written in the final leg order after all gates; t_out must
 * not alias t_in.  Workspace (tnc_absorb_chain_workspace): the oriented gate
 * table (256 B per gate), plus one tensor-sized buffer when the chain needs
 * more than one HBM pass.  The gate values stay on the device (no host round
 * trip, no sync): each pass's table is copied device-to-device, on the
 * caller's stream, into the library's per-device constant bank; chains
 * launched on different streams are ordered by an event on that bank. */
int tnc_absorb_chain(int32_t t_rank, const void* t_in, void* t_out, int32_t n_gates,
                     const void* const* gates, const int64_t* gate_strides, const int32_t* axes,
                     void* workspace, size_t workspace_bytes, void* stream);
int tnc_absorb_chain_workspace(int32_t t_rank, int32_t n_gates, const int32_t* axes,
                               size_t* workspace_bytes);
/* HBM passes and (<= 5-axis) gate groups the planner uses for this chain. */
int tnc_absorb_chain_info(int32_t t_rank, int32_t n_gates, const int32_t* axes, int32_t* passes,
                          int32_t* groups);

/* ---- K6: accumulation ----------------------------------------------------- */
/* y[i] += x[i] for n complex elements. */
int tnc_axpy(int32_t dtype, int64_t n, const void* x, void* y, void* stream);

/* ---- measurement hooks (bench.py) ------------------------------------------
 * tnc_launch_count: kernels this library has launched since load.
 * tnc_profile_enable(1) clears and starts per-kernel CUDA-event timing on the
 * launching stream; tnc_profile_read sums launches / device ms / algorithmic
 * flops / algorithmic bytes for one kernel kind:
 *   0 tensor-core GEMM, 1 CUDA-core GEMM, 2 permute, 3 3xTF32 operand prep,
 *   4 split-K reduce, 5 absorb chain, 6 axpy, 7 streaming contraction. */
int64_t tnc_launch_count(void);
int tnc_profile_enable(int on);
int tnc_profile_read(int32_t kind, int64_t* launches, double* total_ms, double* flops,
                     double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* TNC_B200_H */
