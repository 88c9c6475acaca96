// K1 permutation entry points beyond the plain copy (tnc_permute.cu).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace tnc {

// Gather + 3xFP16 split in one tiled pass pair: the complex64 tensor `in`
// permuted (perm / dims / in_strides as permute_launch) to a contiguous
// [R, 2^log_k] operand is written straight as the hi / lo fp16 planes that
// f16_split_launch(mode, R, K, Kp = K, ...) would make from the permuted copy
// (identical values and exponents), without materialising the copy.
// `rowmax` is R words of scratch.  Returns TNC_ERR_UNSUPPORTED when the
// permutation does not take the tiled path (caller permutes + splits).
int permute_split_f16_launch(int rank, const int64_t* dims, const int64_t* in_strides, const int32_t* perm,
                             const void* in, int mode, int64_t R, int log_k, void* hi, void* lo, int* exps,
                             unsigned* rowmax, cudaStream_t stream);

}  // namespace tnc
