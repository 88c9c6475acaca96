// K4: step fusion -- a chain of two-leg gate absorptions into one resident
// tensor (reference: successive contract_pair(T, G) calls along a stem,
// execute.py:150-173 over the stems of tree.py:278-384).  Filled in below.
#include "tnc_common.cuh"

namespace tnc {

int absorb_chain_launch(int t_rank, const void* t_in, void* t_out, int n_gates,
                        const void* const* gates, const int32_t* axes, void* workspace,
                        size_t workspace_bytes, cudaStream_t stream) {
  (void)t_rank; (void)t_in; (void)t_out; (void)n_gates; (void)gates; (void)axes;
  (void)workspace; (void)workspace_bytes; (void)stream;
  TNC_RET(TNC_ERR_UNSUPPORTED, "absorb chain not built yet");
}

}  // namespace tnc
