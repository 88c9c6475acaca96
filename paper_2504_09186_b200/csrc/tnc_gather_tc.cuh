// K6 gather-fed tensor-core contraction (tnc_gather_tc.cu): host interface.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

namespace tnc {

// One leg of extent 2.  kind: 0 = X-free, 1 = common, 2 = Y-free.  Strides in
// complex elements: x/y = operand strides, out = final output stride,
// canon = stride in the canonical [rows_x][rows_y] partial layout (row index
// = X-free legs in plan order, first most significant; column = Y-free legs).
struct GatherTcLeg {
  int kind;
  int64_t x_stride, y_stride, out_stride, canon_stride;
};

struct GatherTcPlan;
int gather_tc_prepare(int n_legs, const GatherTcLeg* legs, GatherTcPlan** out);
int gather_tc_splits(const GatherTcPlan* plan);
void gather_tc_destroy(GatherTcPlan* plan);
// splits == 1: writes c_final in the final order; splits > 1: writes fp32
// partials [splits][rows_x][rows_y] (canonical) for tree_reduce_launch
int gather_tc_launch(const GatherTcPlan* plan, const void* x, const void* y, void* c_final, void* parts,
                     cudaStream_t stream);

}  // namespace tnc
