// ts_lstm_tc.cuh - FAST scoring path (placeholder until the tcgen05 kernel lands).
#pragma once
#include <cuda_runtime.h>
#include "ts_core.cuh"

namespace ts {
inline int tc_pack_weights(cudaStream_t, const double*, const double*, const double*, const double*, int,
                           void**, size_t*) {
  return TS_OK;
}
inline int tc_score_states(cudaStream_t, const PipelineDesc*, int, const ts_decision*, const int64_t*, int64_t,
                           int64_t, const double*, const double*, const double*, const double*, void*, int,
                           double, double, uint64_t, void**, size_t*, uint64_t*, void**, size_t*, void**,
                           size_t*, int*, double*, int64_t*) {
  return TS_ERR_ARG;
}
}  // namespace ts
