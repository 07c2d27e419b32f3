// ts_f16.cuh - the split-fp16 operand encoding of the tensor-core leg,
// shared by the featurizer (which writes pre-split input rows) and k_lstm_tc
// (which splits h every timestep), so both produce identical operands.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>

namespace ts {

// v ~= hi + lo with hi = fp16(v), lo = fp16(v - hi) (22 significant bits);
// eight floats -> two 16-byte chunks of packed halves
__device__ __forceinline__ void split8(const float* v, uint4& hi, uint4& lo) {
  uint32_t h[4], l[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const __half2 hh = __floats2half2_rn(v[2 * i], v[2 * i + 1]);
    const float2 back = __half22float2(hh);
    const __half2 ll = __floats2half2_rn(v[2 * i] - back.x, v[2 * i + 1] - back.y);
    h[i] = *reinterpret_cast<const uint32_t*>(&hh);
    l[i] = *reinterpret_cast<const uint32_t*>(&ll);
  }
  hi = make_uint4(h[0], h[1], h[2], h[3]);
  lo = make_uint4(l[0], l[1], l[2], l[3]);
}

}  // namespace ts
