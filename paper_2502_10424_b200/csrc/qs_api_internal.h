// Internal glue between the C ABI (include/quantspec_b200.h) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include "../../include/quantspec_b200.h"

#define QS_MAX_COLS 48  // activation rows of one linear launch (B * T)

namespace qs {
using AttnParams = qs_attn_args;
using LinearParams = qs_linear_args;

cudaError_t launch_attention(const AttnParams& p, int mode, cudaStream_t s);
// query tiles per CTA for `per` query columns: the target view runs 8 queries per MMA tile
// (hi/lo on the M rows), the draft and fp16 views 4 (hi/lo column pairs); queries per CTA = nt * that
inline int attention_nt(int per, int mode) {
  const int w = mode == QS_VIEW_TARGET ? 8 : 4;
  const int nt = (per + w - 1) / w;
  return nt < 1 ? 1 : nt;
}
inline int attention_queries_per_cta(int per, int mode) {
  return attention_nt(per, mode) * (mode == QS_VIEW_TARGET ? 8 : 4);
}
int attention_occupancy(int hd, int per, int mode);
cudaError_t launch_linear(const LinearParams& p, cudaStream_t s);
cudaError_t launch_prep_act(const float* x, const float* gain, float eps, void* xh, long long ldxh, float* xs,
                            long long ldxs, int n, int d, cudaStream_t s);

// error reporting shared by all translation units
void set_error(const char* fmt, ...);
}  // namespace qs
