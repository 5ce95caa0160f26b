// Internal glue between the C ABI (include/quantspec_b200.h) and the kernels.
#pragma once
#include <cuda_runtime.h>
#include "../../include/quantspec_b200.h"

namespace qs {
using AttnParams = qs_attn_args;
using LinearParams = qs_linear_args;

cudaError_t launch_attention(const AttnParams& p, int mode, cudaStream_t s);
int attention_smem_bytes(int hd, int nt, int mode);
int attention_occupancy(int hd, int nt, int mode);
cudaError_t launch_linear(const LinearParams& p, cudaStream_t s);
int linear_maxc(int wmode, int N, int K, int nctas);
int linear_occupancy(int wmode, int wgroup, int ncols);
cudaError_t launch_prep_act(const float* x, const float* gain, float eps, void* xh, long long ldxh, float* xs,
                            long long ldxs, int n, int d, cudaStream_t s);

// error reporting shared by all translation units
void set_error(const char* fmt, ...);
}  // namespace qs
