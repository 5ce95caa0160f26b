// Small fused decode ops (sm_100a): RMSNorm, embedding gather, greedy argmax
// and the device-side greedy accept/rollback bookkeeping.
//   rmsnorm          /root/reference/pkg/src/quantspec/tensor.py:35-42
//   embedding        /root/reference/pkg/src/quantspec/model.py:375
//   argmax selection /root/reference/pkg/src/quantspec/specdec.py:209-212
//   greedy verify    /root/reference/pkg/src/quantspec/specdec.py:276-299
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#include "qs_common.cuh"
#include "qs_api_internal.h"

namespace qs {

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("QS_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}


__global__ void rmsnorm_kernel(const float* __restrict__ x, const float* __restrict__ gain, float* __restrict__ out,
                               int d, float eps) {
  pdl_wait();
  pdl_trigger();
  const float* xr = x + (size_t)blockIdx.x * d;
  float* orow = out + (size_t)blockIdx.x * d;
  __shared__ float red[32];
  float a = 0.f;
  for (int i = threadIdx.x; i < d; i += blockDim.x) a += __fmul_rn(xr[i], xr[i]);
  a = warp_sum(a);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.f;
    v = warp_sum(v);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  float ms = __fdiv_rn(red[0], (float)d);
  float r = __fsqrt_rn(__fadd_rn(ms, eps));
  for (int i = threadIdx.x; i < d; i += blockDim.x) orow[i] = __fmul_rn(__fdiv_rn(xr[i], r), gain[i]);
}

__global__ void embed_kernel(const float* __restrict__ table, const int* __restrict__ tok, int tok_stride, int T,
                             float* __restrict__ out, int d, int vocab, int* flags) {
  pdl_wait();
  pdl_trigger();
  const int c = blockIdx.x;
  int t = tok[(c / T) * tok_stride + c % T];
  if (t < 0 || t >= vocab) {
    if (threadIdx.x == 0 && flags) atomicOr(flags, 2);
    t = 0;
  }
  const float4* src = reinterpret_cast<const float4*>(table + (size_t)t * d);
  float4* dst = reinterpret_cast<float4*>(out + (size_t)c * d);
  for (int i = threadIdx.x; i < d / 4; i += blockDim.x) dst[i] = src[i];
  for (int i = (d / 4) * 4 + threadIdx.x; i < d; i += blockDim.x) out[(size_t)c * d + i] = table[(size_t)t * d + i];
}

// larger value wins; NaN counts as the maximum (np.argmax returns the first NaN);
// ties go to the lower index
__device__ __forceinline__ bool better(float va, int ia, float vb, int ib) {
  bool na = isnan(va), nb = isnan(vb);
  if (na || nb) {
    if (na && nb) return ia < ib;
    return na;
  }
  if (va != vb) return va > vb;
  return ia < ib;
}

__global__ void argmax_kernel(const float* __restrict__ logits, int vocab, int* __restrict__ out, int out_stride) {
  pdl_wait();
  pdl_trigger();
  const float* row = logits + (size_t)blockIdx.x * vocab;
  float bv = -INFINITY;
  int bi = 0x7fffffff;
  // 16-byte loads, four in flight per thread per round (a long scan of dependent scalar loads
  // was L2-latency bound); the (value, first index) order makes the result independent of it
  const bool vec = (vocab & 3) == 0 && (reinterpret_cast<uintptr_t>(row) & 15) == 0;
  const int nv = vec ? vocab / 4 : 0;
  const float4* row4 = reinterpret_cast<const float4*>(row);
  for (int b = threadIdx.x; b < nv; b += 4 * blockDim.x) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = b + u * blockDim.x;
      v[u] = j < nv ? row4[j] : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int j = b + u * blockDim.x;
      if (j < nv) {
        const float e[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
        for (int q = 0; q < 4; ++q)
          if (better(e[q], 4 * j + q, bv, bi)) {
            bv = e[q];
            bi = 4 * j + q;
          }
      }
    }
  }
  for (int i = 4 * nv + threadIdx.x; i < vocab; i += blockDim.x) {
    float v = row[i];
    if (better(v, i, bv, bi)) {
      bv = v;
      bi = i;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    float ov = __shfl_xor_sync(0xffffffffu, bv, o);
    int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (better(ov, oi, bv, bi)) {
      bv = ov;
      bi = oi;
    }
  }
  __shared__ float sv[32];
  __shared__ int si[32];
  if ((threadIdx.x & 31) == 0) {
    sv[threadIdx.x >> 5] = bv;
    si[threadIdx.x >> 5] = bi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w)
      if (better(sv[w], si[w], bv, bi)) {
        bv = sv[w];
        bi = si[w];
      }
    out[(size_t)blockIdx.x * out_stride] = bi;
  }
}

// Greedy rule of Q/specdec.py:279-298 for a ragged batch: sequence b's verify tokens are
// tok[b*stride + 0..T-1] = (pending, d_0, ...), tgt[b*T + i] = argmax of its target row i, and only
// its first gamma_step[b] drafts count (rows past them are the batch's padding).
__global__ void greedy_accept_kernel(int* __restrict__ tok, int stride, const int* __restrict__ tgt, int T,
                                     const int* __restrict__ gs, int B, int* __restrict__ res, int* fp2_len,
                                     int* pos) {
  pdl_wait();
  pdl_trigger();
  for (int b = threadIdx.x; b < B; b += blockDim.x) {
    const int gamma = gs ? min(gs[b], T - 1) : T - 1;
    const int* drafts = tok + (size_t)b * stride + 1;
    const int* t = tgt + (size_t)b * T;
    int v = 0;
    while (v < gamma && drafts[v] == t[v]) ++v;
    const int nxt = t[v];
    res[2 * b] = v;
    res[2 * b + 1] = nxt;
    tok[(size_t)b * stride] = nxt;
    if (fp2_len) fp2_len[b] += v + 1;  // rows kept after rollback(gamma - v)
    if (pos) pos[b] += v + 1;
  }
}

__global__ void add_int_kernel(int* p, int n, int delta) {
  pdl_wait();
  pdl_trigger();
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] += delta;
}

cudaError_t launch_rmsnorm(const float* x, const float* gain, float* out, int n, int d, float eps, cudaStream_t s) {
  return launch_pdl(rmsnorm_kernel, dim3(n), dim3(256), 0, s, x, gain, out, d, eps);
}
cudaError_t launch_embed(const float* table, const int* tok, int tok_stride, int T, float* out, int n, int d,
                         int vocab, int* flags, cudaStream_t s) {
  return launch_pdl(embed_kernel, dim3(n), dim3(256), 0, s, table, tok, tok_stride, T, out, d, vocab, flags);
}
cudaError_t launch_argmax(const float* logits, int n, int vocab, int* out, int out_stride, cudaStream_t s) {
  return launch_pdl(argmax_kernel, dim3(n), dim3(512), 0, s, logits, vocab, out, out_stride);
}
cudaError_t launch_greedy_accept(int* tok, int tok_stride, const int* tgt, int T, const int* gs, int B, int* res,
                                 int* fp2_len, int* pos, cudaStream_t s) {
  return launch_pdl(greedy_accept_kernel, dim3(1), dim3(32), 0, s, tok, tok_stride, tgt, T, gs, B, res, fp2_len, pos);
}
cudaError_t launch_add_int(int* p, int n, int delta, cudaStream_t s) {
  return launch_pdl(add_int_kernel, dim3((n + 127) / 128), dim3(128), 0, s, p, n, delta);
}

}  // namespace qs
