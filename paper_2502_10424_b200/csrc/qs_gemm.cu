// Small-M linear layers for decode (sm_100a): y[col][n] = sum_k x[col][k] * W[k][n]
// for the few activation rows of a draft (1 row) or verify (gamma+1 rows) forward.
//
// Replaces the fp32 `h @ W` products of decode_step
//   /root/reference/pkg/src/quantspec/model.py:379-397, :405
// and, in INT4 mode, the dequantised f32 weight copies of the draft path
//   /root/reference/pkg/src/quantspec/model.py:141-168 (quantize_model_weights)
// with a weight-streaming tensor-core kernel: W^T tiles are pre-permuted into
// mma.sync A-fragment order (frag16: one 16-byte load per lane per 16x16 tile;
// frag4: one u32 of packed codes per tile, dequantised in registers with the
// per-(row, group) scale applied to the fp32 partial of each group), and the
// activation rows ride as the N=8 columns (swap-AB).  Split-K across CTAs is
// reduced in a fixed order by the last CTA of each 64-row tile, so every
// column's result is independent of how many columns share the launch.
// Fused epilogues: residual add, SiLU*up (Q/model.py:397), and q/k RoPE
// (Q/tensor.py:65-82) + k/v append into the fp16 recent-token buffer
// (Q/cache.py:216-234).
#include <math.h>

#include "qs_common.cuh"
#include "qs_layout.h"
#include "qs_api_internal.h"

namespace qs {

constexpr int kGemmThreads = 128;

template <int NTC>
struct LinCfg {
  static constexpr int COLS = 8 * NTC;
};

__device__ __forceinline__ float silu_f32(float x) { return __fdiv_rn(x, __fadd_rn(1.0f, expf(-x))); }

template <int WMODE, int NTC, int EPI, int GKS>
__global__ void __launch_bounds__(kGemmThreads) linear_kernel(const __grid_constant__ LinearParams P) {
  constexpr int COLS = 8 * NTC;
  extern __shared__ __align__(16) uint8_t sm[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int mg = blockIdx.x, ksp = blockIdx.y;
  const int KS = P.K / 16;
  const int ks0 = ksp * P.krange;
  const int ks1 = min(KS, ks0 + P.krange);
  const int nks = ks1 - ks0;
  const int MT = P.N / 16;
  const int ncols = P.ncols;
  // INT4: k-steps per weight group is the compile-time GKS (the host checks P.wgroup == 16*GKS)
  const int ngr = (WMODE == QS_W_INT4) ? (nks + GKS - 1) / GKS : 0;
  const int ngr_max = (WMODE == QS_W_INT4) ? (P.krange + GKS - 1) / GKS : 0;

  uint2* bs = reinterpret_cast<uint2*>(sm);                                   // [krange][NTC][32]
  float4* psm = reinterpret_cast<float4*>(bs + (size_t)P.krange * NTC * 32);   // [4 mtiles][ngr_max][8]
  float* xsum = reinterpret_cast<float*>(psm + (WMODE == QS_W_INT4 ? (size_t)4 * ngr_max * 8 : 0));  // [ngr][COLS]
  float* ys = xsum + (WMODE == QS_W_INT4 ? (size_t)ngr_max * COLS : 0);       // [64][COLS]
  int* ticket = reinterpret_cast<int*>(ys + 64 * COLS);

  const int mt = mg * 4 + warp;
  // ---- issue this warp's first weight loads before staging (overlaps the prologue) ----
  constexpr int U = 8;  // uint4 per lane per buffer: 8 k-steps (f16) or 32 k-steps (INT4)
  const uint4* wp;
  int nq4;  // uint4 steps of this warp
  if constexpr (WMODE == QS_W_F16) {
    wp = reinterpret_cast<const uint4*>(P.w) + ((size_t)mt * KS + ks0) * 32 + lane;
    nq4 = nks;
  } else {
    const int ks_pad = (KS + 3) / 4 * 4;  // frag4 words [mt][KSpad/4][32][4]; ks0 % 4 == 0
    wp = reinterpret_cast<const uint4*>(P.w) + ((size_t)mt * (ks_pad / 4) + ks0 / 4) * 32 + lane;
    nq4 = (nks + 3) / 4;
  }
  const bool active = mt < MT;
  uint4 buf0[U], buf1[U];
  auto ld = [&](uint4 (&b)[U], int base) {
#pragma unroll
    for (int u = 0; u < U; ++u)
      b[u] = (active && base + u < nq4) ? ldg_nc_v4(wp + (size_t)(base + u) * 32) : make_uint4(0, 0, 0, 0);
  };
  ld(buf0, 0);
  if (nq4 > U) ld(buf1, U);

  // ---- stage the activation slice as f16 B fragments ----
  for (int i = tid; i < nks * NTC * 32; i += kGemmThreads) {
    int ln = i & 31, nt = (i >> 5) % NTC, kk = i / (NTC * 32);
    int gg = ln >> 2, tt = ln & 3;
    int col = nt * 8 + gg;
    uint2 v = make_uint2(0u, 0u);
    if (col < ncols) {
      const float* xr = P.x + (size_t)col * P.K + (size_t)(ks0 + kk) * 16 + 2 * tt;
      v.x = h2_as_u32(__floats2half2_rn(xr[0], xr[1]));
      v.y = h2_as_u32(__floats2half2_rn(xr[8], xr[9]));
    }
    bs[i] = v;
  }
  if constexpr (WMODE == QS_W_INT4) {
    // per-group column sums of the f16-rounded activations (zero-point term)
    for (int i = tid; i < ngr * COLS; i += kGemmThreads) {
      int col = i % COLS, gr = i / COLS;
      float a = 0.f;
      if (col < ncols) {
        int k0 = (ks0 + gr * GKS) * 16, k1 = min(ks1, ks0 + (gr + 1) * GKS) * 16;
        const float* xr = P.x + (size_t)col * P.K;
        for (int k = k0; k < k1; ++k) a += __half2float(__float2half_rn(xr[k]));
      }
      xsum[i] = a;
    }
    // (S, Z) of rows g and g+8 of the CTA's 4 m-tiles for the groups of this k-range
    const int gpr = (P.K + P.wgroup - 1) / P.wgroup;
    const int gr0 = ks0 / GKS;
    const float4* pp = reinterpret_cast<const float4*>(P.wparams);
    for (int i = tid; i < 4 * ngr * 8; i += kGemmThreads) {
      int gg = i & 7, gr = (i >> 3) % ngr, w = i / (8 * ngr);
      int m = mg * 4 + w;
      psm[(w * ngr_max + gr) * 8 + gg] = m < MT ? __ldg(pp + ((size_t)m * gpr + gr0 + gr) * 8 + gg) : make_float4(0, 0, 0, 0);
    }
  }
  __syncthreads();

  float acc[NTC][4];
#pragma unroll
  for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
    for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;

  if (active) {
    if constexpr (WMODE == QS_W_F16) {
      auto mm = [&](uint4 (&b)[U], int base) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          if (base + u < nks) {
            uint32_t a[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
            for (int nt = 0; nt < NTC; ++nt) {
              uint2 bb = bs[((size_t)(base + u) * NTC + nt) * 32 + lane];
              mma16816(acc[nt], a, bb.x, bb.y);
            }
          }
        }
      };
      for (int base = 0; base < nks; base += 2 * U) {
        mm(buf0, base);
        if (base + 2 * U < nks) ld(buf0, base + 2 * U);
        if (base + U < nks) {
          mm(buf1, base + U);
          if (base + 3 * U < nks) ld(buf1, base + 3 * U);
        }
      }
    } else {
      const float4* pw4 = psm + (size_t)warp * ngr_max * 8 + g;
      float tmp[NTC][4];
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) tmp[nt][e] = 0.f;
      auto flush_group = [&](int gl) {
        const float4 sp = pw4[gl * 8];
#pragma unroll
        for (int nt = 0; nt < NTC; ++nt) {
          const int c0 = nt * 8 + 2 * t4;
          const float x0 = xsum[gl * COLS + c0], x1 = xsum[gl * COLS + c0 + 1];
          acc[nt][0] += sp.x * tmp[nt][0] + sp.y * x0;
          acc[nt][1] += sp.x * tmp[nt][1] + sp.y * x1;
          acc[nt][2] += sp.z * tmp[nt][2] + sp.w * x0;
          acc[nt][3] += sp.z * tmp[nt][3] + sp.w * x1;
          tmp[nt][0] = tmp[nt][1] = tmp[nt][2] = tmp[nt][3] = 0.f;
        }
      };
      // base counts uint4 steps (4 k-steps each); 4*U k-steps per buffer is a multiple of GKS
      auto mm = [&](uint4 (&b)[U], int base) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const uint32_t wv[4] = {b[u].x, b[u].y, b[u].z, b[u].w};
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            const int kk = (base + u) * 4 + v;  // local k-step
            if (kk < nks) {
              uint32_t a[4];
              unpack_u4(wv[v], a);
#pragma unroll
              for (int nt = 0; nt < NTC; ++nt) {
                uint2 bb = bs[((size_t)kk * NTC + nt) * 32 + lane];
                mma16816(tmp[nt], a, bb.x, bb.y);
              }
              if (((u * 4 + v + 1) % GKS) == 0 || kk + 1 == nks) flush_group(kk / GKS);
            }
          }
        }
      };
      for (int base = 0; base < nq4; base += 2 * U) {
        mm(buf0, base);
        if (base + 2 * U < nq4) ld(buf0, base + 2 * U);
        if (base + U < nq4) {
          mm(buf1, base + U);
          if (base + 3 * U < nq4) ld(buf1, base + 3 * U);
        }
      }
    }
  }

  // ---- collect the 64 x COLS tile (split-K reduced in fixed order) ----
  const int row0 = mg * 64;
  if (P.ksplit > 1) {
    float* wk = P.work + (size_t)ksp * ncols * P.N;  // [ksplit][ncols][N]
    if (mt < MT) {
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt) {
        int c0 = nt * 8 + 2 * t4;
        int r = mt * 16 + g;
        if (c0 < ncols) {
          wk[(size_t)c0 * P.N + r] = acc[nt][0];
          wk[(size_t)c0 * P.N + r + 8] = acc[nt][2];
        }
        if (c0 + 1 < ncols) {
          wk[(size_t)(c0 + 1) * P.N + r] = acc[nt][1];
          wk[(size_t)(c0 + 1) * P.N + r + 8] = acc[nt][3];
        }
      }
    }
    __threadfence();
    __syncthreads();
    if (tid == 0) *ticket = atomicAdd(&P.counters[mg], 1);
    __syncthreads();
    if (*ticket != P.ksplit - 1) return;
    __threadfence();
    for (int i = tid; i < 64 * ncols; i += kGemmThreads) {
      int r = i % 64, c = i / 64;
      float a = 0.f;
      if (row0 + r < P.N)
        for (int s = 0; s < P.ksplit; ++s) a += __ldcg(P.work + ((size_t)s * ncols + c) * P.N + row0 + r);
      ys[r * COLS + c] = a;
    }
    if (tid == 0) P.counters[mg] = 0;
  } else {
    if (mt < MT) {
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt) {
        int c0 = nt * 8 + 2 * t4;
        int r = warp * 16 + g;
        ys[r * COLS + c0] = acc[nt][0];
        ys[r * COLS + c0 + 1] = acc[nt][1];
        ys[(r + 8) * COLS + c0] = acc[nt][2];
        ys[(r + 8) * COLS + c0 + 1] = acc[nt][3];
      }
    }
  }
  __syncthreads();

  // ---- fused epilogue ----
  if constexpr (EPI == QS_EPI_STORE || EPI == QS_EPI_ADD) {
    for (int i = tid; i < 64 * ncols; i += kGemmThreads) {
      int r = i % 64, c = i / 64;
      int n = row0 + r;
      if (n >= P.N) continue;
      float v = ys[r * COLS + c];
      float* dst = P.y + (size_t)c * P.ldy + n;
      if (EPI == QS_EPI_ADD) *dst = __fadd_rn(*dst, v);
      else *dst = v;
    }
  } else if constexpr (EPI == QS_EPI_SILU_MUL) {
    // m-tiles interleaved: local tiles (0,1) = (gate, up) of output tile 2*mg, (2,3) of 2*mg+1
    for (int i = tid; i < 32 * ncols; i += kGemmThreads) {
      int rr = i % 32, c = i / 32;
      int pair = rr / 16, r16 = rr % 16;
      int rg = pair * 32 + r16, ru = rg + 16;
      int n = (mg * 2 + pair) * 16 + r16;
      if ((row0 + rg) >= P.N) continue;
      float gv = ys[rg * COLS + c], uv = ys[ru * COLS + c];
      P.y[(size_t)c * P.ldy + n] = __fmul_rn(silu_f32(gv), uv);
    }
  } else if constexpr (EPI == QS_EPI_QKV) {
    const float2* rope = reinterpret_cast<const float2*>(P.rope);
    const int hd = P.hd;
    for (int i = tid; i < 32 * ncols; i += kGemmThreads) {
      int pr = i % 32, c = i / 32;
      int r = 2 * pr;
      int n = row0 + r;
      if (n >= P.N) continue;
      int seq = c / P.T, t = c % P.T;
      float e = ys[r * COLS + c], o = ys[(r + 1) * COLS + c];
      if (n < P.Nq + P.Nk) {
        int nn = n < P.Nq ? n : n - P.Nq;
        int d = nn % hd;
        int pos = P.pos_base[seq] + P.row_offset + t;
        float2 cs = rope[(size_t)pos * (hd / 2) + d / 2];
        float e2 = __fsub_rn(__fmul_rn(e, cs.x), __fmul_rn(o, cs.y));
        float o2 = __fadd_rn(__fmul_rn(e, cs.y), __fmul_rn(o, cs.x));
        e = e2;
        o = o2;
      }
      if (n < P.Nq) {
        P.q_out[(size_t)c * P.Nq + n] = e;
        P.q_out[(size_t)c * P.Nq + n + 1] = o;
      } else {
        bool isk = n < P.Nq + P.Nk;
        int nn = isk ? n - P.Nq : n - P.Nq - P.Nk;
        int head = nn / hd, d = nn % hd;
        int row = P.row_base[seq] + P.row_offset + t;
        __half* dst = reinterpret_cast<__half*>(isk ? P.k_dst : P.v_dst) + (size_t)seq * P.kv_seq_stride +
                      (size_t)head * P.kv_head_stride + (size_t)row * hd + d;
        *reinterpret_cast<__half2*>(dst) = __floats2half2_rn(e, o);
      }
    }
  }
}

template <int WMODE, int NTC, int EPI, int GKS>
static cudaError_t launch_lin_t(const LinearParams& p, cudaStream_t s) {
  constexpr int COLS = 8 * NTC;
  size_t ngr = (WMODE == QS_W_INT4) ? (size_t)((p.krange + GKS - 1) / GKS) : 0;
  size_t smem = (size_t)p.krange * NTC * 32 * 8 + ngr * 4 * 8 * 16 + ngr * COLS * 4 + 64 * COLS * 4 + 16;
  auto kern = linear_kernel<WMODE, NTC, EPI, GKS>;
  static size_t configured = 48 * 1024;
  if (smem > configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dim3 grid((p.N + 63) / 64, p.ksplit);
  kern<<<grid, kGemmThreads, smem, s>>>(p);
  return cudaGetLastError();
}

template <int WMODE, int NTC, int GKS>
static cudaError_t launch_lin_e(const LinearParams& p, cudaStream_t s) {
  switch (p.epi) {
    case QS_EPI_STORE: return launch_lin_t<WMODE, NTC, QS_EPI_STORE, GKS>(p, s);
    case QS_EPI_ADD: return launch_lin_t<WMODE, NTC, QS_EPI_ADD, GKS>(p, s);
    case QS_EPI_QKV: return launch_lin_t<WMODE, NTC, QS_EPI_QKV, GKS>(p, s);
    case QS_EPI_SILU_MUL: return launch_lin_t<WMODE, NTC, QS_EPI_SILU_MUL, GKS>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int WMODE, int GKS>
static cudaError_t launch_lin_n(const LinearParams& p, cudaStream_t s) {
  int ntc = (p.ncols + 7) / 8;
  if (ntc <= 1) return launch_lin_e<WMODE, 1, GKS>(p, s);
  if (ntc <= 2) return launch_lin_e<WMODE, 2, GKS>(p, s);
  if (ntc <= 4) return launch_lin_e<WMODE, 4, GKS>(p, s);
  if (ntc <= 8) return launch_lin_e<WMODE, 8, GKS>(p, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_linear(const LinearParams& p, cudaStream_t s) {
  if (p.wmode == QS_W_F16) return launch_lin_n<QS_W_F16, 1>(p, s);
  if (p.wmode == QS_W_INT4) {
    switch (p.wgroup) {
      case 16: return launch_lin_n<QS_W_INT4, 1>(p, s);
      case 32: return launch_lin_n<QS_W_INT4, 2>(p, s);
      case 64: return launch_lin_n<QS_W_INT4, 4>(p, s);
      case 128: return launch_lin_n<QS_W_INT4, 8>(p, s);
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaErrorInvalidValue;
}

}  // namespace qs
