// Small-M linear layers for decode (sm_100a): y[col][n] = sum_k x[col][k] * W[k][n]
// for the few activation rows of a draft (1 row) or verify (gamma+1 rows) forward.
//
// Replaces the fp32 `h @ W` products of decode_step
//   /root/reference/pkg/src/quantspec/model.py:379-397, :405
// and, in INT4 mode, the dequantised f32 weight copies of the draft path
//   /root/reference/pkg/src/quantspec/model.py:141-168 (quantize_model_weights).
//
// Weight-streaming persistent kernels.  W^T is pre-permuted into mma.sync
// A-fragment order (frag16: 16 B per lane per 16x16 tile; frag4: one u32 of
// packed codes per tile), tile-pair major, so a stage of k-steps of one pair of
// 16-row tiles is one contiguous range.  One CTA per SM owns whole tile pairs
// over the full K range (no tile spans CTAs, so nothing is reduced through
// global memory); a producer warp streams weights, f16 activations and the INT4
// scales / activation group sums into a shared-memory TMA ring that runs across
// pair boundaries; 16 consumer warps (2 tiles x 8 k-parts) run swap-AB
// tensor-core MMAs (activation rows ride as the N=8 columns) and sum their
// k-parts in a fixed order, so each column's result is independent of how many
// columns share the launch.  Fused epilogues: residual add, SiLU*up
// (Q/model.py:397) producing the next layer's f16 input, and q/k RoPE
// (Q/tensor.py:65-82) + k/v append into the fp16 recent-token buffer
// (Q/cache.py:216-234).
#include <math.h>

#include "qs_common.cuh"
#include "qs_layout.h"
#include "qs_api_internal.h"

namespace qs {



// mma.sync without `volatile` (pure: lets ptxas interleave the group's MMAs with unpacking)
__device__ __forceinline__ void mma_acc(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_zc(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  const float z = 0.f;
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%10,%10,%10,%10};\n"
      : "=f"(d[0]), "=f"(d[1]), "=f"(d[2]), "=f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1), "f"(z));
}

// sum of N consecutive floats in shared memory (N in {1,2,4,8}; 4N-byte aligned)
template <int N>
__device__ __forceinline__ float sum_n(const float* p) {
  if constexpr (N == 1) {
    return p[0];
  } else if constexpr (N == 2) {
    const float2 v = *reinterpret_cast<const float2*>(p);
    return __fadd_rn(v.x, v.y);
  } else {
    float a = 0.f;
#pragma unroll
    for (int i = 0; i < N; i += 4) {
      const float4 v = *reinterpret_cast<const float4*>(p + i);
      a = __fadd_rn(a, __fadd_rn(__fadd_rn(v.x, v.y), __fadd_rn(v.z, v.w)));
    }
    return a;
  }
}

__device__ __forceinline__ float silu_f32(float x) { return __fdiv_rn(x, __fadd_rn(1.0f, expf(-x))); }



// Fused epilogue over an nrows x ncols tile of results (ysm[r * COLS + c]) starting at output row
// row0, run by the NTH consumer threads: store / residual add / SiLU*up -> f16 + 16-sums
// (16-row tiles interleaved gate, up) / q,k RoPE + q store + k,v append.
template <int EPI, int COLS, int NTH>
__device__ __forceinline__ void linear_epilogue(const LinearParams& P, float* ysm, int row0, int nrows, int tid,
                                                int ncols) {
  constexpr int nthr = NTH;
  if constexpr (EPI == QS_EPI_STORE || EPI == QS_EPI_ADD) {
    for (int e = tid; e < nrows * ncols; e += nthr) {
      const int r = e % nrows, c = e / nrows;
      const int n = row0 + r;
      if (n >= P.N) continue;
      const float v = ysm[r * COLS + c];
      float* dst = P.y + (size_t)c * P.ldy + n;
      if (EPI == QS_EPI_ADD) *dst = __fadd_rn(*dst, v);
      else *dst = v;
    }
  } else if constexpr (EPI == QS_EPI_SILU_MUL) {
    // 16-row tiles interleaved: local tiles (2p, 2p+1) = (gate, up) of output tile row0/32 + p;
    // output: f16 input of the down projection + its 16-sums (one sum per output tile)
    for (int e = tid; e < (nrows / 2) * ncols; e += nthr) {
      const int rr = e % (nrows / 2), c = e / (nrows / 2);
      const int pair = rr / 16, r16 = rr % 16;
      const int rg = pair * 32 + r16, ru = rg + 16;
      if (row0 + rg >= P.N) continue;
      const int n = (row0 / 32 + pair) * 16 + r16;
      const float h = __fmul_rn(silu_f32(ysm[rg * COLS + c]), ysm[ru * COLS + c]);
      const __half hh = __float2half_rn(h);
      reinterpret_cast<__half*>(P.yh)[(size_t)c * P.ldyh + n] = hh;
      if (P.y) P.y[(size_t)c * P.ldy + n] = h;
      ysm[rg * COLS + c] = __half2float(hh);  // gate slot now holds the f16-rounded output
    }
    asm volatile("bar.sync 2, %0;" ::"n"(NTH));
    for (int e = tid; e < (nrows / 32) * ncols; e += nthr) {
      const int pair = e % (nrows / 32), c = e / (nrows / 32);
      if (row0 + pair * 32 >= P.N) continue;
      float a = 0.f;
      for (int r16 = 0; r16 < 16; ++r16) a += ysm[(pair * 32 + r16) * COLS + c];
      P.ys[(size_t)c * P.ldys + row0 / 32 + pair] = a;
    }
  } else if constexpr (EPI == QS_EPI_QKV) {
    const float2* rope = reinterpret_cast<const float2*>(P.rope);
    const int hd = P.hd;
    for (int e = tid; e < (nrows / 2) * ncols; e += nthr) {
      const int pr = e % (nrows / 2), c = e / (nrows / 2);
      const int r = 2 * pr;
      const int n = row0 + r;
      if (n >= P.N) continue;
      const int sq = c / P.T, t = c % P.T;
      float ev = ysm[r * COLS + c], ov = ysm[(r + 1) * COLS + c];
      if (n < P.Nq + P.Nk) {
        const int nn = n < P.Nq ? n : n - P.Nq;
        const int d = nn % hd;
        int pos = P.pos_base[sq] + P.row_offset + t;
        if (pos >= P.max_pos) {  // beyond the rope table: ConfigError on the host (Q/model.py:334-336)
          if (P.flags) atomicOr(P.flags, 8);
          pos = P.max_pos - 1;
        }
        const float2 cs = rope[(size_t)pos * (hd / 2) + d / 2];
        const float e2 = __fsub_rn(__fmul_rn(ev, cs.x), __fmul_rn(ov, cs.y));
        const float o2 = __fadd_rn(__fmul_rn(ev, cs.y), __fmul_rn(ov, cs.x));
        ev = e2;
        ov = o2;
      }
      if (n < P.Nq) {
        P.q_out[(size_t)c * P.Nq + n] = ev;
        P.q_out[(size_t)c * P.Nq + n + 1] = ov;
      } else {
        const bool isk = n < P.Nq + P.Nk;
        const int nn = isk ? n - P.Nq : n - P.Nq - P.Nk;
        const int head = nn / hd, d = nn % hd;
        const int row = P.row_base[sq] + P.row_offset + t;
        if (row >= P.row_cap) {  // past the buffer: BufferOverflowError on the host
          if (P.flags) atomicOr(P.flags, 4);
          continue;
        }
        __half* dst = reinterpret_cast<__half*>(isk ? P.k_dst : P.v_dst) + (size_t)sq * P.kv_seq_stride +
                      (size_t)head * P.kv_head_stride + (size_t)row * hd + d;
        *reinterpret_cast<__half2*>(dst) = __floats2half2_rn(ev, ov);
      }
    }
  }
}


// One activation row -> f16 copy (RMS-normalised when gain != NULL, Q/tensor.py:35-42) + the sums
// of every 16 f16-rounded values.  Work is done by threads [0, 256) in a fixed mapping (one 16-element
// group per thread per round, fixed reduction tree), so every caller produces identical bits --
// qs_prep_act and the linear kernels' in-kernel prep must agree for a T-row verify to equal T
// single-row steps.  BAR: 0 = __syncthreads, else a named barrier over BAR threads (all of which call).
template <int BAR>
__device__ __forceinline__ void act_prep_row(const float* __restrict__ xr, const float* __restrict__ gain, float eps,
                                             int d, __half* __restrict__ hr, float* __restrict__ sr, float* red,
                                             int tid) {
  constexpr int NW = 256;
  auto sync = [] {
    if constexpr (BAR == 0) __syncthreads();
    else asm volatile("bar.sync 3, %0;" ::"n"(BAR));
  };
  const int ng = d / 16;
  float scale = 1.f;
  if (gain) {
    if (tid < NW) {
      float a = 0.f;
      for (int gi = tid; gi < ng; gi += NW) {
        const float4* p = reinterpret_cast<const float4*>(xr + gi * 16);
        float4 v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = p[j];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          a += __fmul_rn(v[j].x, v[j].x);
          a += __fmul_rn(v[j].y, v[j].y);
          a += __fmul_rn(v[j].z, v[j].z);
          a += __fmul_rn(v[j].w, v[j].w);
        }
      }
      a = warp_sum(a);
      if ((tid & 31) == 0) red[tid >> 5] = a;
    }
    sync();
    if (tid < 32) {
      float v = tid < NW / 32 ? red[tid] : 0.f;
      v = warp_sum(v);
      if (tid == 0) red[32] = __fsqrt_rn(__fadd_rn(__fdiv_rn(v, (float)d), eps));
    }
    sync();
    scale = red[32];
  }
  if (tid < NW) {
    for (int gi = tid; gi < ng; gi += NW) {
      float xv[16], gv[16];
      const float4* p = reinterpret_cast<const float4*>(xr + gi * 16);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float4 v = p[j];
        xv[4 * j] = v.x; xv[4 * j + 1] = v.y; xv[4 * j + 2] = v.z; xv[4 * j + 3] = v.w;
      }
      if (gain) {
        const float4* gp = reinterpret_cast<const float4*>(gain + gi * 16);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float4 v = gp[j];
          gv[4 * j] = v.x; gv[4 * j + 1] = v.y; gv[4 * j + 2] = v.z; gv[4 * j + 3] = v.w;
        }
      }
      float s = 0.f;
      __align__(16) __half hv[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const float v = gain ? __fmul_rn(__fdiv_rn(xv[j], scale), gv[j]) : xv[j];
        hv[j] = __float2half_rn(v);
        s += __half2float(hv[j]);
      }
      *reinterpret_cast<uint4*>(hr + gi * 16) = *reinterpret_cast<uint4*>(hv);
      *reinterpret_cast<uint4*>(hr + gi * 16 + 8) = *reinterpret_cast<uint4*>(hv + 8);
      sr[gi] = s;
    }
  }
  sync();
}

// ---------------------------------------------------------------------------
// INT4 W4A16 GEMV/GEMM without cross-CTA reduction (the draft's weights).
//
// One CTA owns a pair of 16-row tiles (32 output rows; for the gate/up projection exactly
// the (gate, up) rows of one output tile) over the FULL K range, so no tile spans CTAs:
// the stream-K fix-up (partials through L2, a ticket, the last CTA's reduction) was the
// limiter of these short INT4 launches.  Weights are stored pair-major
// ([pair][k-quad][2 tiles][32 lanes][16 B], params [pair][group][2 tiles][8 slots][float4], row g in slot g ^ i4_param_swz(group)), so
// a 64-k-step stage of a pair is one contiguous bulk copy of codes and one of params.
// Persistent: one CTA per SM takes pairs b, b + grid, ...; its TMA ring (up to 8 stages of 64
// k-steps) runs straight across pair boundaries.  Warps 0-7: tile w&1, k-quarter w>>1 of every
// stage; the four k-quarters of a tile are summed through shared memory in fixed order at the
// pair's end.  PDL overlaps the first weight stages with the previous kernel.
// ---------------------------------------------------------------------------
#ifndef QS_I4_BREG
#define QS_I4_BREG 0  // A/B builds: single-row B words held in registers per window (measured -1%: off)
#endif
#ifndef QS_I4_CHAINS
#define QS_I4_CHAINS 2  // A/B builds: MMA accumulator chains per window (power of two)
#endif
#ifndef QS_I4_KP1
#define QS_I4_KP1 8  // k-parts (consumer warps per tile) of the single-row INT4 config (A/B: 4 is 4% faster in
                     // isolation but 1.3% slower over the whole decode cycle, profiles/r02/NOTES.md)
#endif
#ifndef QS_I4_KCH1
#define QS_I4_KCH1 128  // A/B builds: k-steps per stage of the single-row INT4 config
#endif
#ifndef QS_I4_L2PF
#define QS_I4_L2PF 0  // A/B: L2 bulk prefetch this many ring depths ahead of the TMA ring (0: off)
#endif
// KC: k-steps per stage of the single-row config (0: QS_I4_KCH1); with QS_I4_BIGK the dispatch takes 256
// for K <= QS_I4_BIGK (A/B: with 4 k-parts 8% faster in isolation, slower inside the decode cycle)
template <int NTC, int GKS, int CW, int KC = 0>
struct I4Cfg {
  static constexpr bool SINGLE = NTC == 1 && CW == 1;             // one activation row
  static constexpr int KP = SINGLE ? QS_I4_KP1 : 8;               // k-parts: warps per tile
  static constexpr int NCW = 2 * KP;                              // tile w&1, k-part w>>1
  static constexpr int THREADS = (NCW + 1) * 32;
  static constexpr int KCH = SINGLE ? (KC ? KC : QS_I4_KCH1) : 128;  // k-steps per stage
#ifdef QS_I4_MINB1
  static constexpr int MINB = SINGLE ? QS_I4_MINB1 : 1;             // A/B builds: resident CTAs per SM
#else
  static constexpr int MINB = (SINGLE && KCH <= 64) ? 2 : 1;      // resident CTAs per SM
#endif
  static constexpr int SMEM_CAP = MINB == 2 ? 233472 / 2 - 1024 : 232448;
  static constexpr int HKS = KCH / KP;                            // k-steps per consumer warp per stage
  static constexpr int WBYTES = (KCH / 4) * 2 * 512;              // codes of both tiles
  static constexpr int ROWS = NTC == 1 ? CW : 16;
  static constexpr int RPAD = ROWS > 1 ? 16 : 0;                  // bank skew between activation rows
  static constexpr int BROW = KCH * 32 + RPAD;
  static constexpr int PBYTES = (KCH / GKS) * 2 * 128;            // {S,Z} x 16 rows x 2 tiles per group
  static constexpr int XROW = KCH * 4 + RPAD;
  static constexpr int OFF_B = WBYTES;
  static constexpr int OFF_P = OFF_B + ROWS * BROW;
  static constexpr int OFF_X = OFF_P + PBYTES;
  static constexpr int STAGE = (OFF_X + ROWS * XROW + 127) / 128 * 128;
  static constexpr int YCOLS = 8 * NTC;
  // in-kernel activation prep (P.xf): the f16 row + 16-sums of up to ACT_K inputs
  // (one activation row -- the draft's T = 1 -- of up to 4096 inputs: the normed projections)
  static constexpr int ACT_K = 4096;
  static constexpr int ACT_ROW = ACT_K * 2;
  static constexpr int ACT_SROW = ACT_K / 16;
  static constexpr int ACT_BYTES = (NTC == 1 && CW == 1) ? ACT_ROW + ACT_SROW * 4 : 0;
  // k-part partials (the results ysm alias slot 0) + barriers + act row; trimmed so that the
  // single-row config holds four 52.5 KB stages (210 KB of weights in flight per SM)
  static constexpr int FIXED = (KP - 1) * 32 * YCOLS * 4 + 2 * 8 * 8 + 16 + ACT_BYTES;
  static constexpr int NSTAGE = (SMEM_CAP - FIXED) / STAGE < 8 ? (SMEM_CAP - FIXED) / STAGE : 8;
  static constexpr int SMEM = NSTAGE * STAGE + FIXED;
};

// HKS k-steps of one 16-row tile for one consumer warp (window / group-slot scheme of
// int4_unit; pair-major strides).  wa: this lane's first uint4 of the k-range; bbase: B rows
// at the k-range; pp: float4 params of the first group (this tile, slot 0), whose absolute group
// index is gb (the slot of row g is g ^ i4_param_swz(group)); xsm: 16-sums.
template <class C, int NTC, int GKS, int CW, bool NOMMA = false>
__device__ __forceinline__ void i4_steps(const uint4* __restrict__ wa, const uint8_t* bbase, const float4* pp,
                                         const float* xsm, const int nks, const int g, const int t4,
                                         float (&acc)[NTC][4], const int brs, const int XW, const int gb) {
  constexpr int G8 = 8 / CW;
  constexpr int WIN = (G8 * GKS < C::HKS) ? G8 * GKS : C::HKS;  // k-steps per window
  constexpr int NSLOT = WIN / GKS;
  const int my_slot = g / CW;
#pragma unroll
  for (int w = 0; w < C::HKS / WIN; ++w) {
    const int k0 = w * WIN;
    if (k0 >= nks) break;
    constexpr int NCH = QS_I4_CHAINS;  // independent MMA accumulator chains per window
    float D2[NCH][NTC][4];
#pragma unroll
    for (int c2 = 0; c2 < NCH; ++c2)
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) D2[c2][nt][e] = 0.f;
    if constexpr (NTC == 1 && CW == 1 && !NOMMA && QS_I4_BREG) {
      // one activation row: this lane only ever feeds its own slot (g) -> load those GKS k-steps'
      // B words once per window and select them (or zero) per k-step, instead of a predicated
      // pair of shared loads + zeroing per k-step
      uint32_t xb[GKS][2];
      const uint8_t* brow = bbase + 4 * t4;
#pragma unroll
      for (int j = 0; j < GKS; ++j) {
        const int ks = k0 + my_slot * GKS + j;
        const bool ok = my_slot < NSLOT && ks < nks;
        xb[j][0] = ok ? *reinterpret_cast<const uint32_t*>(brow + ks * 32) : 0u;
        xb[j][1] = ok ? *reinterpret_cast<const uint32_t*>(brow + ks * 32 + 16) : 0u;
      }
#pragma unroll
      for (int sl = 0; sl < NSLOT; ++sl) {
        const bool mine = my_slot == sl;
#pragma unroll
        for (int j = 0; j < GKS; ++j) {
          const int ks = k0 + sl * GKS + j;
          if (ks < nks) {
            const uint4 w4 = wa[(ks >> 2) * 64];
            const uint32_t wv = (ks & 3) == 0 ? w4.x : (ks & 3) == 1 ? w4.y : (ks & 3) == 2 ? w4.z : w4.w;
            uint32_t a[4];
            unpack_u4_raw(wv, a);
            mma_acc(D2[(sl * GKS + j) % NCH][0], a, mine ? xb[j][0] : 0u, mine ? xb[j][1] : 0u);
          }
        }
      }
    } else {
#pragma unroll
    for (int sl = 0; sl < NSLOT; ++sl) {
      const bool mine = my_slot == sl;
      const uint8_t* brow[NTC];
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt) brow[nt] = bbase + (nt * 8 + g % CW) * brs + 4 * t4;
#pragma unroll
      for (int j = 0; j < GKS; ++j) {
        const int ks = k0 + sl * GKS + j;
        if (ks < nks) {
          const uint4 w4 = wa[(ks >> 2) * 64];
          const uint32_t wv = (ks & 3) == 0 ? w4.x : (ks & 3) == 1 ? w4.y : (ks & 3) == 2 ? w4.z : w4.w;
          uint32_t a[4];
          unpack_u4_raw(wv, a);
#pragma unroll
          for (int nt = 0; nt < NTC; ++nt) {
            uint32_t b0 = 0u, b1 = 0u;
            if (mine) {
              b0 = *reinterpret_cast<const uint32_t*>(brow[nt] + ks * 32);
              b1 = *reinterpret_cast<const uint32_t*>(brow[nt] + ks * 32 + 16);
            }
            if constexpr (NOMMA)  // diagnostic (dbg bit 2): same operand traffic, no tensor-core op
              D2[(sl * GKS + j) % NCH][nt][0] += __uint_as_float((a[0] ^ a[1] ^ a[2] ^ a[3] ^ b0 ^ b1) & 0x3fffffffu);
            else
              mma_acc(D2[(sl * GKS + j) % NCH][nt], a, b0, b1);
          }
        }
      }
    }
    }
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt) {
      float D[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        // fixed pairwise order over the chains
        float t[NCH];
#pragma unroll
        for (int c2 = 0; c2 < NCH; ++c2) t[c2] = D2[c2][nt][e];
#pragma unroll
        for (int h = NCH / 2; h > 0; h >>= 1)
#pragma unroll
          for (int c2 = 0; c2 < h; ++c2) t[c2] = __fadd_rn(t[c2], t[c2 + h]);
        D[e] = t[0];
      }
      float vg[2], v8[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int n = 2 * t4 + e;
        const int sl = n / CW, c = nt * 8 + n % CW;
        const int gl = k0 / GKS + sl;
        const int kk0 = gl * GKS;
        vg[e] = v8[e] = 0.f;
        if (sl < NSLOT && kk0 < nks) {
          const float4 p = pp[gl * 16 + (g ^ i4_param_swz(gb + gl))];  // {S_g, Z_g - 1024 S_g, S_g8 / 16, Z_g8 - 64 S_g8}
          const float* xc = xsm + c * XW + kk0;
          float X;
          if (kk0 + GKS <= nks) {
            X = sum_n<GKS>(xc);
          } else {
            X = 0.f;
            for (int q = 0; q < nks - kk0; ++q) X = __fadd_rn(X, xc[q]);
          }
          vg[e] = __fmaf_rn(p.x, D[e], __fmul_rn(p.y, X));
          v8[e] = __fmaf_rn(p.z, D[e + 2], __fmul_rn(p.w, X));
        }
      }
      if constexpr (CW == 1) {
        // lane-local partials of this lane's group slots; the quad sum happens once per tile
        // pair (i4_quad_sum) instead of once per window
        acc[nt][0] = __fadd_rn(acc[nt][0], __fadd_rn(vg[0], vg[1]));
        acc[nt][2] = __fadd_rn(acc[nt][2], __fadd_rn(v8[0], v8[1]));
      } else {
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if constexpr (CW == 2) {
            vg[e] = __fadd_rn(vg[e], __shfl_xor_sync(0xffffffffu, vg[e], 1));
            v8[e] = __fadd_rn(v8[e], __shfl_xor_sync(0xffffffffu, v8[e], 1));
          }
          if constexpr (CW <= 4) {
            vg[e] = __fadd_rn(vg[e], __shfl_xor_sync(0xffffffffu, vg[e], 2));
            v8[e] = __fadd_rn(v8[e], __shfl_xor_sync(0xffffffffu, v8[e], 2));
          }
          acc[nt][e] = __fadd_rn(acc[nt][e], vg[e]);
          acc[nt][e + 2] = __fadd_rn(acc[nt][e + 2], v8[e]);
        }
      }
    }
  }
}

#ifndef QS_I4_EARLY
#define QS_I4_EARLY 0  // A/B builds: single-row consumers copy their stage slice to registers and release it first
#endif
// Single activation row (NTC = CW = 1), early release: the warp's codes, its two param slots per
// window, its own slot's B words and the 16-sums are copied into registers first, the stage is
// handed back to the producer (`release`), and the MMA chain then runs from registers -- the ring
// stage is held for one round of shared loads instead of the whole window.  Same operations in the
// same order as i4_steps, so the results are bit-identical.
template <class C, int GKS, class Rel>
__device__ __forceinline__ void i4_steps_early(const uint4* __restrict__ wa, const uint8_t* bbase, const float4* pp,
                                               const float* xsm, const int nks, const int g, const int t4,
                                               float (&acc)[1][4], const int gb, Rel release) {
  constexpr int WIN = (8 * GKS < C::HKS) ? 8 * GKS : C::HKS;  // k-steps per window
  constexpr int NSLOT = WIN / GKS;
  constexpr int NW = C::HKS / WIN;
  constexpr int NQ4 = (C::HKS + 3) / 4;
  uint4 wr[NQ4];
  uint32_t xb[NW][GKS][2];
  float4 pr[NW][2];
  float X[NW][2];
#pragma unroll
  for (int i = 0; i < NQ4; ++i) wr[i] = (4 * i < nks) ? wa[i * 64] : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int k0 = w * WIN;
#pragma unroll
    for (int j = 0; j < GKS; ++j) {
      const int ks = k0 + g * GKS + j;
      const bool ok = g < NSLOT && ks < nks;
      xb[w][j][0] = ok ? *reinterpret_cast<const uint32_t*>(bbase + 4 * t4 + ks * 32) : 0u;
      xb[w][j][1] = ok ? *reinterpret_cast<const uint32_t*>(bbase + 4 * t4 + ks * 32 + 16) : 0u;
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int sl = 2 * t4 + e, gl = k0 / GKS + sl, kk0 = gl * GKS;
      pr[w][e] = make_float4(0.f, 0.f, 0.f, 0.f);
      X[w][e] = 0.f;
      if (sl < NSLOT && kk0 < nks) {
        pr[w][e] = pp[gl * 16 + (g ^ i4_param_swz(gb + gl))];
        const float* xc = xsm + kk0;
        if (kk0 + GKS <= nks) {
          X[w][e] = sum_n<GKS>(xc);
        } else {
          for (int q = 0; q < nks - kk0; ++q) X[w][e] = __fadd_rn(X[w][e], xc[q]);
        }
      }
    }
  }
  release();
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    const int k0 = w * WIN;
    if (k0 >= nks) break;
    constexpr int NCH = QS_I4_CHAINS;
    float D2[NCH][4];
#pragma unroll
    for (int c2 = 0; c2 < NCH; ++c2)
#pragma unroll
      for (int e = 0; e < 4; ++e) D2[c2][e] = 0.f;
#pragma unroll
    for (int sl = 0; sl < NSLOT; ++sl) {
      const bool mine = g == sl;
#pragma unroll
      for (int j = 0; j < GKS; ++j) {
        const int ks = k0 + sl * GKS + j;
        if (ks < nks) {
          const uint4 w4 = wr[ks >> 2];
          const uint32_t wv = (ks & 3) == 0 ? w4.x : (ks & 3) == 1 ? w4.y : (ks & 3) == 2 ? w4.z : w4.w;
          uint32_t a[4];
          unpack_u4_raw(wv, a);
          mma_acc(D2[(sl * GKS + j) % NCH], a, mine ? xb[w][j][0] : 0u, mine ? xb[w][j][1] : 0u);
        }
      }
    }
    float D[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      float t[NCH];
#pragma unroll
      for (int c2 = 0; c2 < NCH; ++c2) t[c2] = D2[c2][e];
#pragma unroll
      for (int h = NCH / 2; h > 0; h >>= 1)
#pragma unroll
        for (int c2 = 0; c2 < h; ++c2) t[c2] = __fadd_rn(t[c2], t[c2 + h]);
      D[e] = t[0];
    }
    float vg[2], v8[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int sl = 2 * t4 + e, kk0 = (k0 / GKS + sl) * GKS;
      vg[e] = v8[e] = 0.f;
      if (sl < NSLOT && kk0 < nks) {
        vg[e] = __fmaf_rn(pr[w][e].x, D[e], __fmul_rn(pr[w][e].y, X[w][e]));
        v8[e] = __fmaf_rn(pr[w][e].z, D[e + 2], __fmul_rn(pr[w][e].w, X[w][e]));
      }
    }
    acc[0][0] = __fadd_rn(acc[0][0], __fadd_rn(vg[0], vg[1]));
    acc[0][2] = __fadd_rn(acc[0][2], __fadd_rn(v8[0], v8[1]));
  }
}

// CW == 1: sum the four lanes' slot partials of rows g, g+8 (every lane of the quad ends with the total)
template <int NTC, int CW>
__device__ __forceinline__ void i4_quad_sum(float (&acc)[NTC][4]) {
  if constexpr (CW == 1) {
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
      for (int e = 0; e < 4; e += 2) {
        acc[nt][e] = __fadd_rn(acc[nt][e], __shfl_xor_sync(0xffffffffu, acc[nt][e], 1));
        acc[nt][e] = __fadd_rn(acc[nt][e], __shfl_xor_sync(0xffffffffu, acc[nt][e], 2));
      }
  }
}

template <int NTC, int EPI, int GKS, int CW, int KC = 0>
__global__ void __launch_bounds__(I4Cfg<NTC, GKS, CW, KC>::THREADS, I4Cfg<NTC, GKS, CW, KC>::MINB) linear_i4_kernel(const __grid_constant__ LinearParams P) {
  using C = I4Cfg<NTC, GKS, CW, KC>;
  constexpr int COLS = 8 * NTC;
  constexpr int KCH = C::KCH;
  extern __shared__ __align__(128) uint8_t sm[];
  float* hsm = reinterpret_cast<float*>(sm + C::NSTAGE * C::STAGE);  // [KP-1][32][COLS] k-part partials
  float* ysm = hsm;  // [32][COLS] results: slot 0, overwritten by the thread that read it
  uint64_t* full_b = reinterpret_cast<uint64_t*>(hsm + (C::KP - 1) * 32 * COLS);
  uint64_t* empty_b = full_b + 8;
  uint8_t* act_h = reinterpret_cast<uint8_t*>(empty_b + 8) + 16;                // [ACT_ROW] f16 row
  float* act_s = reinterpret_cast<float*>(act_h + C::ACT_ROW);                   // [ACT_SROW] 16-sums

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int KS = P.K / 16;
  const int ks_pad = (KS + 3) / 4 * 4;
  constexpr int WG = GKS * 16;  // weight group (the dispatch picks GKS = wgroup / 16)
  const int gpr = (P.K + WG - 1) / WG;
  const int TP = (P.N / 16 + 1) / 2;              // tile pairs
  const bool act_in = C::ACT_BYTES > 0 && P.xf != nullptr;  // activations built here, not streamed
  const int nst = (KS + KCH - 1) / KCH;          // stages per pair (full K range)
  const int npairs = (TP - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;  // pairs b, b+grid, ...
  const int total = npairs * nst;                // stages this CTA streams
  const int ncols = P.ncols;

  if (tid == 0) {
    for (int s = 0; s < C::NSTAGE; ++s) {
      mbar_init(&full_b[s], 1);
      mbar_init(&empty_b[s], C::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::NCW) {
    // ======================= producer warp (lane 0 issues) =======================
    // stage q of this CTA = stage q % nst of pair blockIdx.x + (q / nst) * gridDim.x; the ring
    // runs straight across pair boundaries, so the next pair's weights are already in flight
    auto issue_static = [&](int q) {
      const int s = q % C::NSTAGE;
      const int tp = blockIdx.x + (q / nst) * gridDim.x, u = q % nst;
      const int ks0 = u * KCH, nks = min(KCH, KS - ks0);
      uint8_t* sp = sm + s * C::STAGE;
      const uint32_t wb = (uint32_t)((nks + 3) / 4) * 1024;
      const uint32_t pb = (uint32_t)((nks * 16 + WG - 1) / WG) * 256;
      const uint32_t bb = (uint32_t)nks * 32, xb = (uint32_t)((nks + 3) / 4) * 16;
      mbar_arrive_expect_tx(&full_b[s], wb + pb + (act_in ? 0u : ncols * (bb + xb)));
      bulk_g2s(sp, reinterpret_cast<const uint8_t*>(P.w) + ((size_t)tp * (ks_pad / 4) + ks0 / 4) * 1024, wb, &full_b[s]);
      bulk_g2s(sp + C::OFF_P, reinterpret_cast<const uint8_t*>(P.wparams) + ((size_t)tp * gpr + ks0 * 16 / WG) * 256,
               pb, &full_b[s]);
      if constexpr (QS_I4_L2PF > 0) {
        // stage q + NSTAGE * L2PF to L2 now: the DRAM requests in flight are not capped by the ring
        const int qp = q + C::NSTAGE * QS_I4_L2PF;
        if (qp < total) {
          const int tpp = blockIdx.x + (qp / nst) * gridDim.x, up = qp % nst;
          const int pks0 = up * KCH, pnks = min(KCH, KS - pks0);
          bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(P.w) + ((size_t)tpp * (ks_pad / 4) + pks0 / 4) * 1024,
                           (uint32_t)((pnks + 3) / 4) * 1024);
          bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(P.wparams) + ((size_t)tpp * gpr + pks0 * 16 / WG) * 256,
                           (uint32_t)((pnks * 16 + WG - 1) / WG) * 256);
        }
      }
    };
    auto issue_act = [&](int q) {
      const int s = q % C::NSTAGE, u = q % nst;
      const int ks0 = u * KCH, nks = min(KCH, KS - ks0);
      uint8_t* sp = sm + s * C::STAGE;
      const uint32_t bb = (uint32_t)nks * 32, xb = (uint32_t)((nks + 3) / 4) * 16;
      for (int c = 0; c < ncols; ++c) {
        bulk_g2s(sp + C::OFF_B + c * C::BROW, reinterpret_cast<const __half*>(P.xh) + (size_t)c * P.ldxh + ks0 * 16, bb,
                 &full_b[s]);
        bulk_g2s(sp + C::OFF_X + c * C::XROW, P.xs + (size_t)c * P.ldxs + ks0, xb, &full_b[s]);
      }
    };
    const int npre = min(total, C::NSTAGE);
    if (lane == 0)
      for (int q = 0; q < npre; ++q) issue_static(q);  // weights stream in before the dependency resolves
    pdl_wait();
    pdl_trigger();
    if (lane == 0) {
      for (int q = 0; q < total; ++q) {
        if (q >= npre) {
          mbar_wait(&empty_b[q % C::NSTAGE], ((q / C::NSTAGE) - 1) & 1);
          issue_static(q);
        }
        if (!act_in) issue_act(q);
      }
    }
    __syncwarp();
    return;
  }
  pdl_wait();
  pdl_trigger();
  if (act_in) {
    // f16 activation (+ RMS norm) and its 16-sums for the whole K range, once per CTA, while the
    // first weight stages are still in flight (the same bits qs_prep_act would write)
    act_prep_row<C::NCW * 32>(P.xf, P.gain, P.eps, P.K, reinterpret_cast<__half*>(act_h), act_s, ysm, tid);
  }

  // ======================= consumer warps =======================
  const int tile = warp & 1, kp = warp >> 1;
  const int rr = tile * 16 + g;
  int s = 0, ph = 0;
  for (int pi = 0; pi < npairs; ++pi) {
    const int tp = blockIdx.x + pi * gridDim.x;
    float acc[NTC][4];
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = 0.f;
    for (int u = 0; u < nst; ++u) {
      mbar_wait(&full_b[s], ph);
      const int nks = min(KCH, KS - u * KCH) - kp * C::HKS;  // this warp's k-steps of the stage
      if (nks > 0 && !(P.dbg & 1)) {
        const uint8_t* sp = sm + s * C::STAGE;
        const int ko = kp * C::HKS;
        const uint4* wa = reinterpret_cast<const uint4*>(sp) + (ko / 4) * 64 + tile * 32 + lane;
        const float4* pp = reinterpret_cast<const float4*>(sp + C::OFF_P) + (ko * 16 / WG) * 16 + tile * 8;
        const int gb = (u * KCH + ko) * 16 / WG;  // absolute group index of pp
        const int kabs = u * KCH + ko;  // absolute k-step (activations built in-kernel)
        const float* xsm = act_in ? act_s + kabs : reinterpret_cast<const float*>(sp + C::OFF_X) + ko;
        const uint8_t* bb = act_in ? act_h + kabs * 32 : sp + C::OFF_B + ko * 32;
        const int brs = act_in ? C::ACT_ROW : C::BROW, xw = act_in ? C::ACT_SROW : C::XROW / 4;
        if constexpr (QS_I4_EARLY && C::SINGLE) {
          auto release = [&] {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty_b[s]);
          };
          if (nks >= C::HKS)
            i4_steps_early<C, GKS>(wa, bb, pp, xsm, C::HKS, g, t4, acc, gb, release);
          else
            i4_steps_early<C, GKS>(wa, bb, pp, xsm, nks, g, t4, acc, gb, release);
          if (++s == C::NSTAGE) {
            s = 0;
            ph ^= 1;
          }
          continue;
        }
        if (P.dbg & 2)
          i4_steps<C, NTC, GKS, CW, true>(wa, bb, pp, xsm, min(nks, C::HKS), g, t4, acc, brs, xw, gb);
        else if (nks >= C::HKS)
          i4_steps<C, NTC, GKS, CW>(wa, bb, pp, xsm, C::HKS, g, t4, acc, brs, xw, gb);
        else
          i4_steps<C, NTC, GKS, CW>(wa, bb, pp, xsm, nks, g, t4, acc, brs, xw, gb);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_b[s]);
      if (++s == C::NSTAGE) {
        s = 0;
        ph ^= 1;
      }
    }
    // ---- sum the k-parts of each tile in order (0 + 1 + ... ), then the epilogue ----
    i4_quad_sum<NTC, CW>(acc);
    if (kp > 0) {
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          hsm[((kp - 1) * 32 + rr + (e >> 1) * 8) * COLS + nt * 8 + 2 * t4 + (e & 1)] = acc[nt][e];
    }
    asm volatile("bar.sync 2, %0;" ::"n"(C::NCW * 32));
    if (kp == 0) {
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = (rr + (e >> 1) * 8) * COLS + nt * 8 + 2 * t4 + (e & 1);
          float a = acc[nt][e];
#pragma unroll
          for (int k = 0; k < C::KP - 1; ++k) a = __fadd_rn(a, hsm[k * 32 * COLS + idx]);
          ysm[idx] = a;
        }
    }
    asm volatile("bar.sync 2, %0;" ::"n"(C::NCW * 32));
    linear_epilogue<EPI, COLS, C::NCW * 32>(P, ysm, tp * 32, 32, tid, ncols);
    asm volatile("bar.sync 2, %0;" ::"n"(C::NCW * 32));  // ysm / hsm reuse by the next pair
  }
}

// ---------------------------------------------------------------------------
// f16 W16A16 GEMV/GEMM (the target's weights): the same persistent tile-pair scheme as
// linear_i4_kernel over pair-major frag16 weights ([pair][k-step][2 tiles][32 lanes][8 halves]).
// The schedule (grid = min(pairs, SMs), 8 k-parts per tile, fixed summation order) does not
// depend on the number of activation rows, so a T-row verify equals T one-row steps bit for bit.
// ---------------------------------------------------------------------------
#ifndef QS_F16_L2PF
#define QS_F16_L2PF 0  // A/B: L2 bulk prefetch this many ring depths ahead of the TMA ring (0: off)
#endif
template <int NTC>
struct F16Cfg {
  static constexpr int KP = 8;
  static constexpr int NCW = 2 * KP;
  static constexpr int THREADS = (NCW + 1) * 32;
  // k-steps per stage (32 KB of weights); fixed for every NTC: the k-step -> (k-part, chain)
  // mapping, hence each column's summation order, must not depend on the number of columns
  static constexpr int KCH = 32;
  static constexpr int HKS = KCH / KP;
  static constexpr int WBYTES = KCH * 1024;
  static constexpr int ROWS = 8 * NTC;
  static constexpr int BROW = KCH * 32 + 16;
  static constexpr int OFF_B = WBYTES;
  static constexpr int STAGE = (OFF_B + ROWS * BROW + 127) / 128 * 128;
  static constexpr int YCOLS = 8 * NTC;
  // single-column steps may build their f16 activation row in-kernel (ACT_K <= 4096)
  static constexpr int ACT_K = 4096;
  static constexpr int ACT_ROW = NTC == 1 ? ACT_K * 2 : 0;
  static constexpr int ACT_SROW = NTC == 1 ? ACT_K / 16 * 4 : 0;
  static constexpr int FIXED = KP * 32 * YCOLS * 4 + 2 * 8 * 8 + 16 + ACT_ROW + ACT_SROW;
  static constexpr int NSTAGE = (232448 - FIXED) / STAGE < 8 ? (232448 - FIXED) / STAGE : 8;
  static constexpr int SMEM = NSTAGE * STAGE + FIXED;
  static_assert(NSTAGE >= 2, "f16 linear ring needs two stages");
};

template <int NTC, int EPI>
__global__ void __launch_bounds__(F16Cfg<NTC>::THREADS) linear_f16p_kernel(const __grid_constant__ LinearParams P) {
  using C = F16Cfg<NTC>;
  constexpr int COLS = 8 * NTC;
  constexpr int KCH = C::KCH;
  extern __shared__ __align__(128) uint8_t sm[];
  float* ysm = reinterpret_cast<float*>(sm + C::NSTAGE * C::STAGE);
  float* hsm = ysm + 32 * COLS;
  uint64_t* full_b = reinterpret_cast<uint64_t*>(hsm + (C::KP - 1) * 32 * COLS);
  uint64_t* empty_b = full_b + 8;
  uint8_t* act_h = reinterpret_cast<uint8_t*>(empty_b + 8) + 16;  // [ACT_ROW] f16 row
  float* act_s = reinterpret_cast<float*>(act_h + C::ACT_ROW);     // 16-sums (unused by the f16 math)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int KS = P.K / 16;
  const int TP = (P.N / 16 + 1) / 2;
  const bool act_in = C::ACT_ROW > 0 && P.xf != nullptr;
  const int nst = (KS + KCH - 1) / KCH;
  const int npairs = (TP - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x;
  const int total = npairs * nst;
  const int ncols = P.ncols;

  if (tid == 0) {
    for (int s = 0; s < C::NSTAGE; ++s) {
      mbar_init(&full_b[s], 1);
      mbar_init(&empty_b[s], C::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == C::NCW) {
    auto issue_static = [&](int q) {
      const int s = q % C::NSTAGE;
      const int tp = blockIdx.x + (q / nst) * gridDim.x, u = q % nst;
      const int ks0 = u * KCH, nks = min(KCH, KS - ks0);
      const uint32_t wb = (uint32_t)nks * 1024, bb = (uint32_t)nks * 32;
      mbar_arrive_expect_tx(&full_b[s], wb + (act_in ? 0u : ncols * bb));
      bulk_g2s(sm + s * C::STAGE, reinterpret_cast<const uint8_t*>(P.w) + ((size_t)tp * KS + ks0) * 1024, wb, &full_b[s]);
      if constexpr (QS_F16_L2PF > 0) {
        const int qp = q + C::NSTAGE * QS_F16_L2PF;
        if (qp < total) {
          const int tpp = blockIdx.x + (qp / nst) * gridDim.x, up = qp % nst;
          const int pks0 = up * KCH, pnks = min(KCH, KS - pks0);
          bulk_prefetch_l2(reinterpret_cast<const uint8_t*>(P.w) + ((size_t)tpp * KS + pks0) * 1024, (uint32_t)pnks * 1024);
        }
      }
    };
    auto issue_act = [&](int q) {
      const int s = q % C::NSTAGE, u = q % nst;
      const int ks0 = u * KCH, nks = min(KCH, KS - ks0);
      const uint32_t bb = (uint32_t)nks * 32;
      for (int c = 0; c < ncols; ++c)
        bulk_g2s(sm + s * C::STAGE + C::OFF_B + c * C::BROW,
                 reinterpret_cast<const __half*>(P.xh) + (size_t)c * P.ldxh + ks0 * 16, bb, &full_b[s]);
    };
    const int npre = min(total, C::NSTAGE);
    if (lane == 0)
      for (int q = 0; q < npre; ++q) issue_static(q);
    pdl_wait();
    pdl_trigger();
    if (lane == 0) {
      for (int q = 0; q < total; ++q) {
        if (q >= npre) {
          mbar_wait(&empty_b[q % C::NSTAGE], ((q / C::NSTAGE) - 1) & 1);
          issue_static(q);
        }
        if (!act_in) issue_act(q);
      }
    }
    __syncwarp();
    return;
  }
  pdl_wait();
  pdl_trigger();
  if (act_in) act_prep_row<C::NCW * 32>(P.xf, P.gain, P.eps, P.K, reinterpret_cast<__half*>(act_h), act_s, ysm, tid);

  const int tile = warp & 1, kp = warp >> 1;
  const int rr = tile * 16 + g;
  int s = 0, ph = 0;
  for (int pi = 0; pi < npairs; ++pi) {
    const int tp = blockIdx.x + pi * gridDim.x;
    float acc[NTC][4], acc1[NTC][4];
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = acc1[nt][e] = 0.f;
    for (int u = 0; u < nst; ++u) {
      mbar_wait(&full_b[s], ph);
      const int ko = kp * C::HKS;
      const int nks = min(KCH, KS - u * KCH) - ko;
      if (nks > 0 && !(P.dbg & 1)) {
        const uint8_t* sp = sm + s * C::STAGE;
        const uint4* wa = reinterpret_cast<const uint4*>(sp) + ko * 64 + tile * 32 + lane;
        // B rows: the streamed activation rows, or every lane on the in-kernel row (ncols == 1)
        const uint8_t* bst = act_in ? act_h + 4 * t4 + (u * KCH + ko) * 32
                                    : sp + C::OFF_B + g * C::BROW + 4 * t4 + ko * 32;
#pragma unroll
        for (int ks = 0; ks < C::HKS; ++ks) {
          if (ks < nks) {
            const uint4 w4 = wa[ks * 64];
            const uint32_t a[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
            for (int nt = 0; nt < NTC; ++nt) {
              const uint8_t* row = bst + nt * 8 * C::BROW + ks * 32;
              mma_acc((ks & 1) ? acc1[nt] : acc[nt], a, *reinterpret_cast<const uint32_t*>(row),
                      *reinterpret_cast<const uint32_t*>(row + 16));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty_b[s]);
      if (++s == C::NSTAGE) {
        s = 0;
        ph ^= 1;
      }
    }
#pragma unroll
    for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[nt][e] = __fadd_rn(acc[nt][e], acc1[nt][e]);
    if (kp > 0) {
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e)
          hsm[((kp - 1) * 32 + rr + (e >> 1) * 8) * COLS + nt * 8 + 2 * t4 + (e & 1)] = acc[nt][e];
    }
    asm volatile("bar.sync 2, %0;" ::"n"(C::NCW * 32));
    if (kp == 0) {
#pragma unroll
      for (int nt = 0; nt < NTC; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int idx = (rr + (e >> 1) * 8) * COLS + nt * 8 + 2 * t4 + (e & 1);
          float a = acc[nt][e];
#pragma unroll
          for (int k = 0; k < C::KP - 1; ++k) a = __fadd_rn(a, hsm[k * 32 * COLS + idx]);
          ysm[idx] = a;
        }
    }
    asm volatile("bar.sync 2, %0;" ::"n"(C::NCW * 32));
    linear_epilogue<EPI, COLS, C::NCW * 32>(P, ysm, tp * 32, 32, tid, ncols);
    asm volatile("bar.sync 2, %0;" ::"n"(C::NCW * 32));
  }
}

template <int NTC, int EPI>
static cudaError_t launch_f16p_t(const LinearParams& p, cudaStream_t s) {
  using C = F16Cfg<NTC>;
  auto kern = linear_f16p_kernel<NTC, EPI>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int pairs = (p.N / 16 + 1) / 2;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return launch_pdl(kern, dim3(pairs < sms ? pairs : sms), dim3(C::THREADS), C::SMEM, s, p);
}

template <int NTC>
static cudaError_t launch_f16p_e(const LinearParams& p, cudaStream_t s) {
  switch (p.epi) {
    case QS_EPI_STORE: return launch_f16p_t<NTC, QS_EPI_STORE>(p, s);
    case QS_EPI_ADD: return launch_f16p_t<NTC, QS_EPI_ADD>(p, s);
    case QS_EPI_QKV: return launch_f16p_t<NTC, QS_EPI_QKV>(p, s);
    case QS_EPI_SILU_MUL: return launch_f16p_t<NTC, QS_EPI_SILU_MUL>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int NTC, int EPI, int GKS, int CW, int KC>
static cudaError_t launch_i4_t(const LinearParams& p, cudaStream_t s) {
  using C = I4Cfg<NTC, GKS, CW, KC>;
  auto kern = linear_i4_kernel<NTC, EPI, GKS, CW, KC>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  const int pairs = (p.N / 16 + 1) / 2;
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int slots = sms * C::MINB;
  return launch_pdl(kern, dim3(pairs < slots ? pairs : slots), dim3(C::THREADS), C::SMEM, s, p);
}

template <int NTC, int GKS, int CW, int KC = 0>
static cudaError_t launch_i4_e(const LinearParams& p, cudaStream_t s) {
  switch (p.epi) {
    case QS_EPI_STORE: return launch_i4_t<NTC, QS_EPI_STORE, GKS, CW, KC>(p, s);
    case QS_EPI_ADD: return launch_i4_t<NTC, QS_EPI_ADD, GKS, CW, KC>(p, s);
    case QS_EPI_QKV: return launch_i4_t<NTC, QS_EPI_QKV, GKS, CW, KC>(p, s);
    case QS_EPI_SILU_MUL: return launch_i4_t<NTC, QS_EPI_SILU_MUL, GKS, CW, KC>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int GKS>
static cudaError_t launch_i4_n(const LinearParams& p, cudaStream_t s) {
#ifndef QS_I4_BIGK
#define QS_I4_BIGK 0  // A/B: single-row launches with K <= this stream 256-k-step stages (0: never)
#endif
  if constexpr (QS_I4_BIGK > 0)
    if (p.ncols == 1 && p.K <= QS_I4_BIGK) return launch_i4_e<1, GKS, 1, 256>(p, s);
  if (p.ncols == 1) return launch_i4_e<1, GKS, 1>(p, s);
  if (p.ncols == 2) return launch_i4_e<1, GKS, 2>(p, s);
  if (p.ncols <= 4) return launch_i4_e<1, GKS, 4>(p, s);
  if (p.ncols <= 8) return launch_i4_e<1, GKS, 8>(p, s);
  if (p.ncols <= 16) return launch_i4_e<2, GKS, 8>(p, s);
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// activation prep: f16 copy (optionally RMS-normalised) + 16-sums
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) prep_act_kernel(const float* __restrict__ x, const float* __restrict__ gain,
                                                       float eps, __half* __restrict__ xh, long long ldxh,
                                                       float* __restrict__ xs, long long ldxs, int d) {
  pdl_wait();
  pdl_trigger();
  __shared__ float red[33];
  act_prep_row<0>(x + (size_t)blockIdx.x * d, gain, eps, d, xh + (size_t)blockIdx.x * ldxh,
                  xs + (size_t)blockIdx.x * ldxs, red, threadIdx.x);
}

cudaError_t launch_prep_act(const float* x, const float* gain, float eps, void* xh, long long ldxh, float* xs,
                            long long ldxs, int n, int d, cudaStream_t s) {
  return launch_pdl(prep_act_kernel, dim3(n), dim3(256), 0, s, x, gain, eps, reinterpret_cast<__half*>(xh), ldxh, xs, ldxs, d);
}

cudaError_t launch_linear(const LinearParams& p, cudaStream_t s) {
  if (p.wmode == QS_W_F16) {
    switch ((p.ncols + 7) / 8) {
      case 1: return launch_f16p_e<1>(p, s);
      case 2: return launch_f16p_e<2>(p, s);
      case 3: return launch_f16p_e<3>(p, s);
      case 4: return launch_f16p_e<4>(p, s);
      case 5: return launch_f16p_e<5>(p, s);
      case 6: return launch_f16p_e<6>(p, s);
      default: return cudaErrorInvalidValue;
    }
  }
  if (p.wmode == QS_W_INT4) {
    switch (p.wgroup) {
      case 16: return launch_i4_n<1>(p, s);
      case 32: return launch_i4_n<2>(p, s);
      case 64: return launch_i4_n<4>(p, s);
      case 128: return launch_i4_n<8>(p, s);
      default: return cudaErrorInvalidValue;
    }
  }
  return cudaErrorInvalidValue;
}


}  // namespace qs
