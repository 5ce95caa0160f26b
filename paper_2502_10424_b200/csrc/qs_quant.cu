// Quantisation kernels (sm_100a): plane encode/decode, INT4 weights, KV-block
// flush.  All code/scale arithmetic runs in f64 with explicitly rounded
// operations (no FMA contraction) so codes, scales and zero points are
// bit-identical to the NumPy reference:
//   asymmetric upper plane   /root/reference/pkg/src/quantspec/quant.py:220-248
//   hierarchical lower plane /root/reference/pkg/src/quantspec/quant.py:251-276
//   round half away          /root/reference/pkg/src/quantspec/quant.py:55-57
//   nibble packing           /root/reference/pkg/src/quantspec/quant.py:137-158
//   weight planes            /root/reference/pkg/src/quantspec/quant.py:335-356
//   KV block quantisation    /root/reference/pkg/src/quantspec/cache.py:283-303
#include <math.h>

#include "qs_common.cuh"
#include "qs_layout.h"
#include "qs_api_internal.h"

namespace qs {

// ---------------------------------------------------------------------------
// exact scalar recipe shared by every encoder
// ---------------------------------------------------------------------------
__device__ __forceinline__ double rha(double x) {
  // trunc(x + copysign(0.5, x)) with the addition rounded in f64
  return trunc(__dadd_rn(x, copysign(0.5, x)));
}

struct UParams {
  float s, z;
};

__device__ __forceinline__ UParams asym_params(double mn, double mx) {
  UParams p;
  p.z = __double2float_rn(mn);
  double s = __ddiv_rn(__dsub_rn(mx, (double)p.z), 15.0);
  s = s > 1e-8 ? s : 1e-8;
  p.s = __double2float_rn(s);
  return p;
}

__device__ __forceinline__ int code_upper(double v, UParams p) {
  double x = rha(__ddiv_rn(__dsub_rn(v, (double)p.z), (double)p.s));
  x = fmin(fmax(x, 0.0), 15.0);
  return (int)x;
}

__device__ __forceinline__ int code_lower(double v, int cu, UParams p) {
  double recon = __dadd_rn(__dmul_rn((double)cu, (double)p.s), (double)p.z);
  double r = __dsub_rn(v, recon);
  double sl = (double)(p.s * 0.0625f);  // f32 division by 16 is exact
  double x = rha(__ddiv_rn(r, sl));
  x = fmin(fmax(x, -8.0), 7.0);
  return (int)x;
}

__device__ __forceinline__ bool finite_d(double v) { return isfinite(v); }

// group geometry of a flat plane (Q/quant.py:210-217)
struct PlaneGeom {
  long long count;
  int group;
  long long row_len;  // 0 = none
  __device__ __forceinline__ bool rows() const { return row_len > 0 && row_len < count; }
  __device__ __forceinline__ long long gpr() const { return (row_len + group - 1) / group; }
  __device__ __forceinline__ long long ngroups() const {
    return rows() ? (count / row_len) * gpr() : (count + group - 1) / group;
  }
  __device__ __forceinline__ void span(long long gi, long long& start, int& len) const {
    if (rows()) {
      long long row = gi / gpr(), j = gi % gpr();
      start = row * row_len + j * group;
      len = (int)min((long long)group, row_len - j * group);
    } else {
      start = gi * group;
      len = (int)min((long long)group, count - start);
    }
  }
  __device__ __forceinline__ long long group_of(long long i) const {
    if (rows()) return (i / row_len) * gpr() + (i % row_len) / group;
    return i / group;
  }
};

// phase 1: one warp per group -> (S, Z)
__global__ void plane_params_kernel(const double* __restrict__ v, PlaneGeom geo, float* __restrict__ s_out,
                                    float* __restrict__ z_out, float* __restrict__ sl_out, int* flags) {
  long long gi = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (gi >= geo.ngroups()) return;
  long long st;
  int len;
  geo.span(gi, st, len);
  double mn = INFINITY, mx = -INFINITY;
  bool bad = false;
  for (int i = lane; i < len; i += 32) {
    double x = v[st + i];
    bad |= !finite_d(x);
    mn = fmin(mn, x);
    mx = fmax(mx, x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    if (bad && flags) atomicOr(flags, 1);
    UParams p = asym_params(mn, mx);
    s_out[gi] = p.s;
    z_out[gi] = p.z;
    if (sl_out) sl_out[gi] = p.s * 0.0625f;
  }
}

// phase 2: one thread per packed byte (two codes, possibly of two groups)
__global__ void plane_codes_kernel(const double* __restrict__ v, PlaneGeom geo, const float* __restrict__ s,
                                   const float* __restrict__ z, uint8_t* __restrict__ up,
                                   uint8_t* __restrict__ lo) {
  long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long nbytes = (geo.count + 1) / 2;
  if (b >= nbytes) return;
  int u[2] = {0, 0}, l[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    long long i = 2 * b + h;
    if (i < geo.count) {
      long long gi = geo.group_of(i);
      UParams p{s[gi], z[gi]};
      double x = v[i];
      u[h] = code_upper(x, p);
      if (lo) l[h] = code_lower(x, u[h], p);
    }
  }
  up[b] = (uint8_t)((u[0] & 0xF) | ((u[1] & 0xF) << 4));
  if (lo) lo[b] = (uint8_t)((l[0] & 0xF) | ((l[1] & 0xF) << 4));
}

__global__ void plane_decode_kernel(const uint8_t* __restrict__ up, const uint8_t* __restrict__ lo,
                                    const float* __restrict__ s, const float* __restrict__ z, PlaneGeom geo,
                                    double* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= geo.count) return;
  long long gi = geo.group_of(i);
  int cu = (up[i >> 1] >> ((i & 1) * 4)) & 0xF;
  double se = (double)s[gi], ze = (double)z[gi];
  double r = __dmul_rn((double)cu, se);
  if (lo) {
    int cl = (lo[i >> 1] >> ((i & 1) * 4)) & 0xF;
    cl = cl >= 8 ? cl - 16 : cl;
    r = __dadd_rn(r, __dmul_rn((double)cl, __ddiv_rn(se, 16.0)));
  }
  out[i] = __dadd_rn(r, ze);
}

// caller-fixed symmetric quantiser (Q/quant.py:83-91): clip(rha(e / f32(scale)), -8, 7)
__global__ void sym_s4_kernel(const double* __restrict__ e, long long n, double scale, int8_t* __restrict__ out,
                              int* flags) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = e[i];
  if (!finite_d(x) && flags) atomicOr(flags, 1);
  double c = fmin(fmax(rha(__ddiv_rn(x, scale)), -8.0), 7.0);
  out[i] = (int8_t)c;
}

cudaError_t launch_sym_s4(const double* e, long long n, float scale, int8_t* out, int* flags, cudaStream_t st) {
  sym_s4_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(e, n, (double)scale, out, flags);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// INT4 weights: W [d_in][d_out] f32 -> plane over W^T rows (groups along d_in)
// ---------------------------------------------------------------------------
struct WGeom {
  int d_in, d_out, g, gpr;
};

__global__ void wq_params_kernel(const float* __restrict__ w, WGeom geo, float* __restrict__ s_out,
                                 float* __restrict__ z_out, int* flags) {
  long long gi = (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  int lane = threadIdx.x & 31;
  if (gi >= (long long)geo.d_out * geo.gpr) return;
  int n = (int)(gi / geo.gpr), j = (int)(gi % geo.gpr);
  int k0 = j * geo.g, len = min(geo.g, geo.d_in - k0);
  double mn = INFINITY, mx = -INFINITY;
  bool bad = false;
  for (int i = lane; i < len; i += 32) {
    double x = (double)w[(size_t)(k0 + i) * geo.d_out + n];
    bad |= !finite_d(x);
    mn = fmin(mn, x);
    mx = fmax(mx, x);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    mn = fmin(mn, __shfl_xor_sync(0xffffffffu, mn, o));
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  }
  bad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    if (bad && flags) atomicOr(flags, 1);
    UParams p = asym_params(mn, mx);
    s_out[gi] = p.s;
    z_out[gi] = p.z;
  }
}

__device__ __forceinline__ int wcode(const float* w, WGeom geo, const float* s, const float* z, int n, int k) {
  int gi = n * geo.gpr + k / geo.g;
  return code_upper((double)w[(size_t)k * geo.d_out + n], UParams{s[gi], z[gi]});
}

// reference packing: flat index i = n*d_in + k, two per byte
__global__ void wq_refcodes_kernel(const float* __restrict__ w, WGeom geo, const float* __restrict__ s,
                                   const float* __restrict__ z, uint8_t* __restrict__ out) {
  long long b = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  long long count = (long long)geo.d_in * geo.d_out;
  if (b >= (count + 1) / 2) return;
  int c[2] = {0, 0};
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    long long i = 2 * b + h;
    if (i < count) c[h] = wcode(w, geo, s, z, (int)(i / geo.d_in), (int)(i % geo.d_in));
  }
  out[b] = (uint8_t)(c[0] | (c[1] << 4));
}

// frag4 words, tile-pair major: [pair][KSpad/4][2 tiles][32 lanes][4]  (tile mt = 2 pair + w; A = W^T
// tile, rows = outputs, cols = d_in).  A 64-k-step stage of one pair (linear_i4_kernel) is one
// contiguous range; a padding tile (odd d_out/16) is zero.
__global__ void wq_frag_kernel(const float* __restrict__ w, WGeom geo, const float* __restrict__ s,
                               const float* __restrict__ z, uint32_t* __restrict__ frag, int ks_pad) {
  long long wi = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int MT = geo.d_out / 16, MT2 = (MT + 1) / 2 * 2;
  long long nwords = (long long)MT2 * ks_pad * 32;
  if (wi >= nwords) return;
  int v4 = (int)(wi & 3);
  long long rest = wi >> 2;
  int lane = (int)(rest & 31);
  rest >>= 5;
  int wt = (int)(rest & 1);
  rest >>= 1;
  int kq = (int)(rest % (ks_pad / 4));
  int mt = (int)(rest / (ks_pad / 4)) * 2 + wt;
  int ks = kq * 4 + v4;
  int g = lane >> 2, t = lane & 3;
  uint32_t word = 0;
  if (ks * 16 < geo.d_in && mt < MT) {
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      int j = p & 3, h = p >> 2;
      int row = g + 8 * (j & 1), col = 2 * t + 8 * (j >> 1) + h;
      int n = mt * 16 + row, k = ks * 16 + col;
      int c = wcode(w, geo, s, z, n, k);
      word |= (uint32_t)c << (4 * p);
    }
  }
  frag[wi] = word;
}

// params, tile-pair major: float4 per [pair][group][2 tiles][8 slots] (zeros for a padding tile);
// row g of group grp sits in slot g ^ i4_param_swz(grp) (qs_common.cuh: the consumer lanes of one
// load read four different groups, which the swizzle spreads over distinct banks)
__global__ void wq_fragparams_kernel(WGeom geo, const float* __restrict__ s, const float* __restrict__ z,
                                     float4* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int MT = geo.d_out / 16, MT2 = (MT + 1) / 2 * 2;
  long long total = (long long)MT2 * geo.gpr * 8;
  if (i >= total) return;
  long long rest = i >> 3;
  int wt = (int)(rest & 1);
  rest >>= 1;
  int grp = (int)(rest % geo.gpr);
  int g = (int)(i & 7) ^ i4_param_swz(grp);
  int mt = (int)(rest / geo.gpr) * 2 + wt;
  if (mt >= MT) {
    out[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  int n0 = mt * 16 + g, n1 = n0 + 8;
  // pre-folded for the offset-form MMA (qs_gemm.cu): rows g carry 1024 + c, rows g+8 carry 1024 + 16c
  //   {S_g, Z_g - 1024 S_g, S_g8 / 16, Z_g8 - 64 S_g8}
  const float s0 = s[n0 * geo.gpr + grp], z0 = z[n0 * geo.gpr + grp];
  const float s1 = s[n1 * geo.gpr + grp], z1 = z[n1 * geo.gpr + grp];
  out[i] = make_float4(s0, __fmaf_rn(-1024.f, s0, z0), __fmul_rn(s1, 0.0625f), __fmaf_rn(-64.f, s1, z1));
}

// fp16 frag layout, tile-pair major: [pair][ks][2 tiles][32 lanes][8 halves] (tile mt = 2 pair + w;
// a padding tile (odd d_out/16) is zero).  A stage of k-steps of one pair is one contiguous range.
__global__ void pack_f16_kernel(const float* __restrict__ w, int d_in, int d_out, __half* __restrict__ out) {
  long long li = (long long)blockIdx.x * blockDim.x + threadIdx.x;  // (pair, ks, w, lane)
  const int KS = d_in / 16, MT = d_out / 16, MT2 = (MT + 1) / 2 * 2;
  long long total = (long long)MT2 * KS * 32;
  if (li >= total) return;
  int lane = (int)(li & 31);
  long long rest = li >> 5;
  int wt = (int)(rest & 1);
  rest >>= 1;
  int ks = (int)(rest % KS), mt = (int)(rest / KS) * 2 + wt;
  int g = lane >> 2, t = lane & 3;
  __align__(16) __half hv[8];
#pragma unroll
  for (int slot = 0; slot < 8; ++slot) {
    int j = slot >> 1, h = slot & 1;
    int row = g + 8 * (j & 1), col = 2 * t + 8 * (j >> 1) + h;
    hv[slot] = mt < MT ? __float2half_rn(w[(size_t)(ks * 16 + col) * d_out + mt * 16 + row]) : __float2half_rn(0.f);
  }
  *reinterpret_cast<uint4*>(out + li * 8) = *reinterpret_cast<uint4*>(hv);
}

// ---------------------------------------------------------------------------
// K1: KV block quantisation into the store (Q/cache.py:283-303).
// One CTA (256 threads) per (seq, layer, kv head, block):
//   1. the block's K rows of this head [G][hd] (one contiguous range of the head-major source)
//      and the V rows of its value group's channels [G][cg1 - cg0] are staged in shared memory
//      with 16-byte coalesced loads;
//   2. key (S, Z): one group per channel over the G tokens (lanes = channels, token parts
//      combined through shared memory); value (S, Z): one group per token over the group's
//      channels (a warp per token, shuffle min/max);
//   3. every thread builds four consecutive frag4 words per plane straight from the staged
//      values -- one 16-byte store per plane, consecutive threads -> consecutive addresses.
// Codes use a two-level division: q = (v - Z) * (1/S) in f64 decides the rounding whenever q is
// farther than 2^-30 from a half-integer; only near a tie does the exact __ddiv_rn path of the
// reference recipe run, so codes stay bit-identical to Q/quant.py:220-276 in every case.
// ---------------------------------------------------------------------------
constexpr int KQ_THREADS = 256;

struct KVQArgs {
  qs_kv_store st;
  int seq, layer0, dst_block0;
  const __half* src_k;
  const __half* src_v;
  long long src_layer_stride, src_head_stride;  // halves
  int* flags;
};

__device__ __forceinline__ bool layer_sensitive(const qs_kv_store& st, int l) {
  return (st.sens_mask[l >> 6] >> (l & 63)) & 1ull;
}
__device__ __forceinline__ int sens_slot(const qs_kv_store& st, int l) {
  int c = 0;
  for (int i = 0; i < l; ++i) c += layer_sensitive(st, i) ? 1 : 0;
  return c;
}
__device__ __forceinline__ int sens_count(const qs_kv_store& st) {
  return __popcll(st.sens_mask[0]) + __popcll(st.sens_mask[1]);
}

// round-half-away of fl(d / s) (the reference's rha((v - Z) / S)), decided by a reciprocal
// multiply unless the quotient sits within 2^-30 of a tie
__device__ __forceinline__ double rha_div(double d, double s, double inv_s) {
  const double q = d * inv_s;
  const double a = fabs(q);
  const double f = a - floor(a);
  if (fabs(f - 0.5) > 9.313225746154785e-10) return copysign(floor(a + 0.5), q);
  return rha(__ddiv_rn(d, s));
}

__device__ __forceinline__ void codes_pair(double v, double s, double z, double inv_s, int& cu, int& cl) {
  double x = rha_div(__dsub_rn(v, z), s, inv_s);
  x = fmin(fmax(x, 0.0), 15.0);
  cu = (int)x;
  const double recon = __dadd_rn(__dmul_rn((double)cu, s), z);
  const double r = __dsub_rn(v, recon);
  const double sl = (double)((float)s * 0.0625f);
  double y = rha_div(r, sl, inv_s * 16.0);
  y = fmin(fmax(y, -8.0), 7.0);
  cl = (int)y;
}

// One (layer, head, block) job: sk / sv point at row 0 of this head's block in a head-major
// source (head stride hs halves, row stride hd); writes planes + params of block dblk.
__device__ void kv_block_job(const qs_kv_store& st, int seq, int layer, int h, int dblk, const __half* sk,
                             const __half* sv_head0, long long hs, int* flags, uint8_t* smem) {
  const int G = st.G, HD = st.hd, H = st.Hkv, kv = H * HD;
  const int tid = threadIdx.x;
  const int cg0 = ((h * HD) / G) * G, cg1 = min(cg0 + G, kv), nv = cg1 - cg0;
  __half* ks = reinterpret_cast<__half*>(smem);  // [G][HD]
  __half* vs = ks + G * HD;                      // [G][nv]
  float2* kpar = reinterpret_cast<float2*>(vs + G * nv);  // [HD]
  float2* vpar = kpar + HD;                               // [G]
  double* kinv = reinterpret_cast<double*>(vpar + G);     // [HD] 1/S_k
  double* vinv = kinv + HD;                               // [G]  1/S_v
  float* red = reinterpret_cast<float*>(vinv + G);        // [KQ_THREADS][2]
  // ---- stage (16-byte loads; the block of one head is contiguous) ----
  {
    const uint4* src = reinterpret_cast<const uint4*>(sk);
    uint4* dst = reinterpret_cast<uint4*>(ks);
    for (int i = tid; i < G * HD / 8; i += KQ_THREADS) dst[i] = src[i];
    for (int i = tid; i < G * nv / 8; i += KQ_THREADS) {
      const int r = i / (nv / 8), cc = (i % (nv / 8)) * 8;  // channel offset inside the group
      const int c = cg0 + cc, hh = c / HD, ci = c % HD;
      reinterpret_cast<uint4*>(vs)[i] =
          reinterpret_cast<const uint4*>(sv_head0 + (size_t)hh * hs + (size_t)r * HD + ci)[0];
    }
  }
  __syncthreads();
  bool bad = false;
  // ---- key params: channel c = tid % HD, token part tid / HD ----
  {
    const int parts = KQ_THREADS / HD;
    const int c = tid % HD, part = tid / HD;
    float mn = INFINITY, mx = -INFINITY;
    for (int r = part; r < G; r += parts) {
      const float x = __half2float(ks[r * HD + c]);
      bad |= !isfinite(x);
      mn = fminf(mn, x);
      mx = fmaxf(mx, x);
    }
    red[2 * tid] = mn;
    red[2 * tid + 1] = mx;
    __syncthreads();
    if (part == 0) {
      for (int p = 1; p < parts; ++p) {
        mn = fminf(mn, red[2 * (p * HD + c)]);
        mx = fmaxf(mx, red[2 * (p * HD + c) + 1]);
      }
      const UParams pr = asym_params((double)mn, (double)mx);
      kpar[c] = make_float2(pr.s, pr.z);
      kinv[c] = 1.0 / (double)pr.s;
    }
  }
  // ---- value params: a warp per token, lanes over the group's channels ----
  {
    const int lane = tid & 31, warp = tid >> 5;
    for (int r = warp; r < G; r += KQ_THREADS / 32) {
      float mn = INFINITY, mx = -INFINITY;
      for (int c = lane; c < nv; c += 32) {
        const float x = __half2float(vs[r * nv + c]);
        bad |= !isfinite(x);
        mn = fminf(mn, x);
        mx = fmaxf(mx, x);
      }
      mn = warp_min_f(mn);
      mx = warp_max(mx);
      if (lane == 0) {
        const UParams pr = asym_params((double)mn, (double)mx);
        vpar[r] = make_float2(pr.s, pr.z);
        vinv[r] = 1.0 / (double)pr.s;
      }
    }
  }
  if (__syncthreads_or(bad) && tid == 0 && flags) atomicOr(flags, 1);
  const size_t slh = ((size_t)seq * st.L + layer) * H + h;
  float2* kp = reinterpret_cast<float2*>(st.kp) + (slh * st.max_blocks + dblk) * HD;
  float2* vp = reinterpret_cast<float2*>(st.vp) + (slh * st.max_blocks + dblk) * G;
  for (int c = tid; c < HD; c += KQ_THREADS) kp[c] = kpar[c];
  for (int r = tid; r < G; r += KQ_THREADS) vp[r] = vpar[r];
  // ---- frag4 words: thread -> 4 consecutive words (inner tiles i4..i4+3 of one (outer, lane)) ----
  const int NI = HD / 16, VEC = qs_vec(NI);
  const int nwords = G * HD / 8;
  const size_t pb = (size_t)G * HD / 2;
  const size_t poff = (slh * st.max_blocks + dblk) * pb;
  uint32_t* oku = reinterpret_cast<uint32_t*>(st.ku + poff);
  uint32_t* okl = reinterpret_cast<uint32_t*>(st.kl + poff);
  uint32_t* ovu = reinterpret_cast<uint32_t*>(st.vu + poff);
  uint32_t* ovl = reinterpret_cast<uint32_t*>(st.vl + poff);
  const int vofs = h * HD - cg0;  // this head's first channel inside the staged value group
  for (int w0 = tid * VEC; w0 < nwords; w0 += KQ_THREADS * VEC) {
    uint32_t wku[4] = {0, 0, 0, 0}, wkl[4] = {0, 0, 0, 0}, wvu[4] = {0, 0, 0, 0}, wvl[4] = {0, 0, 0, 0};
    for (int e = 0; e < VEC; ++e) {
      const int wi = w0 + e;
      const int vp4 = wi % VEC, rest = wi / VEC;
      const int lane = rest % 32, rest2 = rest / 32;
      const int inner = (rest2 % (NI / VEC)) * VEC + vp4, outer = rest2 / (NI / VEC);
      const int g = lane >> 2, t = lane & 3;
#pragma unroll
      for (int p = 0; p < 8; ++p) {
        const int j = p & 3, hb = p >> 2;
        const int row = g + 8 * (j & 1), col = 2 * t + 8 * (j >> 1) + hb;
        // keys: A = K[token][channel]
        const int tk = outer * 16 + row, ck = inner * 16 + col;
        const float2 pk = kpar[ck];
        int cu, cl;
        codes_pair((double)__half2float(ks[tk * HD + ck]), (double)pk.x, (double)pk.y, kinv[ck], cu, cl);
        wku[e] |= (uint32_t)cu << (4 * p);
        wkl[e] |= (uint32_t)(cl + 8) << (4 * p);
        // values: A = V^T[channel][token]
        const int tv = outer * 16 + col, cv = inner * 16 + row;
        const float2 pv = vpar[tv];
        codes_pair((double)__half2float(vs[tv * nv + vofs + cv]), (double)pv.x, (double)pv.y, vinv[tv], cu, cl);
        wvu[e] |= (uint32_t)cu << (4 * p);
        wvl[e] |= (uint32_t)(cl + 8) << (4 * p);
      }
    }
    if (VEC == 4) {
      reinterpret_cast<uint4*>(oku + w0)[0] = make_uint4(wku[0], wku[1], wku[2], wku[3]);
      reinterpret_cast<uint4*>(okl + w0)[0] = make_uint4(wkl[0], wkl[1], wkl[2], wkl[3]);
      reinterpret_cast<uint4*>(ovu + w0)[0] = make_uint4(wvu[0], wvu[1], wvu[2], wvu[3]);
      reinterpret_cast<uint4*>(ovl + w0)[0] = make_uint4(wvl[0], wvl[1], wvl[2], wvl[3]);
    } else {
      for (int e = 0; e < VEC; ++e) {
        oku[w0 + e] = wku[e];
        okl[w0 + e] = wkl[e];
        ovu[w0 + e] = wvu[e];
        ovl[w0 + e] = wvl[e];
      }
    }
  }
}

// sensitive layers archive fp rows instead of quantising (Q/cache.py:286-289)
__device__ void kv_archive_job(const qs_kv_store& st, int seq, int layer, int h, int dblk, const __half* sk,
                               const __half* sv) {
  const int G = st.G, HD = st.hd, H = st.Hkv;
  const size_t cap = (size_t)st.max_blocks * G;
  const size_t base = ((((size_t)seq * sens_count(st) + sens_slot(st, layer)) * H + h) * cap + (size_t)dblk * G) * HD;
  uint4* ak = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(st.arch_k) + base);
  uint4* av = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(st.arch_v) + base);
  for (int i = threadIdx.x; i < G * HD / 8; i += blockDim.x) {
    ak[i] = reinterpret_cast<const uint4*>(sk)[i];
    av[i] = reinterpret_cast<const uint4*>(sv)[i];
  }
}

__host__ __device__ inline int kq_smem(int G, int hd) { return 2 * G * hd + 2 * G * G + 16 * (hd + G) + 8 * KQ_THREADS; }

// prefill: blocks [0, nblk) of one (seq, layer) from head-major rows; grid (nblk, Hkv, nlayers)
__global__ void __launch_bounds__(KQ_THREADS) kv_quant_kernel(const __grid_constant__ KVQArgs A) {
  extern __shared__ __align__(16) uint8_t sm[];
  const int b = blockIdx.x, h = blockIdx.y, layer = A.layer0 + blockIdx.z;
  const __half* sk = A.src_k + (size_t)blockIdx.z * A.src_layer_stride;
  const __half* sv = A.src_v + (size_t)blockIdx.z * A.src_layer_stride;
  const size_t row0 = (size_t)b * A.st.G * A.st.hd;
  if (layer_sensitive(A.st, layer)) {
    kv_archive_job(A.st, A.seq, layer, h, A.dst_block0 + b, sk + (size_t)h * A.src_head_stride + row0,
                   sv + (size_t)h * A.src_head_stride + row0);
    return;
  }
  kv_block_job(A.st, A.seq, layer, h, A.dst_block0 + b, sk + (size_t)h * A.src_head_stride + row0, sv + row0,
               A.src_head_stride, A.flags, sm);
}

// ---------------------------------------------------------------------------
// Decode-time flush (Q/cache.py:249-281, full-fp1 branch), device-conditioned per sequence so it
// runs inside the captured decode cycle: sequence s flushes iff fp2_len[s] == G and fp1_len[s]
// == G.  Three launches (each reads the lengths the previous one left untouched):
//   kv_flush_quant_kernel  grid (Hkv, L, B): fp1 -> block n_blocks[s] (or the fp16 archive)
//   kv_flush_rotate_kernel grid (Hkv, L, B): fp1 <- fp2 rows [0, G)
//   kv_flush_lengths_kernel: n_blocks[s] += 1, fp2_len[s] -= G
// ---------------------------------------------------------------------------
struct FlushArgs {
  qs_kv_store st;
  const int* n_blocks;
  const int* fp1_len;
  const int* fp2_len;
  int* n_blocks_w;
  int* fp2_len_w;
  int* flags;
};

__device__ __forceinline__ bool flush_due(const FlushArgs& A, int seq) {
  return A.fp2_len[seq] == A.st.G && A.fp1_len[seq] == A.st.G;
}

__global__ void __launch_bounds__(KQ_THREADS) kv_flush_quant_kernel(const __grid_constant__ FlushArgs A) {
  extern __shared__ __align__(16) uint8_t sm[];
  pdl_wait();
  pdl_trigger();
  const int h = blockIdx.x, layer = blockIdx.y, seq = blockIdx.z;
  if (!flush_due(A, seq)) return;
  const qs_kv_store& st = A.st;
  const int dblk = A.n_blocks[seq];
  if (dblk >= st.max_blocks) {
    if (threadIdx.x == 0 && A.flags) atomicOr(A.flags, 4);  // arena full: BufferOverflowError
    return;
  }
  const size_t hs = (size_t)st.fp_rows * st.hd;
  const size_t lbase = (((size_t)seq * st.L + layer) * 2 + 0) * st.Hkv * hs;  // fp1 of (seq, layer)
  const __half* fk = reinterpret_cast<const __half*>(st.fp_k) + lbase;
  const __half* fv = reinterpret_cast<const __half*>(st.fp_v) + lbase;
  if (layer_sensitive(st, layer)) {
    kv_archive_job(st, seq, layer, h, dblk, fk + h * hs, fv + h * hs);
    return;
  }
  kv_block_job(st, seq, layer, h, dblk, fk + h * hs, fv, (long long)hs, A.flags, sm);
}

__global__ void __launch_bounds__(256) kv_flush_rotate_kernel(const __grid_constant__ FlushArgs A) {
  pdl_wait();
  pdl_trigger();
  const int h = blockIdx.x, layer = blockIdx.y, seq = blockIdx.z;
  if (!flush_due(A, seq) || A.n_blocks[seq] >= A.st.max_blocks) return;
  const qs_kv_store& st = A.st;
  const size_t hs = (size_t)st.fp_rows * st.hd;
  const size_t b1 = ((((size_t)seq * st.L + layer) * 2 + 0) * st.Hkv + h) * hs;
  const size_t b2 = b1 + (size_t)st.Hkv * hs;
  uint4* k1 = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(st.fp_k) + b1);
  uint4* v1 = reinterpret_cast<uint4*>(reinterpret_cast<__half*>(st.fp_v) + b1);
  const uint4* k2 = reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(st.fp_k) + b2);
  const uint4* v2 = reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(st.fp_v) + b2);
  for (int i = threadIdx.x; i < st.G * st.hd / 8; i += blockDim.x) {
    k1[i] = k2[i];
    v1[i] = v2[i];
  }
}

__global__ void kv_flush_lengths_kernel(const __grid_constant__ FlushArgs A) {
  pdl_wait();
  pdl_trigger();
  for (int seq = threadIdx.x; seq < A.st.B; seq += blockDim.x) {
    if (!flush_due(A, seq) || A.n_blocks[seq] >= A.st.max_blocks) continue;
    A.n_blocks_w[seq] += 1;
    A.fp2_len_w[seq] -= A.st.G;
  }
}

// f32 view of quantised blocks [0, nblk) of one (seq, layer): Q/cache.py:317-343
__global__ void kv_dequant_kernel(qs_kv_store st, int seq, int layer, int target, float* __restrict__ ok,
                                  float* __restrict__ ov) {
  const int G = st.G, HD = st.hd, H = st.Hkv, kvd = H * HD;
  const int b = blockIdx.x, h = blockIdx.y;
  const size_t slh = ((size_t)seq * st.L + layer) * H + h;
  const size_t pb = (size_t)G * HD / 2;
  const size_t poff = (slh * st.max_blocks + b) * pb;
  const uint32_t* ku = reinterpret_cast<const uint32_t*>(st.ku + poff);
  const uint32_t* kl = reinterpret_cast<const uint32_t*>(st.kl + poff);
  const uint32_t* vu = reinterpret_cast<const uint32_t*>(st.vu + poff);
  const uint32_t* vl = reinterpret_cast<const uint32_t*>(st.vl + poff);
  const float2* kp = reinterpret_cast<const float2*>(st.kp) + (slh * st.max_blocks + b) * HD;
  const float2* vp = reinterpret_cast<const float2*>(st.vp) + (slh * st.max_blocks + b) * G;
  const int NI = HD / 16;
  for (int i = threadIdx.x; i < G * HD; i += blockDim.x) {
    int r = i / HD, c = i % HD;
    int lane, nib;
    // key element (token r, channel c): tile (r/16, c/16), A row = r%16, col = c%16
    qs_frag_pos(r & 15, c & 15, &lane, &nib);
    int wk = qs_frag_index(r >> 4, c >> 4, lane, NI);
    int cu = (ku[wk] >> (4 * nib)) & 0xF;
    int cl = (int)((kl[wk] >> (4 * nib)) & 0xF) - 8;
    float2 p = kp[c];
    double se = p.x, ze = p.y;
    double x = __dmul_rn((double)cu, se);
    if (target) x = __dadd_rn(x, __dmul_rn((double)cl, __ddiv_rn(se, 16.0)));
    x = __dadd_rn(x, ze);
    ok[((size_t)b * G + r) * kvd + h * HD + c] = __double2float_rn(x);
    // value element (token r, channel c): tile (r/16, c/16), A row = c%16 (channel), col = r%16
    qs_frag_pos(c & 15, r & 15, &lane, &nib);
    int wv = qs_frag_index(r >> 4, c >> 4, lane, NI);
    cu = (vu[wv] >> (4 * nib)) & 0xF;
    cl = (int)((vl[wv] >> (4 * nib)) & 0xF) - 8;
    p = vp[r];
    se = p.x;
    ze = p.y;
    x = __dmul_rn((double)cu, se);
    if (target) x = __dadd_rn(x, __dmul_rn((double)cl, __ddiv_rn(se, 16.0)));
    x = __dadd_rn(x, ze);
    ov[((size_t)b * G + r) * kvd + h * HD + c] = __double2float_rn(x);
  }
}

// ---------------------------------------------------------------------------
// host launchers (called from qs_capi.cu)
// ---------------------------------------------------------------------------
static inline unsigned blocks_for(long long n, int bs) { return (unsigned)((n + bs - 1) / bs); }

cudaError_t launch_encode_plane(const double* v, long long count, int group, long long row_len, uint8_t* up,
                                uint8_t* lo, float* s, float* z, float* sl, int* flags, cudaStream_t st) {
  PlaneGeom geo{count, group, row_len};
  long long ng = (row_len > 0 && row_len < count) ? (count / row_len) * ((row_len + group - 1) / group)
                                                   : (count + group - 1) / group;
  plane_params_kernel<<<blocks_for(ng, 8), 256, 0, st>>>(v, geo, s, z, sl, flags);
  plane_codes_kernel<<<blocks_for((count + 1) / 2, 256), 256, 0, st>>>(v, geo, s, z, up, lo);
  return cudaGetLastError();
}

cudaError_t launch_decode_plane(const uint8_t* up, const uint8_t* lo, const float* s, const float* z,
                                long long count, int group, long long row_len, double* out, cudaStream_t st) {
  PlaneGeom geo{count, group, row_len};
  plane_decode_kernel<<<blocks_for(count, 256), 256, 0, st>>>(up, lo, s, z, geo, out);
  return cudaGetLastError();
}

cudaError_t launch_quantize_weights(const float* w, int d_in, int d_out, int group, uint8_t* ref, float* s,
                                    float* z, uint32_t* frag4, float4* fparams, int* flags, cudaStream_t st) {
  int g = group < d_in ? group : d_in;
  WGeom geo{d_in, d_out, g, (d_in + g - 1) / g};
  long long ng = (long long)d_out * geo.gpr;
  wq_params_kernel<<<blocks_for(ng, 8), 256, 0, st>>>(w, geo, s, z, flags);
  if (ref) wq_refcodes_kernel<<<blocks_for(((long long)d_in * d_out + 1) / 2, 256), 256, 0, st>>>(w, geo, s, z, ref);
  if (frag4) {
    int ks = d_in / 16, ks_pad = (ks + 3) / 4 * 4;
    long long nwords = (long long)((d_out / 16 + 1) / 2 * 2) * ks_pad * 32;
    wq_frag_kernel<<<blocks_for(nwords, 256), 256, 0, st>>>(w, geo, s, z, frag4, ks_pad);
  }
  if (fparams) {
    long long tot = (long long)((d_out / 16 + 1) / 2 * 2) * geo.gpr * 8;
    wq_fragparams_kernel<<<blocks_for(tot, 256), 256, 0, st>>>(geo, s, z, fparams);
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_f16(const float* w, int d_in, int d_out, __half* out, cudaStream_t st) {
  long long total = (long long)((d_out / 16 + 1) / 2 * 2) * (d_in / 16) * 32;
  pack_f16_kernel<<<blocks_for(total, 256), 256, 0, st>>>(w, d_in, d_out, out);
  return cudaGetLastError();
}

static cudaError_t kq_configure(const void* kern, int smem, int& configured) {
  if (smem > 48 * 1024 && configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  return cudaSuccess;
}

cudaError_t launch_kv_quantize(const qs_kv_store& stt, int seq, int layer0, int nlayers, const __half* sk,
                               const __half* sv, long long layer_stride, long long head_stride, int nblk,
                               int dst_block, int* flags, cudaStream_t s) {
  KVQArgs a;
  a.st = stt;
  a.seq = seq;
  a.layer0 = layer0;
  a.dst_block0 = dst_block;
  a.src_k = sk;
  a.src_v = sv;
  a.src_layer_stride = layer_stride;
  a.src_head_stride = head_stride;
  a.flags = flags;
  const int smem = kq_smem(stt.G, stt.hd);
  static int configured = 0;
  cudaError_t e = kq_configure((const void*)kv_quant_kernel, smem, configured);
  if (e != cudaSuccess) return e;
  dim3 grid(nblk, stt.Hkv, nlayers);
  kv_quant_kernel<<<grid, KQ_THREADS, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_kv_flush(const qs_kv_store& st, int* n_blocks, int* fp1_len, int* fp2_len, int* flags,
                            cudaStream_t s) {
  FlushArgs a;
  a.st = st;
  a.n_blocks = n_blocks;
  a.fp1_len = fp1_len;
  a.fp2_len = fp2_len;
  a.n_blocks_w = n_blocks;
  a.fp2_len_w = fp2_len;
  a.flags = flags;
  const int smem = kq_smem(st.G, st.hd);
  static int configured = 0;
  cudaError_t e = kq_configure((const void*)kv_flush_quant_kernel, smem, configured);
  if (e != cudaSuccess) return e;
  dim3 grid(st.Hkv, st.L, st.B);
  e = launch_pdl(kv_flush_quant_kernel, grid, dim3(KQ_THREADS), smem, s, a);
  if (e != cudaSuccess) return e;
  e = launch_pdl(kv_flush_rotate_kernel, grid, dim3(256), 0, s, a);
  if (e != cudaSuccess) return e;
  return launch_pdl(kv_flush_lengths_kernel, dim3(1), dim3(32), 0, s, a);
}

cudaError_t launch_kv_dequant(const qs_kv_store& st, int seq, int layer, int nblk, int target, float* ok,
                              float* ov, cudaStream_t s) {
  if (nblk <= 0) return cudaSuccess;
  dim3 grid(nblk, st.Hkv);
  kv_dequant_kernel<<<grid, 256, 0, s>>>(st, seq, layer, target, ok, ov);
  return cudaGetLastError();
}

}  // namespace qs
