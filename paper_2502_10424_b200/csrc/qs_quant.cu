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

// params, tile-pair major: float4 per [pair][group][2 tiles][g] (zeros for a padding tile)
__global__ void wq_fragparams_kernel(WGeom geo, const float* __restrict__ s, const float* __restrict__ z,
                                     float4* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int MT = geo.d_out / 16, MT2 = (MT + 1) / 2 * 2;
  long long total = (long long)MT2 * geo.gpr * 8;
  if (i >= total) return;
  int g = (int)(i & 7);
  long long rest = i >> 3;
  int wt = (int)(rest & 1);
  rest >>= 1;
  int grp = (int)(rest % geo.gpr);
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
// KV block quantisation into the store (Q/cache.py:283-303)
// grid: x = block, y = kv head, z = layer offset.  128 threads.
// ---------------------------------------------------------------------------
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

__global__ void __launch_bounds__(128) kv_quant_kernel(const __grid_constant__ KVQArgs A) {
  extern __shared__ __align__(16) uint8_t sm[];
  const qs_kv_store& st = A.st;
  const int G = st.G, HD = st.hd, H = st.Hkv;
  const int kv = H * HD;
  const int b = blockIdx.x, h = blockIdx.y, layer = A.layer0 + blockIdx.z;
  const int tid = threadIdx.x;
  const __half* sk = A.src_k + (size_t)blockIdx.z * A.src_layer_stride;
  const __half* sv = A.src_v + (size_t)blockIdx.z * A.src_layer_stride;
  const int row0 = b * G;
  const int dblk = A.dst_block0 + b;

  if (layer_sensitive(st, layer)) {
    // sensitive layers archive fp rows instead of quantising (Q/cache.py:286-289)
    int slot = sens_slot(st, layer);
    int nsens = 0;
    for (int i = 0; i < st.L; ++i) nsens += layer_sensitive(st, i) ? 1 : 0;
    size_t cap = (size_t)st.max_blocks * G;
    size_t base = ((((size_t)A.seq * nsens + slot) * H + h) * cap + (size_t)dblk * G) * HD;
    __half* ak = reinterpret_cast<__half*>(st.arch_k) + base;
    __half* av = reinterpret_cast<__half*>(st.arch_v) + base;
    for (int i = tid; i < G * HD; i += blockDim.x) {
      int r = i / HD, c = i % HD;
      ak[i] = sk[(size_t)h * A.src_head_stride + (size_t)(row0 + r) * HD + c];
      av[i] = sv[(size_t)h * A.src_head_stride + (size_t)(row0 + r) * HD + c];
    }
    return;
  }

  uint8_t* cku = sm;             // [G][HD] codes
  uint8_t* ckl = cku + G * HD;
  uint8_t* cvu = ckl + G * HD;
  uint8_t* cvl = cvu + G * HD;
  bool bad = false;

  const size_t slh = ((size_t)A.seq * st.L + layer) * H + h;  // (seq, layer, head)
  float2* kp = reinterpret_cast<float2*>(st.kp) + (slh * st.max_blocks + dblk) * HD;
  float2* vp = reinterpret_cast<float2*>(st.vp) + (slh * st.max_blocks + dblk) * G;

  // keys: one group per channel over the block's G tokens
  for (int c = tid; c < HD; c += blockDim.x) {
    const __half* col = sk + (size_t)h * A.src_head_stride + (size_t)row0 * HD + c;
    double mn = INFINITY, mx = -INFINITY;
    for (int r = 0; r < G; ++r) {
      double x = (double)__half2float(col[(size_t)r * HD]);
      bad |= !finite_d(x);
      mn = fmin(mn, x);
      mx = fmax(mx, x);
    }
    UParams p = asym_params(mn, mx);
    kp[c] = make_float2(p.s, p.z);
    for (int r = 0; r < G; ++r) {
      double x = (double)__half2float(col[(size_t)r * HD]);
      int cu = code_upper(x, p);
      int cl = code_lower(x, cu, p);
      cku[r * HD + c] = (uint8_t)cu;
      ckl[r * HD + c] = (uint8_t)(cl + 8);
    }
  }
  // values: per token, groups of G channels inside the token (row_len = kv_dim)
  const int cg0 = ((h * HD) / G) * G;          // first channel of this head's value group
  const int cg1 = min(cg0 + G, kv);
  for (int r = tid; r < G; r += blockDim.x) {
    double mn = INFINITY, mx = -INFINITY;
    for (int c = cg0; c < cg1; ++c) {
      int hh = c / HD, cc = c % HD;
      double x = (double)__half2float(sv[(size_t)hh * A.src_head_stride + (size_t)(row0 + r) * HD + cc]);
      bad |= !finite_d(x);
      mn = fmin(mn, x);
      mx = fmax(mx, x);
    }
    UParams p = asym_params(mn, mx);
    vp[r] = make_float2(p.s, p.z);
    for (int c = 0; c < HD; ++c) {
      double x = (double)__half2float(sv[(size_t)h * A.src_head_stride + (size_t)(row0 + r) * HD + c]);
      int cu = code_upper(x, p);
      int cl = code_lower(x, cu, p);
      cvu[r * HD + c] = (uint8_t)cu;
      cvl[r * HD + c] = (uint8_t)(cl + 8);
    }
  }
  if (__syncthreads_or(bad) && tid == 0 && A.flags) atomicOr(A.flags, 1);

  // assemble frag4 words
  const int NI = HD / 16;
  const int nwords = G * HD / 8;
  const size_t pb = (size_t)G * HD / 2;
  const size_t poff = (slh * st.max_blocks + dblk) * pb;
  uint32_t* oku = reinterpret_cast<uint32_t*>(st.ku + poff);
  uint32_t* okl = reinterpret_cast<uint32_t*>(st.kl + poff);
  uint32_t* ovu = reinterpret_cast<uint32_t*>(st.vu + poff);
  uint32_t* ovl = reinterpret_cast<uint32_t*>(st.vl + poff);
  const int vec = qs_vec(NI);
  for (int wi = tid; wi < nwords; wi += blockDim.x) {
    int vp4 = wi % vec;
    int rest = wi / vec;
    int lane = rest % 32;
    int rest2 = rest / 32;
    int inner = (rest2 % (NI / vec)) * vec + vp4;
    int outer = rest2 / (NI / vec);
    int g = lane >> 2, t = lane & 3;
    uint32_t wku = 0, wkl = 0, wvu = 0, wvl = 0;
#pragma unroll
    for (int p = 0; p < 8; ++p) {
      int j = p & 3, hb = p >> 2;
      int row = g + 8 * (j & 1), col = 2 * t + 8 * (j >> 1) + hb;
      // keys: outer = token tile, inner = channel tile; A[token][channel]
      int tk = outer * 16 + row, ck = inner * 16 + col;
      wku |= (uint32_t)cku[tk * HD + ck] << (4 * p);
      wkl |= (uint32_t)ckl[tk * HD + ck] << (4 * p);
      // values: outer = token tile, inner = channel tile; A[channel][token]
      int tv = outer * 16 + col, cv = inner * 16 + row;
      wvu |= (uint32_t)cvu[tv * HD + cv] << (4 * p);
      wvl |= (uint32_t)cvl[tv * HD + cv] << (4 * p);
    }
    oku[wi] = wku;
    okl[wi] = wkl;
    ovu[wi] = wvu;
    ovl[wi] = wvl;
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

// fp1 <- fp2 for every layer of one sequence (the rotation of Q/cache.py:263-264)
__global__ void fp_rotate_kernel(__half* fk, __half* fv, size_t seq_off, int L, size_t buf_elems) {
  size_t n = (size_t)L * buf_elems / 8;  // uint4 = 8 halves
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    size_t l = i / (buf_elems / 8), j = i % (buf_elems / 8);
    size_t base = seq_off + l * 2 * buf_elems;
    uint4* k1 = reinterpret_cast<uint4*>(fk + base);
    const uint4* k2 = reinterpret_cast<const uint4*>(fk + base + buf_elems);
    uint4* v1 = reinterpret_cast<uint4*>(fv + base);
    const uint4* v2 = reinterpret_cast<const uint4*>(fv + base + buf_elems);
    k1[j] = k2[j];
    v1[j] = v2[j];
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
  int smem = 4 * stt.G * stt.hd;
  static int configured = 0;
  if (smem > 48 * 1024 && configured < smem) {
    cudaError_t e = cudaFuncSetAttribute(kv_quant_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    configured = smem;
  }
  dim3 grid(nblk, stt.Hkv, nlayers);
  kv_quant_kernel<<<grid, 128, smem, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_kv_dequant(const qs_kv_store& st, int seq, int layer, int nblk, int target, float* ok,
                              float* ov, cudaStream_t s) {
  if (nblk <= 0) return cudaSuccess;
  dim3 grid(nblk, st.Hkv);
  kv_dequant_kernel<<<grid, 256, 0, s>>>(st, seq, layer, target, ok, ov);
  return cudaGetLastError();
}

cudaError_t launch_fp_rotate(const qs_kv_store& st, int seq, cudaStream_t s) {
  size_t buf = (size_t)st.Hkv * st.G * st.hd;
  size_t seq_off = (size_t)seq * st.L * 2 * buf;
  size_t n = (size_t)st.L * buf / 8;
  unsigned nb = (unsigned)((n + 255) / 256);
  if (nb > 4096) nb = 4096;
  fp_rotate_kernel<<<nb, 256, 0, s>>>(reinterpret_cast<__half*>(st.fp_k), reinterpret_cast<__half*>(st.fp_v),
                                      seq_off, st.L, buf);
  return cudaGetLastError();
}

}  // namespace qs
