// Split-K flash-decoding attention over the hierarchical KV store (sm_100a).
//
// Replaces, for one layer and all query rows of a forward:
//   HierarchicalKVCache.draft_view/target_view (+ the f32 memo copies)
//     /root/reference/pkg/src/quantspec/cache.py:309-378
//   _merged_attention (running max / denom / acc merge across segments)
//     /root/reference/pkg/src/quantspec/model.py:176-195
//   the gamma+1 *sequential* target decode_steps of verify_phase
//     /root/reference/pkg/src/quantspec/specdec.py:270-273 (here: T queries at once)
//
// Grid: x = main-region splits + 2 tail splits (fp1, fp2), y = kv_head * qgroups, z = seq.
// Every CTA (4 warps) streams its chunks through a multi-stage shared-memory
// pipeline (TMA bulk copies for the packed planes, cp.async for fp16 rows),
// dequantises in registers straight into f16 MMA fragments (swap-AB: tokens
// or channels on M, query columns hi/lo on N), keeps a per-warp online softmax
// with lazy rescaling, then merges warps and splits in a fixed order (last CTA
// of a head reduces), so results are independent of how many query rows ride
// in the launch (greedy losslessness needs that).
#include "qs_common.cuh"
#include "qs_layout.h"
#include "qs_api_internal.h"

namespace qs {

enum { MODE_QDRAFT = 0, MODE_QTARGET = 1, MODE_FP16 = 2 };

constexpr int kThreads = 128;
#define kNegInf (-__int_as_float(0x7f800000))
constexpr float kLazy = 0.0f;  // rescale whenever the running max grows (p <= 1 keeps p*S in f16 range)

template <int HD, int NT, int MODE>
struct AttnCfg {
  static constexpr int KS = HD / 16;                       // channel tiles
  static constexpr int VEC = KS >= 4 ? 4 : KS;
  static constexpr int PLANE_CHUNK = HD * QS_CHUNK_Q / 2;  // bytes of one plane per 128-token chunk
  static constexpr int NPLANE = (MODE == MODE_QTARGET) ? 4 : 2;
  // quant stage: planes + key params + value params (128 tokens).  Valid
  // layouts have G >= HD, so a chunk holds (128/G)*HD <= 128 key channels-blocks.
  static constexpr int KP_BYTES = QS_CHUNK_Q * 8;
  static constexpr int QSTAGE = NPLANE * PLANE_CHUNK + KP_BYTES + QS_CHUNK_Q * 8;
  static constexpr int NSTAGE_Q = (MODE == MODE_QTARGET) ? 3 : 4;
  static constexpr int FSTAGE = 2 * QS_CHUNK_F * HD * 2;  // K + V fp16 rows
  static constexpr int NSTAGE_F = 2;
  static constexpr int REGION_Q = (MODE == MODE_FP16) ? 0 : NSTAGE_Q * QSTAGE;
  static constexpr int REGION_F = NSTAGE_F * FSTAGE;
  static constexpr int REGION = REGION_Q > REGION_F ? REGION_Q : REGION_F;
  static constexpr int NQ = NT * 4;                        // query columns (hi/lo pairs) per CTA
  static constexpr int BQ_WORDS = 8 * NT * 32 * 2;         // u32 per Bq buffer: (128/G)*KS <= 8 tiles
  static constexpr int PW_HALVES = 2 * NT * 8 * 16;        // per-warp P transpose tile
  // merge scratch reuses REGION: 4 warps * NQ * (HD + 4) floats
  static constexpr int MERGE_FLOATS = 4 * NQ * (HD + 4);
  static_assert(MERGE_FLOATS * 4 <= REGION, "merge scratch must fit in the stage region");
  static constexpr int SMEM =
      REGION + 2 * BQ_WORDS * 4 + 2 * 8 * NQ * 4 + NQ * HD * 4 + 4 * PW_HALVES * 2 + 8 * 8 + 16;
};

__device__ __forceinline__ int swz16(int chunk, int row, int nchunk) {
  return nchunk >= 8 ? (chunk ^ (row & 7)) : chunk;
}

template <int NI>
__device__ __forceinline__ void load_words(const uint32_t* base, int outer, int lane, uint32_t (&w)[NI]) {
  constexpr int VEC = NI >= 4 ? 4 : NI;
#pragma unroll
  for (int v = 0; v < NI / VEC; ++v) {
    const uint32_t* p = base + ((outer * (NI / VEC) + v) * 32 + lane) * VEC;
    if constexpr (VEC == 4) {
      uint4 u = *reinterpret_cast<const uint4*>(p);
      w[v * 4 + 0] = u.x; w[v * 4 + 1] = u.y; w[v * 4 + 2] = u.z; w[v * 4 + 3] = u.w;
    } else if constexpr (VEC == 2) {
      uint2 u = *reinterpret_cast<const uint2*>(p);
      w[v * 2 + 0] = u.x; w[v * 2 + 1] = u.y;
    } else {
      w[v] = p[0];
    }
  }
}

struct Softmax {
  float m, l, z;
};

// per-warp online softmax update for one query column owned by this lane.
// s[] holds NS scores (log2 domain, -inf = masked).  Returns the rescale
// factor applied to the running accumulators (1 when unchanged).
template <int NS>
__device__ __forceinline__ float softmax_update(Softmax& st, float (&s)[NS], float (&p)[NS]) {
  float mx = kNegInf;
#pragma unroll
  for (int i = 0; i < NS; ++i) mx = fmaxf(mx, s[i]);
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  float alpha = 1.0f;
  if (mx > st.m + kLazy) {
    alpha = exp2f(st.m - mx);  // st.m == -inf -> 0
    st.l *= alpha;
    st.z *= alpha;
    st.m = mx;
  }
#pragma unroll
  for (int i = 0; i < NS; ++i) p[i] = (s[i] == kNegInf) ? 0.0f : exp2f(s[i] - st.m);
  return alpha;
}

template <int HD, int NT, int MODE>
__global__ void __launch_bounds__(kThreads) attn_kernel(const __grid_constant__ AttnParams P) {
  using C = AttnCfg<HD, NT, MODE>;
  constexpr int KS = C::KS;
  constexpr int NQ = C::NQ;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* region = smem;
  uint32_t* bq = reinterpret_cast<uint32_t*>(smem + C::REGION);              // [2][BQ_WORDS]
  float* bias_s = reinterpret_cast<float*>(bq + 2 * C::BQ_WORDS);            // [2][8][NQ]
  float* q_s = bias_s + 2 * 8 * NQ;                                          // [NQ][HD]
  __half* pw_all = reinterpret_cast<__half*>(q_s + NQ * HD);                  // [4][PW_HALVES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(pw_all + 4 * C::PW_HALVES);   // [8]
  int* ticket_s = reinterpret_cast<int*>(bars + 8);

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int seq = blockIdx.z;
  const int head = blockIdx.y / P.n_qgroups, qg = blockIdx.y % P.n_qgroups;
  const int split = blockIdx.x;
  const int n_main = P.n_main;
  const int n_split_tot = n_main + 2;
  const int nq = min(NQ, P.n_queries - qg * NQ);  // real query columns in this CTA
  __half* pw = pw_all + warp * C::PW_HALVES;

  // ---- queries of this CTA (column q -> (t, j) with q_global = qg*NQ + q) ----
  for (int i = tid; i < NQ * HD; i += kThreads) {
    int q = i / HD, c = i % HD;
    float v = 0.f;
    if (q < nq) {
      int qgl = qg * NQ + q;
      int t = qgl / P.r, j = qgl % P.r;
      v = P.q[((size_t)seq * P.T + t) * P.q_row_stride + (size_t)(head * P.r + j) * HD + c];
    }
    q_s[i] = v;
  }
  for (int i = tid; i < 2 * C::BQ_WORDS; i += kThreads) bq[i] = 0u;
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) mbar_init(&bars[i], 1);
    fence_mbar_init();
  }
  __syncthreads();

  // ---- which region does this CTA own? ----
  const int fp1_len = P.fp1_len ? P.fp1_len[seq] : 0;
  const int fp2_base = P.fp2_len ? P.fp2_len[seq] + P.row_offset : 0;
  int region_kind;  // 0 quant, 1 fp16 main, 2 fp1, 3 fp2
  int n_tok = 0, c_begin = 0, c_end = 0, causal = 0;
  const __half* fk = nullptr;
  const __half* fv = nullptr;
  if (split < n_main) {
    if (MODE == MODE_FP16) {
      region_kind = 1;
      if (P.main_is_fpcache) {
        n_tok = P.fp_len[seq] + P.row_offset + P.T;
        causal = 1;
      } else {
        n_tok = P.n_blocks[seq] * P.G;
      }
      int nch = (n_tok + QS_CHUNK_F - 1) / QS_CHUNK_F;
      int cps = P.main_is_fpcache ? P.fpcache_cps : (nch + n_main - 1) / n_main;
      c_begin = split * cps;
      c_end = min(nch, c_begin + cps);
      size_t hoff = ((size_t)seq * P.main_seq_stride + (size_t)head * P.main_head_stride);
      fk = reinterpret_cast<const __half*>(P.main_k) + hoff;
      fv = reinterpret_cast<const __half*>(P.main_v) + hoff;
    } else {
      region_kind = 0;
      n_tok = P.n_blocks[seq] * P.G;
      int nch = (n_tok + QS_CHUNK_Q - 1) / QS_CHUNK_Q;
      int cps = (nch + n_main - 1) / n_main;
      c_begin = split * cps;
      c_end = min(nch, c_begin + cps);
    }
  } else if (split == n_main) {
    region_kind = 2;
    n_tok = fp1_len;
    c_begin = 0;
    c_end = (n_tok + QS_CHUNK_F - 1) / QS_CHUNK_F;
    size_t hoff = (size_t)seq * P.fp_seq_stride + (size_t)head * P.G * HD;
    fk = P.fp1_k ? reinterpret_cast<const __half*>(P.fp1_k) + hoff : nullptr;
    fv = P.fp1_v ? reinterpret_cast<const __half*>(P.fp1_v) + hoff : nullptr;
    if (!fk) c_end = 0;
  } else {
    region_kind = 3;
    n_tok = fp2_base + P.T;
    causal = 1;
    c_begin = 0;
    c_end = (n_tok + QS_CHUNK_F - 1) / QS_CHUNK_F;
    size_t hoff = (size_t)seq * P.fp_seq_stride + (size_t)head * P.G * HD;
    fk = P.fp2_k ? reinterpret_cast<const __half*>(P.fp2_k) + hoff : nullptr;
    fv = P.fp2_v ? reinterpret_cast<const __half*>(P.fp2_v) + hoff : nullptr;
    if (!fk) c_end = 0;
  }

  // per-lane softmax state for query columns nt*4 + t4
  Softmax st[NT];
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) st[nt] = {kNegInf, 0.f, 0.f};
  float acc[KS][NT][4];
#pragma unroll
  for (int a = 0; a < KS; ++a)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[a][nt][e] = 0.f;

  const float sl2 = P.sm_scale_log2;

  // visible-token limit for query column q (causal tail): tokens j < lim
  auto vis_limit = [&](int q) -> int {
    if (!causal) return n_tok;
    int qgl = qg * NQ + q;
    int t = min(qgl / P.r, P.T - 1);
    return n_tok - (P.T - 1 - t);
  };

  if (region_kind == 0 && c_end > c_begin) {
    // ===================== quantised chunks =====================
    if constexpr (MODE != MODE_FP16) {
      const int G = P.G;
      const int bpc = QS_CHUNK_Q / G;  // blocks per chunk
      const int n_blocks = P.n_blocks[seq];
      const size_t plane_blk = (size_t)G * HD / 2;
      const size_t ph = ((size_t)seq * P.plane_seq_stride) + (size_t)head * P.plane_head_stride;
      const uint8_t* ku = P.ku + ph;
      const uint8_t* vu = P.vu + ph;
      const uint8_t* kl = (MODE == MODE_QTARGET) ? P.kl + ph : nullptr;
      const uint8_t* vl = (MODE == MODE_QTARGET) ? P.vl + ph : nullptr;
      const float2* kp = reinterpret_cast<const float2*>(P.kp) + (size_t)seq * P.kp_seq_stride + (size_t)head * P.kp_head_stride;
      const float2* vp = reinterpret_cast<const float2*>(P.vp) + (size_t)seq * P.vp_seq_stride + (size_t)head * P.vp_head_stride;
      const int nchunk = c_end - c_begin;

      auto stage_ptr = [&](int s) { return region + s * C::QSTAGE; };
      auto issue = [&](int i) {
        int c = c_begin + i;
        int s = i % C::NSTAGE_Q;
        uint8_t* sp = stage_ptr(s);
        int b0 = c * bpc;
        int nb = min(bpc, n_blocks - b0);
        uint32_t pbytes = (uint32_t)(nb * plane_blk);
        uint32_t kpb = (uint32_t)(nb * HD * 8), vpb = (uint32_t)(nb * G * 8);
        uint32_t total = pbytes * C::NPLANE + kpb + vpb;
        mbar_arrive_expect_tx(&bars[s], total);
        bulk_g2s(sp, ku + b0 * plane_blk, pbytes, &bars[s]);
        bulk_g2s(sp + C::PLANE_CHUNK, vu + b0 * plane_blk, pbytes, &bars[s]);
        if constexpr (MODE == MODE_QTARGET) {
          bulk_g2s(sp + 2 * C::PLANE_CHUNK, kl + b0 * plane_blk, pbytes, &bars[s]);
          bulk_g2s(sp + 3 * C::PLANE_CHUNK, vl + b0 * plane_blk, pbytes, &bars[s]);
        }
        bulk_g2s(sp + C::NPLANE * C::PLANE_CHUNK, kp + (size_t)b0 * HD, kpb, &bars[s]);
        bulk_g2s(sp + C::NPLANE * C::PLANE_CHUNK + C::KP_BYTES, vp + (size_t)b0 * G, vpb, &bars[s]);
      };
      if (tid == 0) {
        for (int i = 0; i < C::NSTAGE_Q - 1 && i < nchunk; ++i) issue(i);
      }
      for (int i = 0; i < nchunk; ++i) {
        const int stg = i % C::NSTAGE_Q;
        uint8_t* sp = stage_ptr(stg);
        mbar_wait(&bars[stg], (i / C::NSTAGE_Q) & 1);
        const int c = c_begin + i;
        const int ntok_chunk = min(QS_CHUNK_Q, n_tok - c * QS_CHUNK_Q);
        const int nbl = (ntok_chunk + G - 1) / G;
        const float2* kps = reinterpret_cast<const float2*>(sp + C::NPLANE * C::PLANE_CHUNK);
        const float2* vps = reinterpret_cast<const float2*>(sp + C::NPLANE * C::PLANE_CHUNK + C::KP_BYTES);
        uint32_t* bqb = bq + (i & 1) * C::BQ_WORDS;
        float* bsb = bias_s + (i & 1) * 8 * NQ;
        // --- fold key scales into the queries: q'_c = q_c * S_c (/16 for target) ---
        for (int idx = tid; idx < nbl * (HD / 2) * nq; idx += kThreads) {
          int q = idx % nq;
          int cp = (idx / nq) % (HD / 2);
          int bl = idx / (nq * (HD / 2));
          float2 p0 = kps[bl * HD + 2 * cp], p1 = kps[bl * HD + 2 * cp + 1];
          float s0 = p0.x, s1 = p1.x;
          if (MODE == MODE_QTARGET) { s0 *= 0.0625f; s1 *= 0.0625f; }
          float v0 = q_s[q * HD + 2 * cp] * s0, v1 = q_s[q * HD + 2 * cp + 1] * s1;
          __half h0, l0, h1, l1;
          split_hl(v0, h0, l0);
          split_hl(v1, h1, l1);
          int ks = cp >> 3, j = cp & 7;
          int tt = j & 3, which = j >> 2;
          int col_hi = 2 * q, col_lo = 2 * q + 1;
          int nt = col_hi >> 3;
          int gh = col_hi & 7, gl = col_lo & 7;
          size_t base = ((size_t)(bl * KS + ks) * NT + nt) * 32;
          bqb[(base + gh * 4 + tt) * 2 + which] = h2_as_u32(__halves2half2(h0, h1));
          bqb[(base + gl * 4 + tt) * 2 + which] = h2_as_u32(__halves2half2(l0, l1));
        }
        // --- per-block bias sum_c q_c * Z_c ---
        for (int pr = warp; pr < nbl * nq; pr += 4) {
          int bl = pr / nq, q = pr % nq;
          float a = 0.f;
          for (int cc = lane; cc < HD; cc += 32) a += q_s[q * HD + cc] * kps[bl * HD + cc].y;
          a = warp_sum(a);
          if (lane == 0) bsb[bl * NQ + q] = a;
        }
        __syncthreads();
        if (tid == 0 && i + C::NSTAGE_Q - 1 < nchunk) issue(i + C::NSTAGE_Q - 1);

        // --- this warp: m-tiles warp and warp+4 (32 tokens) ---
        const uint32_t* kuw = reinterpret_cast<const uint32_t*>(sp);
        const uint32_t* vuw = reinterpret_cast<const uint32_t*>(sp + C::PLANE_CHUNK);
        const uint32_t* klw = reinterpret_cast<const uint32_t*>(sp + 2 * C::PLANE_CHUNK);
        const uint32_t* vlw = reinterpret_cast<const uint32_t*>(sp + 3 * C::PLANE_CHUNK);
        float s[NT][4];  // [nt][mi*2 + (g | g+8)]
        bool live[2];
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          const int mt = warp + 4 * mi;
          live[mi] = mt * 16 < ntok_chunk;
          float d[NT][4];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) d[nt][e] = 0.f;
          const int bl = (mt * 16) / G;
          if (live[mi]) {
            uint32_t wu[KS];
            load_words<KS>(kuw, mt, lane, wu);
            uint32_t wl[KS];
            if constexpr (MODE == MODE_QTARGET) load_words<KS>(klw, mt, lane, wl);
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
              uint32_t a[4];
              if constexpr (MODE == MODE_QTARGET) unpack_u4l4(wu[ks], wl[ks], a);
              else unpack_u4(wu[ks], a);
#pragma unroll
              for (int nt = 0; nt < NT; ++nt) {
                uint2 b = *reinterpret_cast<const uint2*>(bqb + (((size_t)(bl * KS + ks) * NT + nt) * 32 + lane) * 2);
                mma16816(d[nt], a, b.x, b.y);
              }
            }
          }
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const int q = nt * 4 + t4;
            const float bias = (q < nq) ? bsb[bl * NQ + q] : 0.f;
            const int lim = vis_limit(q);
            int tok0 = c * QS_CHUNK_Q + mt * 16 + g;
            float v0 = (d[nt][0] + d[nt][1] + bias) * sl2;
            float v1 = (d[nt][2] + d[nt][3] + bias) * sl2;
            s[nt][mi * 2 + 0] = (live[mi] && tok0 < lim) ? v0 : kNegInf;
            s[nt][mi * 2 + 1] = (live[mi] && tok0 + 8 < lim) ? v1 : kNegInf;
          }
        }
        // --- online softmax, value-scale fold, P transpose ---
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float p[4];
          float alpha = softmax_update<4>(st[nt], s[nt], p);
          if (alpha != 1.0f) {
#pragma unroll
            for (int a = 0; a < KS; ++a) {
              acc[a][nt][0] *= alpha; acc[a][nt][1] *= alpha;
              acc[a][nt][2] *= alpha; acc[a][nt][3] *= alpha;
            }
          }
#pragma unroll
          for (int mi = 0; mi < 2; ++mi) {
            const int mt = warp + 4 * mi;
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
              const int tl = mt * 16 + g + 8 * hh;  // token within chunk
              float pv = p[mi * 2 + hh];
              float2 sz = live[mi] ? vps[tl] : make_float2(0.f, 0.f);
              st[nt].l += pv;
              st[nt].z += pv * sz.y;
              float ps = pv * sz.x * ((MODE == MODE_QTARGET) ? 0.0625f : 1.0f);
              __half hi, lo;
              split_hl(ps, hi, lo);
              pw[(mi * NT * 8 + nt * 8 + 2 * t4) * 16 + g + 8 * hh] = hi;
              pw[(mi * NT * 8 + nt * 8 + 2 * t4 + 1) * 16 + g + 8 * hh] = lo;
            }
          }
        }
        __syncwarp();
        // --- PV: A = V^T (channels x tokens) from the value planes ---
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
          if (!live[mi]) continue;
          const int mt = warp + 4 * mi;
          uint32_t bpv[NT][2];
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            const __half* row = pw + (mi * NT * 8 + nt * 8 + g) * 16;
            bpv[nt][0] = *reinterpret_cast<const uint32_t*>(row + 2 * t4);
            bpv[nt][1] = *reinterpret_cast<const uint32_t*>(row + 2 * t4 + 8);
          }
          uint32_t wu[KS];
          load_words<KS>(vuw, mt, lane, wu);
          uint32_t wl[KS];
          if constexpr (MODE == MODE_QTARGET) load_words<KS>(vlw, mt, lane, wl);
#pragma unroll
          for (int cm = 0; cm < KS; ++cm) {
            uint32_t a[4];
            if constexpr (MODE == MODE_QTARGET) unpack_u4l4(wu[cm], wl[cm], a);
            else unpack_u4(wu[cm], a);
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) mma16816(acc[cm][nt], a, bpv[nt][0], bpv[nt][1]);
          }
        }
        __syncwarp();
      }
    }
  } else if (region_kind >= 1 && c_end > c_begin) {
    // ===================== fp16 chunks (fp1 / fp2 / archive / fp cache) =====================
    // B fragments for the raw queries (no per-block scale): built once.
    uint32_t* bqf = bq;  // [KS][NT][32][2]
    for (int idx = tid; idx < (HD / 2) * nq; idx += kThreads) {
      int q = idx % nq, cp = idx / nq;
      __half h0, l0, h1, l1;
      split_hl(q_s[q * HD + 2 * cp], h0, l0);
      split_hl(q_s[q * HD + 2 * cp + 1], h1, l1);
      int ks = cp >> 3, j = cp & 7, tt = j & 3, which = j >> 2;
      int col_hi = 2 * q, col_lo = 2 * q + 1, nt = col_hi >> 3;
      size_t base = ((size_t)ks * NT + nt) * 32;
      bqf[(base + (col_hi & 7) * 4 + tt) * 2 + which] = h2_as_u32(__halves2half2(h0, h1));
      bqf[(base + (col_lo & 7) * 4 + tt) * 2 + which] = h2_as_u32(__halves2half2(l0, l1));
    }
    const int nchunk = c_end - c_begin;
    constexpr int NCH16 = HD / 8;  // 16-byte chunks per row
    auto fstage = [&](int s) { return reinterpret_cast<__half*>(region + s * C::FSTAGE); };
    auto issue_f = [&](int i) {
      if (i < nchunk) {
        int c = c_begin + i;
        __half* ks_ = fstage(i % C::NSTAGE_F);
        __half* vs_ = ks_ + QS_CHUNK_F * HD;
        for (int idx = tid; idx < QS_CHUNK_F * NCH16; idx += kThreads) {
          int row = idx / NCH16, ch = idx % NCH16;
          int tok = c * QS_CHUNK_F + row;
          bool ok = tok < n_tok;
          int tk = ok ? tok : 0;
          int pc = swz16(ch, row, NCH16);
          cp_async16(smem_u32(ks_ + row * HD + pc * 8), fk + (size_t)tk * HD + ch * 8, ok);
          cp_async16(smem_u32(vs_ + row * HD + pc * 8), fv + (size_t)tk * HD + ch * 8, ok);
        }
      }
      cp_async_commit();
    };
    for (int i = 0; i < C::NSTAGE_F - 1; ++i) issue_f(i);
    for (int i = 0; i < nchunk; ++i) {
      cp_async_wait<C::NSTAGE_F - 2>();
      __syncthreads();
      issue_f(i + C::NSTAGE_F - 1);
      const int c = c_begin + i;
      const __half* ks_ = fstage(i % C::NSTAGE_F);
      const __half* vs_ = ks_ + QS_CHUNK_F * HD;
      const int ntok_chunk = min(QS_CHUNK_F, n_tok - c * QS_CHUNK_F);
      const int mt = warp;  // one 16-token tile per warp
      const bool live = mt * 16 < ntok_chunk;
      float d[NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) d[nt][e] = 0.f;
      if (live) {
        const int ii = lane >> 3, rr = lane & 7;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks) {
          int row = mt * 16 + (ii & 1) * 8 + rr;
          int ch = ks * 2 + (ii >> 1);
          uint32_t a[4];
          ldmatrix_x4(a, smem_u32(ks_ + row * HD + swz16(ch, row, NCH16) * 8));
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            uint2 b = *reinterpret_cast<const uint2*>(bqf + (((size_t)ks * NT + nt) * 32 + lane) * 2);
            mma16816(d[nt], a, b.x, b.y);
          }
        }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int q = nt * 4 + t4;
        const int lim = vis_limit(q);
        int tok0 = c * QS_CHUNK_F + mt * 16 + g;
        float sv[2], p[2];
        sv[0] = (live && tok0 < lim) ? (d[nt][0] + d[nt][1]) * sl2 : kNegInf;
        sv[1] = (live && tok0 + 8 < lim) ? (d[nt][2] + d[nt][3]) * sl2 : kNegInf;
        float alpha = softmax_update<2>(st[nt], sv, p);
        if (alpha != 1.0f) {
#pragma unroll
          for (int a = 0; a < KS; ++a) {
            acc[a][nt][0] *= alpha; acc[a][nt][1] *= alpha;
            acc[a][nt][2] *= alpha; acc[a][nt][3] *= alpha;
          }
        }
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          st[nt].l += p[hh];
          __half hi, lo;
          split_hl(p[hh], hi, lo);
          pw[(nt * 8 + 2 * t4) * 16 + g + 8 * hh] = hi;
          pw[(nt * 8 + 2 * t4 + 1) * 16 + g + 8 * hh] = lo;
        }
      }
      __syncwarp();
      if (live) {
        uint32_t bpv[NT][2];
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const __half* row = pw + (nt * 8 + g) * 16;
          bpv[nt][0] = *reinterpret_cast<const uint32_t*>(row + 2 * t4);
          bpv[nt][1] = *reinterpret_cast<const uint32_t*>(row + 2 * t4 + 8);
        }
        const int ii = lane >> 3, rr = lane & 7;
#pragma unroll
        for (int cm = 0; cm < KS; ++cm) {
          int row = mt * 16 + (ii >> 1) * 8 + rr;
          int ch = cm * 2 + (ii & 1);
          uint32_t a[4];
          ldmatrix_x4_trans(a, smem_u32(vs_ + row * HD + swz16(ch, row, NCH16) * 8));
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma16816(acc[cm][nt], a, bpv[nt][0], bpv[nt][1]);
        }
      }
      __syncwarp();
    }
    cp_async_wait<0>();
  }

  // ===================== merge the 4 warps of this CTA =====================
  __syncthreads();  // stage region is free for scratch now
  float* mrg = reinterpret_cast<float*>(region);  // [4][NQ][HD + 4]: m, l, acc...
  constexpr int MS = HD + 4;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    float l = st[nt].l, z = st[nt].z;
    l += __shfl_xor_sync(0xffffffffu, l, 4);
    l += __shfl_xor_sync(0xffffffffu, l, 8);
    l += __shfl_xor_sync(0xffffffffu, l, 16);
    z += __shfl_xor_sync(0xffffffffu, z, 4);
    z += __shfl_xor_sync(0xffffffffu, z, 8);
    z += __shfl_xor_sync(0xffffffffu, z, 16);
    const int q = nt * 4 + t4;
    float* row = mrg + (warp * NQ + q) * MS;
    if (g == 0) {
      row[0] = st[nt].m;
      row[1] = l;
    }
#pragma unroll
    for (int cm = 0; cm < KS; ++cm) {
      row[4 + cm * 16 + g] = acc[cm][nt][0] + acc[cm][nt][1] + z;
      row[4 + cm * 16 + g + 8] = acc[cm][nt][2] + acc[cm][nt][3] + z;
    }
  }
  __syncthreads();
  const size_t hidx = ((size_t)seq * P.Hkv + head) * P.n_qgroups + qg;
  float* part = P.partials + (hidx * n_split_tot + split) * (size_t)NQ * (HD + 2);
  for (int i = tid; i < NQ * (HD + 2); i += kThreads) {
    int q = i / (HD + 2), c = i % (HD + 2);
    float mx = kNegInf;
#pragma unroll
    for (int w = 0; w < 4; ++w) mx = fmaxf(mx, mrg[(w * NQ + q) * MS]);
    float v = 0.f;
    if (c == 0) {
      v = mx;
    } else if (mx != kNegInf) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float* row = mrg + (w * NQ + q) * MS;
        float f = exp2f(row[0] - mx);
        v += f * (c == 1 ? row[1] : row[4 + c - 2]);
      }
    }
    part[i] = v;
  }
  __threadfence();
  __syncthreads();
  if (tid == 0) *ticket_s = atomicAdd(&P.counters[hidx], 1);
  __syncthreads();
  if (*ticket_s != n_split_tot - 1) return;
  __threadfence();
  // ===================== last CTA: merge splits in fixed order =====================
  const float* allp = P.partials + hidx * n_split_tot * (size_t)NQ * (HD + 2);
  for (int i = tid; i < nq * HD; i += kThreads) {
    int q = i / HD, c = i % HD;
    float mx = kNegInf;
    for (int s = 0; s < n_split_tot; ++s) mx = fmaxf(mx, __ldcg(allp + ((size_t)s * NQ + q) * (HD + 2)));
    float num = 0.f, den = 0.f;
    if (mx != kNegInf) {
      for (int s = 0; s < n_split_tot; ++s) {
        const float* pr = allp + ((size_t)s * NQ + q) * (HD + 2);
        float m = __ldcg(pr);
        float f = exp2f(m - mx);
        den += f * __ldcg(pr + 1);
        num += f * __ldcg(pr + 2 + c);
      }
    }
    int qgl = qg * NQ + q;
    int t = qgl / P.r, j = qgl % P.r;
    P.out[((size_t)seq * P.T + t) * P.q_row_stride + (size_t)(head * P.r + j) * HD + c] = den > 0.f ? num / den : 0.f;
  }
  if (tid == 0) P.counters[hidx] = 0;
}

template <int HD, int NT, int MODE>
static cudaError_t launch_attn_t(const AttnParams& p, cudaStream_t stream) {
  using C = AttnCfg<HD, NT, MODE>;
  auto kern = attn_kernel<HD, NT, MODE>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.n_main + 2, p.Hkv * p.n_qgroups, p.B);
  kern<<<grid, kThreads, C::SMEM, stream>>>(p);
  return cudaGetLastError();
}

template <int HD, int MODE>
static cudaError_t launch_attn_nt(const AttnParams& p, int nt, cudaStream_t s) {
  switch (nt) {
    case 1: return launch_attn_t<HD, 1, MODE>(p, s);
    case 2: return launch_attn_t<HD, 2, MODE>(p, s);
    case 3: return launch_attn_t<HD, 3, MODE>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int MODE>
static cudaError_t launch_attn_hd(const AttnParams& p, int nt, cudaStream_t s) {
  switch (p.hd) {
    case 16: return launch_attn_nt<16, MODE>(p, nt, s);
    case 32: return launch_attn_nt<32, MODE>(p, nt, s);
    case 64: return launch_attn_nt<64, MODE>(p, nt, s);
    case 128: return launch_attn_nt<128, MODE>(p, nt, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attention(const AttnParams& p, int mode, cudaStream_t s) {
  // columns per CTA: NT*4 queries (each query uses a hi/lo column pair)
  int nt = (p.n_queries + p.n_qgroups - 1) / p.n_qgroups;
  nt = (nt + 3) / 4;
  if (nt < 1) nt = 1;
  switch (mode) {
    case MODE_QDRAFT: return launch_attn_hd<MODE_QDRAFT>(p, nt, s);
    case MODE_QTARGET: return launch_attn_hd<MODE_QTARGET>(p, nt, s);
    case MODE_FP16: return launch_attn_hd<MODE_FP16>(p, nt, s);
    default: return cudaErrorInvalidValue;
  }
}

int attention_smem_bytes(int hd, int nt, int mode) {
#define QS_SM(H, N, M) \
  if (hd == H && nt == N && mode == M) return AttnCfg<H, N, M>::SMEM;
#define QS_SM_M(M) QS_SM(16, 1, M) QS_SM(16, 2, M) QS_SM(16, 3, M) QS_SM(32, 1, M) QS_SM(32, 2, M) QS_SM(32, 3, M) \
  QS_SM(64, 1, M) QS_SM(64, 2, M) QS_SM(64, 3, M) QS_SM(128, 1, M) QS_SM(128, 2, M) QS_SM(128, 3, M)
  QS_SM_M(0) QS_SM_M(1) QS_SM_M(2)
#undef QS_SM_M
#undef QS_SM
  return -1;
}

}  // namespace qs
