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
// Grid: x = kv_head * qgroups, y = split (main-region splits, then the fp1
// and fp2 tail splits -- launched last so every main split is resident in
// the first wave), z = sequence.
//
// Quantised kernel (draft: upper plane; target: upper+lower): warp-specialised.
// One producer warp keeps NSTAGE 128-token chunks in flight with TMA bulk
// copies (packed code planes + f32 params) and, per chunk, folds the key
// scales into the queries (q'_c = q_c S_c as f16 hi/lo mma B fragments) and
// the zero points into a per-block score bias; eight consumer warps, one per
// 16-token tile, dequantise the packed nibbles in registers straight into f16
// mma.sync A fragments (swap-AB: tokens on M for Q.K^T, channels on M for
// P.V, query hi/lo columns on N).  The magic-number f16 offset of each code
// (1024, or 1024+16c for the high nibble) is never subtracted per element: it
// rides through the MMA and is removed by the per-block bias (Q.K^T) or a
// per-column probability sum (P.V, draft), so the unpack is 5 instructions per
// 8 codes.  Full/empty mbarriers replace block-wide barriers in the loop.
//
// Each consumer warp keeps its own online softmax; warps and then splits are
// merged in a fixed order (the last CTA of a head reduces), so one query row's
// result does not depend on how many rows share the launch (greedy
// losslessness needs a T-row verify to equal T single-row steps bit for bit).
#include "qs_common.cuh"
#include "qs_layout.h"
#include "qs_api_internal.h"

namespace qs {

enum { MODE_QDRAFT = 0, MODE_QTARGET = 1, MODE_FP16 = 2 };

#define kNegInf (-__int_as_float(0x7f800000))

// mma.sync without `volatile`: pure, so ptxas may interleave it with the nibble unpacking
__device__ __forceinline__ void mma_nv(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

constexpr int PSTRIDE = 24;
#ifndef QS_WAIT_SLEEP
#define QS_WAIT_SLEEP 0  // A/B builds: ring waits suspend in hardware (try_wait with a time hint) instead of spinning
#endif
__device__ __forceinline__ void attn_wait(uint64_t* bar, uint32_t parity) {
  if constexpr (QS_WAIT_SLEEP) mbar_wait_sleep(bar, parity);
  else mbar_wait(bar, parity);
}
#ifndef QS_LAZY_MAX_LOG2
#define QS_LAZY_MAX_LOG2 8  // draft online softmax: raise the reference max only past 2^8 (0: exact max every chunk)
#endif
#ifndef QS_PARK_MIN_NT
#define QS_PARK_MIN_NT 3  // query tiles from which the verify's P.V accumulators live in TMEM (NT = 2 fits registers)
#endif
#ifndef QS_TGT_PLO
#define QS_TGT_PLO 0  // target view P.V: p' as f16 hi only (1: hi + lo); |error| <= 2^-12 |p'|, as the draft view
#endif
#ifndef QS_DRAFT_TPW
#define QS_DRAFT_TPW 1  // A/B: draft consumer warps own this many 16-token tiles of a chunk (2: 5% slower, and
                         // breaks T-row == one-row invariance against the NT > 1 launches)
#endif  // halves per P row (16 tokens + pad: conflict-free transposes)

// NT: quantised modes -> query tiles of 8 queries (QK runs queries on the MMA M rows:
// hi parts in rows 0-7, lo parts in rows 8-15); fp16 mode -> n-tiles of 4 queries
// (hi/lo column pairs).  The fp16 tails inside a quantised launch use NTO = NQ/4 of the latter.
// NT: quantised modes -> query tiles of 8 queries (QK runs queries on the MMA M rows:
// hi parts in rows 0-7, lo parts in rows 8-15); fp16 mode -> n-tiles of 4 queries
// (hi/lo column pairs).  QR (quantised, NT == 1): query rows actually stored in the
// q' fragment buffers (the MHA draft has one query per KV head: QR = 1 keeps the stage small).
template <int HD, int NT, int MODE, int QR = 8>
struct AttnCfg {
  static constexpr bool QUANT = MODE != MODE_FP16;
  static constexpr int KS = HD / 16;
  // target view: queries on the QK M rows (ROWQ); draft and fp16 views: hi/lo column pairs
  static constexpr bool ROWQ = MODE == MODE_QTARGET;
  static constexpr int NCW = QUANT ? 8 / ((!ROWQ && NT == 1) ? QS_DRAFT_TPW : 1) : 4;  // compute warps
  static constexpr int NQ = ROWQ ? NT * 8 : NT * 4;      // queries per CTA
  static constexpr int NTO = NQ / 4;                     // hi/lo column-pair n-tiles of the fp16 path
  static constexpr int AQ = QR * 16;                     // words per (k-tile, query tile) of q' A fragments
  // ---- quantised stage: planes | key params | value params | Aq fragments | biases ----
  static constexpr int PLANE_CHUNK = HD * QS_CHUNK_Q / 2;
  static constexpr int NPLANE = (MODE == MODE_QTARGET) ? 4 : 2;
  static constexpr int KP_OFF = NPLANE * PLANE_CHUNK;
  static constexpr int VP_OFF = KP_OFF + QS_CHUNK_Q * 8;  // (128/G)*HD <= 128 key params (G >= HD)
  static constexpr int BQ_OFF = VP_OFF + QS_CHUNK_Q * 8;
  // ROWQ: A fragments [(128/G)*KS <= 8 k-tiles][NT][QR*4 lanes][a0..a3]; else B fragments [k-tile][NT][lane][b0 b1]
  static constexpr int BQ_WORDS = ROWQ ? 8 * NT * AQ : 8 * NT * 64;
  static constexpr int BIAS_OFF = BQ_OFF + BQ_WORDS * 4;
  static constexpr int BIAS_FLOATS = 8 * NQ * 2;          // [block][q][x1 tokens | x16 tokens]
  static constexpr int QSTAGE = (BIAS_OFF + BIAS_FLOATS * 4 + 127) / 128 * 128;
  // ---- fp16 chunks: 64 tokens in the fp16 kernel, 32 in the quantised kernel's tails ----
  // quantised kernels' fp1/fp2 tails: the whole 128-token buffer in one pass over all 8 warps
  // (the tail CTAs run in the second wave, after the main splits, so their latency is exposed)
  static constexpr int CF = QUANT ? 128 : 64;
  static constexpr int FSTAGE = 2 * CF * HD * 2;
  static constexpr int NSTAGE_F = QUANT ? 1 : 2;
  static constexpr int REGION_F = NSTAGE_F * FSTAGE;
  static constexpr int MS = HD + 4;
  static constexpr int MERGE_BYTES = NCW * NQ * MS * 4;
  static constexpr int BQF_WORDS = ROWQ ? KS * NT * AQ : KS * NTO * 64;  // query fragments of fp16 chunks
  static constexpr int PW_HALVES = NTO * 8 * PSTRIDE;
  // 16-token tiles per consumer warp per chunk in the draft view (and the fp16 tails of a draft
  // launch): TPW = 2 halves the consumer warps and shares each warp's per-chunk overhead over two tiles
  static constexpr int TPW = (QUANT && !ROWQ && NT == 1) ? QS_DRAFT_TPW : 1;
  static constexpr int PW_WARP = PW_HALVES * TPW;  // halves of P transpose buffer per warp
  static constexpr int FIXED = BQF_WORDS * 4 + NQ * HD * 4 + (ROWQ ? 0 : NCW * PW_WARP * 2) + 4 * 8 * 8 + 16;
  // TMA ring: two CTAs per SM when at least 4 stages fit each (of 228 KB, 1 KB reserved per CTA),
  // else one CTA with the deepest ring that fits; at most 6 stages
  static constexpr int S2 = (233472 / 2 - 1024 - FIXED) / QSTAGE;
  static constexpr int S1 = (232448 - FIXED) / QSTAGE;
  static constexpr int MIN_BLOCKS = QUANT ? ((NT == 1 && S2 >= 4) ? 2 : 1) : 3;  // wide launches: registers
  // TMAW (one CTA per SM, the target's wide fold): NPW = NSTAGE fold warps each own one ring stage
  // -- fold its chunk, hand it to the consumers, and refill it with the chunk NSTAGE ahead as soon
  // as they release it -- so every mbarrier's phases are waited in order by a single warp (a parity
  // wait can never run a phase ahead) and no separate TMA warp is needed: 8 + 4 = 12 warps, three
  // per SM sub-partition, 168 registers each.  Otherwise (two CTAs per SM, or the draft's cheap
  // fold) two fold warps alternate chunks and refill the ring themselves behind the consumers.
  static constexpr bool TMAW = ROWQ && MIN_BLOCKS == 1;
  static constexpr int NSTAGE =
      QUANT ? (MIN_BLOCKS == 2 ? (S2 < 6 ? S2 : 6) : TMAW ? (S1 < 4 ? S1 : 4) : (S1 < 6 ? S1 : 6)) : 1;
  static constexpr int NPW = QUANT ? (TMAW ? NSTAGE : (NSTAGE > 2 ? 2 : 1)) : 0;
  static constexpr int NWARPS = NCW + NPW;
  static constexpr int THREADS = NWARPS * 32;
  static constexpr int REGION_Q = QUANT ? NSTAGE * QSTAGE : 0;
  static constexpr int R0 = REGION_Q > REGION_F ? REGION_Q : REGION_F;
  static constexpr int REGION = R0 > MERGE_BYTES ? R0 : MERGE_BYTES;
  // query slots the fold computes: the draft stores QR live queries per CTA (MHA draft: 1 of NQ = 4)
  static constexpr int NQF = (QR < 8 && QR < NQ) ? QR : NQ;  // QR = 8: every slot
  static constexpr int VPAD = 2 * NQF <= 2 ? 2 : 2 * NQF <= 4 ? 4 : 2 * NQF <= 8 ? 8 : 2 * NQF <= 16 ? 16 :
                              2 * NQF <= 32 ? 32 : 64;  // fold reduce-scatter width
  static constexpr int SMEM = REGION + FIXED;
  // wide-query verify (NT >= 2 query tiles: GQA r*T queries, or T > 8): the consumers' P.V
  // accumulators of every query tile live in tensor memory between chunks (32 columns per tile per
  // warp; warps w, w+4 share a lane quarter) -- one CTA streams a head's chunks once for all its
  // queries without the register file holding NT x 32 accumulators per thread
  static constexpr bool PARK = ROWQ && NT >= QS_PARK_MIN_NT;
  static constexpr int TMEM_COLS = !PARK ? 0 : (2 * NT * 32 <= 128 ? 128 : 256);
  // registers per thread: each SM sub-partition holds 16K registers and gets every 4th resident
  // warp, so the busiest one holds ceil(MIN_BLOCKS * NWARPS / 4) warps (8-register granules)
  static constexpr int WPS = (MIN_BLOCKS * NWARPS + 3) / 4;
  static constexpr int MAXREG_ = (16384 / (WPS * 32)) / 8 * 8;
  static constexpr int MAXREG = MAXREG_ > 255 ? 255 : MAXREG_;
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
  float m, l, z, ps;  // running max (log2), denominator, sum p*Z_v, sum of fed f16 p' (offset removal)
};

// per-warp online softmax for the query column owned by this lane (t4)
// LAZY: the running max is only a reference point -- it is raised (warp max, rescale) when some
// score exceeds it by more than 2^QS_LAZY_MAX_LOG2 (p then stays <= 2^QS_LAZY_MAX_LOG2), which takes
// the three max shuffles off most chunks' dependency chain; the result is normalised by the same
// reference, so only the rounding of p changes (deterministic, independent of the other rows)
template <int NS, bool LAZY = false>
__device__ __forceinline__ float softmax_update(Softmax& st, const float (&s)[NS], float (&p)[NS]) {
  float mx = kNegInf;
#pragma unroll
  for (int i = 0; i < NS; ++i) mx = fmaxf(mx, s[i]);
  if constexpr (LAZY) {
    if (!__any_sync(0xffffffffu, mx > st.m + (float)QS_LAZY_MAX_LOG2)) {
      const float mu = st.m == kNegInf ? 0.f : st.m;  // a dead first tile: p = 0, not NaN
#pragma unroll
      for (int i = 0; i < NS; ++i) p[i] = ex2_approx(s[i] - mu);
      return 1.0f;
    }
  }
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 4));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 8));
  mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
  float alpha = 1.0f;
  // the raise is decided per query on its own (column-reduced) max, so a query's reference --
  // and every rounding after it -- does not depend on which other queries share the warp
  if (mx > st.m + (LAZY ? (float)QS_LAZY_MAX_LOG2 : 0.f)) {
    alpha = ex2_approx(st.m - mx);  // st.m == -inf -> 0
    st.l *= alpha;
    st.z *= alpha;
    st.ps *= alpha;
    st.m = mx;
  }
  const float mu = st.m == kNegInf ? 0.f : st.m;  // every score -inf: p = ex2(-inf) = 0, not NaN
#pragma unroll
  for (int i = 0; i < NS; ++i) p[i] = ex2_approx(s[i] - mu);
  return alpha;
}

template <int KS, int NT>
__device__ __forceinline__ void rescale(float (&acc)[KS][NT][4], int nt, float alpha) {
#pragma unroll
  for (int a = 0; a < KS; ++a) {
    acc[a][nt][0] *= alpha;
    acc[a][nt][1] *= alpha;
    acc[a][nt][2] *= alpha;
    acc[a][nt][3] *= alpha;
  }
}

// write p' hi/lo for tokens g, g+8 of column pair (2 t4, 2 t4 + 1) of n-tile nt
__device__ __forceinline__ void put_p(__half* pw, int nt, int g, int t4, __half h0, __half l0, __half h1, __half l1) {
  __half* row = pw + (nt * 8 + 2 * t4) * PSTRIDE;
  row[g] = h0;
  row[g + 8] = h1;
  row[PSTRIDE + g] = l0;
  row[PSTRIDE + g + 8] = l1;
}

template <int NT>
__device__ __forceinline__ void get_pv_b(const __half* pw, int g, int t4, uint32_t (&bpv)[NT][2]) {
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const __half* row = pw + (nt * 8 + g) * PSTRIDE;
    bpv[nt][0] = *reinterpret_cast<const uint32_t*>(row + 2 * t4);
    bpv[nt][1] = *reinterpret_cast<const uint32_t*>(row + 2 * t4 + 8);
  }
}

// B fragment words of (scaled) query q at channel pair cp of one 16-channel tile
// (layout [tile][nt][lane][2]; column 2q = hi, 2q+1 = lo)
__device__ __forceinline__ void put_qfrag(uint32_t* tile_base, int cp, int q, __half h0, __half h1, __half l0,
                                          __half l1) {
  const int jj = cp & 7, tt = jj & 3, which = jj >> 2;
  const int col = 2 * q;
  uint32_t* bb = tile_base + (col >> 3) * 64 + (col & 7) * 8 + tt * 2 + which;
  bb[0] = h2_as_u32(__halves2half2(h0, h1));
  bb[8] = h2_as_u32(__halves2half2(l0, l1));
}

// ---------------------------------------------------------------------------
// fp16 region (fp1 / fp2 tails, sensitive-layer archive, fp16 cache): all warps
// ---------------------------------------------------------------------------
template <typename C, int HD, int NT>
__device__ __forceinline__ void fp16_region(uint8_t* region, uint32_t* bqf, const float* q_s, __half* pw, int nq,
                                            const __half* fk, const __half* fv, int n_tok, int c_begin, int c_end,
                                            int causal, int qg, const AttnParams& P, Softmax (&st)[NT],
                                            float (&acc)[C::KS][NT][4]) {
  constexpr int KS = C::KS, NQ = C::NQ, NTH = C::THREADS, CF = C::CF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const float sl2 = P.sm_scale_log2;
  for (int i = tid; i < C::BQF_WORDS; i += NTH) bqf[i] = 0u;
  __syncthreads();
  for (int j = tid; j < (HD / 2) * nq; j += NTH) {
    const int cp = j % (HD / 2), q = j / (HD / 2);
    __half h0, l0, h1, l1;
    split_hl(q_s[q * HD + 2 * cp], h0, l0);
    split_hl(q_s[q * HD + 2 * cp + 1], h1, l1);
    put_qfrag(bqf + (size_t)(cp >> 3) * NT * 64, cp, q, h0, h1, l0, l1);
  }
  const int nchunk = c_end - c_begin;
  constexpr int NCH16 = HD / 8;
  auto fstage = [&](int s) { return reinterpret_cast<__half*>(region + s * C::FSTAGE); };
  auto issue_f = [&](int i) {
    if (i < nchunk) {
      int c = c_begin + i;
      __half* ks_ = fstage(i % C::NSTAGE_F);
      __half* vs_ = ks_ + CF * HD;
      for (int idx = tid; idx < CF * NCH16; idx += NTH) {
        int row = idx / NCH16, ch = idx % NCH16;
        int tok = c * CF + row;
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
    if constexpr (C::NSTAGE_F == 1) {
      if (i > 0) __syncthreads();  // every warp is done with the previous chunk
      issue_f(i);
      cp_async_wait<0>();
    } else {
      cp_async_wait<C::NSTAGE_F - 2>();
    }
    __syncthreads();
    if constexpr (C::NSTAGE_F > 1) issue_f(i + C::NSTAGE_F - 1);
    // the warp's TPW 16-token tiles of the chunk, one after another (one softmax state per warp)
    for (int tt = 0; tt < C::TPW; ++tt) {
    const int mt = warp * C::TPW + tt;
    if (!(mt * 16 < CF && warp < C::NCW)) continue;
    const int c = c_begin + i;
    const __half* ks_ = fstage(i % C::NSTAGE_F);
    const __half* vs_ = ks_ + CF * HD;
    const int ntok_chunk = min(CF, n_tok - c * CF);
    const bool live = mt * 16 < ntok_chunk;
    float d0[NT][4], d1[NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int e = 0; e < 4; ++e) d0[nt][e] = d1[nt][e] = 0.f;
    const int ii = lane >> 3, rr = lane & 7;
    if (live) {
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        int row = mt * 16 + (ii & 1) * 8 + rr;
        int ch = ks * 2 + (ii >> 1);
        uint32_t a[4];
        ldmatrix_x4(a, smem_u32(ks_ + row * HD + swz16(ch, row, NCH16) * 8));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          uint2 b = *reinterpret_cast<const uint2*>(bqf + (((size_t)ks * NT + nt) * 32 + lane) * 2);
          if (ks & 1) mma16816(d1[nt], a, b.x, b.y);
          else mma16816(d0[nt], a, b.x, b.y);
        }
      }
    }
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      int lim = n_tok;
      if (causal) {
        int qgl = qg * NQ + nt * 4 + t4;
        int t = min(qgl / P.r, P.T - 1);
        lim = n_tok - (P.T - 1 - t);
      }
      const int tok0 = c * CF + mt * 16 + g;
      float sv[2], p[2];
      sv[0] = (live && tok0 < lim) ? ((d0[nt][0] + d0[nt][1]) + (d1[nt][0] + d1[nt][1])) * sl2 : kNegInf;
      sv[1] = (live && tok0 + 8 < lim) ? ((d0[nt][2] + d0[nt][3]) + (d1[nt][2] + d1[nt][3])) * sl2 : kNegInf;
      float alpha = softmax_update<2>(st[nt], sv, p);
      if (alpha != 1.0f) rescale<KS, NT>(acc, nt, alpha);
      st[nt].l += p[0] + p[1];
      __half h0, l0, h1, l1;
      split_hl(p[0], h0, l0);
      split_hl(p[1], h1, l1);
      put_p(pw, nt, g, t4, h0, l0, h1, l1);
    }
    __syncwarp();
    if (live) {
      uint32_t bpv[NT][2];
      get_pv_b<NT>(pw, g, t4, bpv);
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
  }
  cp_async_wait<0>();
}

// TMA bulk copies of quantised chunk i of this CTA's range (planes + key/value params)
// into ring stage i % NSTAGE; completion is counted on tma_b[stage].  Reads only
// blocks below n_blocks, which no kernel of a decode forward modifies, so the
// first NSTAGE chunks are issued before the grid dependency resolves (PDL).
#ifndef QS_ATTN_L2PF
#define QS_ATTN_L2PF 0  // A/B: L2 bulk prefetch this many ring depths ahead of the TMA ring (0: off)
#endif
template <typename C, int HD, int MODE>
__device__ __forceinline__ void quant_issue(const AttnParams& P, uint8_t* region, uint64_t* tma_b, int seq, int head,
                                            int n_blocks, int c_begin, int i, int nchunk) {
  constexpr bool TGT = MODE == MODE_QTARGET;
  const int G = P.G;
  const int bpc = QS_CHUNK_Q >> (31 - __clz(G));  // G is a power of two: no integer division per issue
  const size_t plane_blk = (size_t)G * HD / 2;
  const size_t ph = ((size_t)seq * P.plane_seq_stride) + (size_t)head * P.plane_head_stride;
  const float2* kp = reinterpret_cast<const float2*>(P.kp) + (size_t)seq * P.kp_seq_stride + (size_t)head * P.kp_head_stride;
  const float2* vp = reinterpret_cast<const float2*>(P.vp) + (size_t)seq * P.vp_seq_stride + (size_t)head * P.vp_head_stride;
  const int c = c_begin + i, s = i % C::NSTAGE;
  uint8_t* sp = region + s * C::QSTAGE;
  const int b0 = c * bpc, nb = min(bpc, n_blocks - b0);
  const uint32_t pbytes = (uint32_t)(nb * plane_blk);
  const uint32_t kpb = (uint32_t)(nb * HD * 8), vpb = (uint32_t)(nb * G * 8);
  // planes complete on tma_b[s]; the (S, Z) params on their own barrier (tma_b[24 + s]), so the
  // fold -- which needs only the key params -- starts while the planes are still streaming in
  // (the target's stage-owning fold only: the draft's cheap fold measured 2% better on one barrier)
  uint64_t* tma_p = C::TMAW ? tma_b + 24 : tma_b;
  if constexpr (C::TMAW) {
    mbar_arrive_expect_tx(&tma_b[s], pbytes * C::NPLANE);
    mbar_arrive_expect_tx(&tma_p[s], kpb + vpb);
  } else {
    mbar_arrive_expect_tx(&tma_b[s], pbytes * C::NPLANE + kpb + vpb);
  }
  bulk_g2s(sp + C::KP_OFF, kp + (size_t)b0 * HD, kpb, &tma_p[s]);
  bulk_g2s(sp + C::VP_OFF, vp + (size_t)b0 * G, vpb, &tma_p[s]);
  bulk_g2s(sp, P.ku + ph + b0 * plane_blk, pbytes, &tma_b[s]);
  bulk_g2s(sp + C::PLANE_CHUNK, P.vu + ph + b0 * plane_blk, pbytes, &tma_b[s]);
  if constexpr (TGT) {
    bulk_g2s(sp + 2 * C::PLANE_CHUNK, P.kl + ph + b0 * plane_blk, pbytes, &tma_b[s]);
    bulk_g2s(sp + 3 * C::PLANE_CHUNK, P.vl + ph + b0 * plane_blk, pbytes, &tma_b[s]);
  }
  if constexpr (QS_ATTN_L2PF > 0) {
    // the chunk one ring depth further on goes to L2 now: twice the ring's bytes in flight to DRAM
    const int ip = i + C::NSTAGE * QS_ATTN_L2PF;
    if (ip < nchunk) {
      const int pb0 = (c_begin + ip) * bpc, pnb = min(bpc, n_blocks - pb0);
      const uint32_t pby = (uint32_t)(pnb * plane_blk);
      bulk_prefetch_l2(kp + (size_t)pb0 * HD, (uint32_t)(pnb * HD * 8));
      bulk_prefetch_l2(vp + (size_t)pb0 * G, (uint32_t)(pnb * G * 8));
      bulk_prefetch_l2(P.ku + ph + pb0 * plane_blk, pby);
      bulk_prefetch_l2(P.vu + ph + pb0 * plane_blk, pby);
      if constexpr (TGT) {
        bulk_prefetch_l2(P.kl + ph + pb0 * plane_blk, pby);
        bulk_prefetch_l2(P.vl + ph + pb0 * plane_blk, pby);
      }
    }
  }
}

// fp16 tails of a quantised launch (fp1 / fp2 recent-token buffers) in the quantised
// path's register layout: queries on the MMA M rows (hi rows g, lo rows g+8), tokens on N,
// so P feeds P.V straight from registers and the merge is shared with quant_region.
template <typename C, int HD, int NT>
__device__ __forceinline__ void fp16_region_q(uint8_t* region, uint32_t* aqf, const float* q_s, int nq,
                                              const __half* fk, const __half* fv, int n_tok, int c_begin, int c_end,
                                              int causal, int qg, const AttnParams& P, Softmax (&st)[NT],
                                              float (&acc)[C::KS][NT][4], uint32_t tacc = 0) {
  constexpr int KS = C::KS, NQ = C::NQ, NTH = C::THREADS, CF = C::CF;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const float sl2 = P.sm_scale_log2;
  for (int i = tid; i < C::BQF_WORDS; i += NTH) aqf[i] = 0u;
  __syncthreads();
  // A fragments of the raw queries: [k-tile][query tile][lane][a0..a3]
  for (int j = tid; j < (HD / 2) * nq; j += NTH) {
    const int cp = j % (HD / 2), q = j / (HD / 2);
    const float2 qv = *reinterpret_cast<const float2*>(q_s + q * HD + 2 * cp);
    const __half2 hi = __floats2half2_rn(qv.x, qv.y);
    const float2 hf = __half22float2(hi);
    const __half2 lo = __floats2half2_rn(qv.x - hf.x, qv.y - hf.y);
    const int jj = cp & 7;
    uint32_t* bb = aqf + (size_t)((cp >> 3) * NT + (q >> 3)) * C::AQ + (q & 7) * 16 + (jj & 3) * 4 + 2 * (jj >> 2);
    bb[0] = h2_as_u32(hi);
    bb[1] = h2_as_u32(lo);
  }
  const int nchunk = c_end - c_begin;
  constexpr int NCH16 = HD / 8;
  auto fstage = [&](int s) { return reinterpret_cast<__half*>(region + s * C::FSTAGE); };
  auto issue_f = [&](int i) {
    if (i < nchunk) {
      int c = c_begin + i;
      __half* ks_ = fstage(i % C::NSTAGE_F);
      __half* vs_ = ks_ + CF * HD;
      for (int idx = tid; idx < CF * NCH16; idx += NTH) {
        int row = idx / NCH16, ch = idx % NCH16;
        int tok = c * CF + row;
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
  const int mt = warp;
  const bool has_tile = mt * 16 < CF && warp < C::NCW;
  const int ii = lane >> 3, rr = lane & 7;
  for (int i = 0; i < nchunk; ++i) {
    if constexpr (C::NSTAGE_F == 1) {
      if (i > 0) __syncthreads();  // every warp is done with the previous chunk
      issue_f(i);
      cp_async_wait<0>();
    } else {
      cp_async_wait<C::NSTAGE_F - 2>();
    }
    __syncthreads();
    if constexpr (C::NSTAGE_F > 1) issue_f(i + C::NSTAGE_F - 1);
    if (!has_tile) continue;
    const int c = c_begin + i;
    const __half* ks_ = fstage(i % C::NSTAGE_F);
    const __half* vs_ = ks_ + CF * HD;
    const int tok_base = c * CF + mt * 16;
    if (tok_base < n_tok) {
      float d[2][NT][4];
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) d[j][nt][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        // x4: (tokens 0-7 | 8-15) x (channels lo | hi) of the k-tile = B fragments of both token n-tiles
        const int row = mt * 16 + (ii & 1) * 8 + rr;
        const int ch = ks * 2 + (ii >> 1);
        uint32_t b[4];
        ldmatrix_x4(b, smem_u32(ks_ + row * HD + swz16(ch, row, NCH16) * 8));
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint4 a4 = lane < C::AQ / 4 ? reinterpret_cast<const uint4*>(aqf)[(ks * NT + nt) * (C::AQ / 4) + lane]
                                          : make_uint4(0u, 0u, 0u, 0u);
          const uint32_t af[4] = {a4.x, a4.y, a4.z, a4.w};
          mma_nv(d[0][nt], af, b[0], b[2]);
          mma_nv(d[1][nt], af, b[1], b[3]);
        }
      }
      uint32_t bph[NT][2], bpl[NT][2];
      bool resc[NT];
      float al0[NT], al1[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        int lim = n_tok;
        if (causal) {
          const int qgl = qg * NQ + nt * 8 + g;
          const int t = min(qgl / P.r, P.T - 1);
          lim = n_tok - (P.T - 1 - t);
        }
        float sv[2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int tok = tok_base + 8 * j + 2 * t4 + e;
            sv[j][e] = tok < lim ? (d[j][nt][e] + d[j][nt][e + 2]) * sl2 : kNegInf;
          }
        float mx = fmaxf(fmaxf(sv[0][0], sv[0][1]), fmaxf(sv[1][0], sv[1][1]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
        float alpha = 1.0f;
        if (mx > st[nt].m) {
          alpha = ex2_approx(st[nt].m - mx);
          st[nt].l *= alpha;
          st[nt].m = mx;
        }
        if constexpr (C::PARK) {
          resc[nt] = __any_sync(0xffffffffu, alpha != 1.0f);
          al0[nt] = __shfl_sync(0xffffffffu, alpha, 8 * t4);
          al1[nt] = __shfl_sync(0xffffffffu, alpha, 8 * t4 + 4);
        } else if (__any_sync(0xffffffffu, alpha != 1.0f)) {
          const float a0 = __shfl_sync(0xffffffffu, alpha, 8 * t4);
          const float a1 = __shfl_sync(0xffffffffu, alpha, 8 * t4 + 4);
#pragma unroll
          for (int cm = 0; cm < KS; ++cm) {
            acc[cm][nt][0] *= a0;
            acc[cm][nt][1] *= a1;
            acc[cm][nt][2] *= a0;
            acc[cm][nt][3] *= a1;
          }
        }
        const float m = st[nt].m == kNegInf ? 0.f : st[nt].m;
        float p[2][2];
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) p[j][e] = ex2_approx(sv[j][e] - m);
        st[nt].l += (p[0][0] + p[0][1]) + (p[1][0] + p[1][1]);
        const __half2 h0 = __floats2half2_rn(p[0][0], p[0][1]), h1 = __floats2half2_rn(p[1][0], p[1][1]);
        const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
        bph[nt][0] = h2_as_u32(h0);
        bph[nt][1] = h2_as_u32(h1);
        bpl[nt][0] = h2_as_u32(__floats2half2_rn(p[0][0] - f0.x, p[0][1] - f0.y));
        bpl[nt][1] = h2_as_u32(__floats2half2_rn(p[1][0] - f1.x, p[1][1] - f1.y));
      }
      if constexpr (C::PARK) {
        uint32_t va[KS][4];
#pragma unroll
        for (int cm = 0; cm < KS; ++cm) {
          const int row = mt * 16 + (ii >> 1) * 8 + rr;
          const int ch = cm * 2 + (ii & 1);
          ldmatrix_x4_trans(va[cm], smem_u32(vs_ + row * HD + swz16(ch, row, NCH16) * 8));
        }
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float aw[32];
          tmem_ld32(tacc + nt * 32, aw);
          if (resc[nt]) {
#pragma unroll
            for (int cm = 0; cm < KS; ++cm) {
              aw[cm * 4 + 0] *= al0[nt];
              aw[cm * 4 + 1] *= al1[nt];
              aw[cm * 4 + 2] *= al0[nt];
              aw[cm * 4 + 3] *= al1[nt];
            }
          }
#pragma unroll
          for (int cm = 0; cm < KS; ++cm) {
            float (&a4)[4] = *reinterpret_cast<float(*)[4]>(aw + cm * 4);
            mma_nv(a4, va[cm], bph[nt][0], bph[nt][1]);
            if constexpr (QS_TGT_PLO) mma_nv(a4, va[cm], bpl[nt][0], bpl[nt][1]);
          }
          tmem_st32(tacc + nt * 32, aw);
        }
      } else {
#pragma unroll
        for (int cm = 0; cm < KS; ++cm) {
          const int row = mt * 16 + (ii >> 1) * 8 + rr;
          const int ch = cm * 2 + (ii & 1);
          uint32_t a[4];
          ldmatrix_x4_trans(a, smem_u32(vs_ + row * HD + swz16(ch, row, NCH16) * 8));
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma_nv(acc[cm][nt], a, bph[nt][0], bph[nt][1]);
            if constexpr (QS_TGT_PLO) mma_nv(acc[cm][nt], a, bpl[nt][0], bpl[nt][1]);
          }
        }
      }
    }
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// quantised region: producer warp + 8 consumer warps
// ---------------------------------------------------------------------------
template <typename C, int HD, int NT, int MODE>
__device__ __forceinline__ void quant_region(uint8_t* region, uint64_t* bars, const float* q_s, __half* pw, int nq,
                                             int seq, int head, int n_tok, int c_begin, int c_end,
                                             const AttnParams& P, Softmax (&st)[NT], float (&acc)[C::KS][NT][4],
                                             uint32_t tacc = 0) {
  constexpr int KS = C::KS, NQ = C::NQ, S = C::NSTAGE;
  constexpr bool TGT = MODE == MODE_QTARGET;
  constexpr float kvs = TGT ? 0.0625f : 1.0f;  // target code = 16 c_u + c_l -> scale S/16
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  uint64_t* tma_b = bars;
  uint64_t* full_b = bars + 8;
  uint64_t* empty_b = bars + 16;
  const int G = P.G;
  const int lgG = 31 - __clz(G);
  const int n_blocks = P.n_blocks[seq];
  const int nchunk = c_end - c_begin;
  const int tok_left = n_tok - c_begin * QS_CHUNK_Q;  // tokens from this CTA's first chunk on
  auto stage_ptr = [&](int s) { return region + s * C::QSTAGE; };

  if (warp >= C::NCW) {
    // ======================= producer warps (NPW) =======================
    auto issue = [&](int i) { quant_issue<C, HD, MODE>(P, region, tma_b, seq, head, n_blocks, c_begin, i, nchunk); };
    const int pwid = warp - C::NCW;
    // Producer warp p folds whole chunks j = p (mod NPW) on its own (no inter-warp
    // synchronisation: the per-chunk fold is a latency chain, so independent warps
    // overlap it), then refills the stage of its previous chunk once the consumers
    // have released it.  Lane l folds channel pairs cp = l + 32 k.
    constexpr int NPW = C::NPW;
    constexpr int CPL = (HD / 2 + 31) / 32;
    constexpr bool QREG = false;  // queries re-read from shared memory (keeps the 2-CTA/SM register budget)
    float2 qr[QREG ? NQ : 1][CPL];
    if constexpr (QREG) {
#pragma unroll
      for (int q = 0; q < NQ; ++q)
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const int cp = lane + 32 * k;
          qr[q][k] = cp < HD / 2 ? *reinterpret_cast<const float2*>(q_s + q * HD + 2 * cp) : make_float2(0.f, 0.f);
        }
    }
    // chunks 0..S-1 were issued by the kernel prologue (before pdl_wait)
    static_assert(NPW <= S, "fold warps step through the ring");
    int s = pwid % S, ph = (pwid / S) & 1, s_prev = 0, ph_prev = 0;
    for (int j = pwid; j < nchunk; j += NPW) {
      uint8_t* sp = stage_ptr(s);
      attn_wait(&tma_b[(C::TMAW ? 24 : 0) + s], ph);  // the chunk's (S, Z) params (target: planes may still be in flight)
      // the consumers' release of this stage's previous chunk (j - S) -- already complete, since the
      // refill that brought chunk j was issued after it, but that edge runs through another fold warp
      // and the TMA engine; waiting here makes the fragment rewrite's ordering explicit (racecheck)
      if (!C::TMAW && j >= S) attn_wait(&empty_b[s], ph ^ 1);
      const int ntok_chunk = min(QS_CHUNK_Q, n_tok - (c_begin + j) * QS_CHUNK_Q);
      const int nbl = (ntok_chunk + G - 1) >> lgG;
      const float2* kps = reinterpret_cast<const float2*>(sp + C::KP_OFF);
      uint32_t* bqb = reinterpret_cast<uint32_t*>(sp + C::BQ_OFF);
      float* bias = reinterpret_cast<float*>(sp + C::BIAS_OFF);
      // q'_c = q_c * S_c as f16 hi/lo B fragments; per (block, query): bias = sum q Z - offset * sum(q').
      // All queries are processed together so the warp reductions overlap (ILP), not serialise.
      constexpr int NQF = C::NQF;
      for (int bl = 0; bl < ((P.dbg & 2) ? 0 : nbl); ++bl) {
        float zs[NQF], bs[NQF];
#pragma unroll
        for (int q = 0; q < NQF; ++q) zs[q] = bs[q] = 0.f;
#pragma unroll
        for (int k = 0; k < CPL; ++k) {
          const int cp = lane + 32 * k;
          if (cp < HD / 2) {
            const float4 pz = *reinterpret_cast<const float4*>(kps + bl * HD + 2 * cp);  // (S0, Z0, S1, Z1)
            const float s0 = pz.x * kvs, s1 = pz.z * kvs;
            // ROWQ: A fragment of k-tile cp/8, lane (q%8)*4 + (cp%4), register 2*((cp/4)%2) (+1 for lo);
            // else B fragment (columns 2q = hi, 2q+1 = lo), lane (col%8)*4 + cp%4, register (cp/4)%2
            const int jj = cp & 7;
            uint32_t* tb = C::ROWQ ? bqb + (size_t)(bl * KS + (cp >> 3)) * NT * C::AQ + (jj & 3) * 4 + 2 * (jj >> 2)
                                   : bqb + (size_t)(bl * KS + (cp >> 3)) * NT * 64 + (jj & 3) * 2 + (jj >> 2);
#pragma unroll
            for (int q = 0; q < NQF; ++q) {
              if (q < nq) {
                const float2 qv = QREG ? qr[QREG ? q : 0][k] : *reinterpret_cast<const float2*>(q_s + q * HD + 2 * cp);
                const float v0 = qv.x * s0, v1 = qv.y * s1;
                const __half2 hi = __floats2half2_rn(v0, v1);
                const float2 hf = __half22float2(hi);
                const __half2 lo = __floats2half2_rn(v0 - hf.x, v1 - hf.y);
                const float2 lf = __half22float2(lo);
                if constexpr (C::ROWQ) {
                  uint32_t* bb = tb + (q >> 3) * C::AQ + (q & 7) * 16;
                  bb[0] = h2_as_u32(hi);
                  bb[1] = h2_as_u32(lo);
                } else {
                  uint32_t* bb = tb + ((2 * q) >> 3) * 64 + ((2 * q) & 7) * 8;
                  bb[0] = h2_as_u32(hi);
                  bb[8] = h2_as_u32(lo);
                }
                zs[q] += qv.x * pz.y + qv.y * pz.w;
                bs[q] += (hf.x + hf.y) + (lf.x + lf.y);
              }
            }
          }
        }
        // warp reduce-scatter of the 2*NQ partial sums (zs then bs): each level halves
        // the values a lane holds, so 2*NQ-1 shuffles replace 5*2*NQ dependent ones
        constexpr int V = C::VPAD;  // 2*NQF padded to a power of two
        constexpr int LV = V == 2 ? 1 : V == 4 ? 2 : V == 8 ? 3 : V == 16 ? 4 : 5;  // levels (V = 64: five, two sums per lane)
        float vals[V];
#pragma unroll
        for (int i = 0; i < V; ++i) vals[i] = 0.f;
#pragma unroll
        for (int q = 0; q < NQF; ++q) {
          vals[q] = zs[q];
          vals[NQF + q] = bs[q];
        }
#pragma unroll
        for (int l = 0, h = V / 2; l < LV; ++l, h >>= 1) {
          const int o = 16 >> l;
          const bool up = lane & o;
#pragma unroll
          for (int i = 0; i < h; ++i) {
            const float send = up ? vals[i] : vals[i + h];
            const float keep = up ? vals[i + h] : vals[i];
            vals[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
          }
        }
        const int qq = lane < nq ? lane : 0;
        float z, b;
        if constexpr (V == 64) {
          // sum idx sits in lane idx >> 1, slot idx & 1
          const float z0 = __shfl_sync(0xffffffffu, vals[0], qq >> 1), z1 = __shfl_sync(0xffffffffu, vals[1], qq >> 1);
          const float b0 = __shfl_sync(0xffffffffu, vals[0], (NQF + qq) >> 1);
          const float b1 = __shfl_sync(0xffffffffu, vals[1], (NQF + qq) >> 1);
          z = (qq & 1) ? z1 : z0;
          b = ((NQF + qq) & 1) ? b1 : b0;
        } else {
          float tot = vals[0];
#pragma unroll
          for (int o = 16 >> LV; o > 0; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
          // lanes [idx << (5-LV), (idx+1) << (5-LV)) now hold sum idx (idx < NQ: zs, else bs)
          z = __shfl_sync(0xffffffffu, tot, qq << (5 - LV));
          b = __shfl_sync(0xffffffffu, tot, (NQF + qq) << (5 - LV));
        }
        // draft tokens g of a 16-token tile carry 1024 + c, tokens g+8 carry (1024 + 16c) (scaled
        // by 1/16 after the MMA); target tokens carry 1032 + (16 c_u + c_l)
        if (lane < nq) {
          bias[(bl * NQ + lane) * 2 + 0] = z - (TGT ? 1032.f : 1024.f) * b;
          bias[(bl * NQ + lane) * 2 + 1] = z - (TGT ? 1032.f : 64.f) * b;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&full_b[s]);
      // refill the stage of this warp's previous chunk (every chunk >= S is issued exactly once)
      const int jp = j - NPW;
      if constexpr (C::TMAW) {
        // this warp's stage: refill it with chunk j + S once the consumers release chunk j
        if (j + S < nchunk) {
          attn_wait(&empty_b[s], ph);
          if (lane == 0) issue(j + S);
          __syncwarp();
        }
      } else if (jp >= 0 && jp + S < nchunk) {
        attn_wait(&empty_b[s_prev], ph_prev);
        if (lane == 0) issue(jp + S);
      }
      s_prev = s;
      ph_prev = ph;
      s += NPW;
      if (s >= S) {
        s -= S;
        ph ^= 1;
      }
    }
    return;
  }

  if constexpr (C::ROWQ) {
  // ======================= consumer warps =======================
  // Warp mt owns token tile mt (16 tokens) of every chunk.
  //   Q.K^T (queries on M): A = q' fragments (rows g: hi, rows g+8: lo of query g), B = the
  //   tile's K codes as two n-tiles (tokens g | g+8: the frag4 word of an A tile K[token][ch]
  //   is exactly the B fragment pair of K^T), so each lane ends up with the scores of query g
  //   for tokens 2t, 2t+1, 2t+8, 2t+9 -- already the B-fragment layout of P for P.V.
  //   P.V (channels on M): A = V^T codes, B = p' = p * S_v (hi, and lo for the target).
  const float sl2 = P.sm_scale_log2;
  const int mt = warp;
  for (int i = 0, s = 0, ph = 0; i < nchunk; ++i) {
    const uint8_t* sp = stage_ptr(s);
    attn_wait(&full_b[s], ph);  // folded query fragments + biases
    attn_wait(&tma_b[s], ph);   // packed planes
    const bool live = mt * 16 + i * QS_CHUNK_Q < tok_left && !(P.dbg & 1);  // tiles are whole: G is a multiple of 16
    if (live) {
      const int bl = (mt * 16) >> lgG;
      const uint4* aq = reinterpret_cast<const uint4*>(sp + C::BQ_OFF) + (size_t)bl * KS * NT * (C::AQ / 4) + lane;
      const float* bias = reinterpret_cast<const float*>(sp + C::BIAS_OFF);
      const float4* vps4 = reinterpret_cast<const float4*>(sp + C::VP_OFF);  // (S, Z) of tokens 2k, 2k+1
      uint32_t wu[KS], wl[KS];
      load_words<KS>(reinterpret_cast<const uint32_t*>(sp), mt, lane, wu);
      if constexpr (TGT) load_words<KS>(reinterpret_cast<const uint32_t*>(sp + 2 * C::PLANE_CHUNK), mt, lane, wl);
      float d[2][NT][4];  // [token half][query tile]: two independent MMA chains
#pragma unroll
      for (int j = 0; j < 2; ++j)
#pragma unroll
        for (int nt = 0; nt < NT; ++nt)
#pragma unroll
          for (int e = 0; e < 4; ++e) d[j][nt][e] = 0.f;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        uint32_t r[4];
        if constexpr (TGT) unpack_u4l4_raw(wu[ks], wl[ks], r);
        else unpack_u4_raw(wu[ks], r);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint4 a4 = lane < C::AQ / 4 ? aq[(ks * NT + nt) * (C::AQ / 4)] : make_uint4(0u, 0u, 0u, 0u);
          const uint32_t af[4] = {a4.x, a4.y, a4.z, a4.w};
          mma_nv(d[0][nt], af, r[0], r[2]);  // tokens g     (draft: 1024 + c)
          mma_nv(d[1][nt], af, r[1], r[3]);  // tokens g + 8 (draft: 1024 + 16 c)
        }
      }
      const float4 vz0 = vps4[mt * 8 + t4], vz1 = vps4[mt * 8 + 4 + t4];
      uint32_t bph[NT][2], bpl[NT][2];
      bool resc[NT];
      float al0[NT], al1[NT];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const float2 bb = *reinterpret_cast<const float2*>(bias + (bl * NQ + nt * 8 + g) * 2);
        float sv[2][2];  // [token half][token 2t + e]
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const float raw = d[j][nt][e] + d[j][nt][e + 2];  // rows g (hi) + g+8 (lo) of query g
            sv[j][e] = (TGT || j == 0) ? (raw + bb.x) * sl2 : fmaf(raw, 0.0625f, bb.y) * sl2;
          }
        float mx = fmaxf(fmaxf(sv[0][0], sv[0][1]), fmaxf(sv[1][0], sv[1][1]));
        float alpha = 1.0f;
        // lazy reference max (softmax_update): a query's reference rises only when its max runs
        // 2^QS_LAZY_MAX_LOG2 past it -- decided per query (quad max), the same rule in every
        // instantiation, so a row's result does not depend on the rows sharing the launch; the
        // quad max is skipped when no lane of the warp gets there (not in the parked wide-query
        // path, where that test measured 3% slower)
        const bool upd = QS_LAZY_MAX_LOG2 == 0 || C::PARK ||
                         __any_sync(0xffffffffu, mx > st[nt].m + (float)QS_LAZY_MAX_LOG2);
        if (upd) {
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
          mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
          if (mx > st[nt].m + (float)QS_LAZY_MAX_LOG2) {
            alpha = ex2_approx(st[nt].m - mx);  // st.m == -inf -> 0
            st[nt].l *= alpha;
            st[nt].z *= alpha;
            st[nt].ps *= alpha;
            st[nt].m = mx;
          }
        }
        // the accumulator columns of query q = nt*8 + 2t + e live in this lane; its alpha in lanes g = q
        if constexpr (C::PARK) {
          resc[nt] = upd && __any_sync(0xffffffffu, alpha != 1.0f);
          al0[nt] = al1[nt] = 1.0f;
          if (resc[nt]) {
            al0[nt] = __shfl_sync(0xffffffffu, alpha, 8 * t4);
            al1[nt] = __shfl_sync(0xffffffffu, alpha, 8 * t4 + 4);
          }
        } else if (upd && __any_sync(0xffffffffu, alpha != 1.0f)) {
          const float a0 = __shfl_sync(0xffffffffu, alpha, 8 * t4);
          const float a1 = __shfl_sync(0xffffffffu, alpha, 8 * t4 + 4);
#pragma unroll
          for (int cm = 0; cm < KS; ++cm) {
            acc[cm][nt][0] *= a0;
            acc[cm][nt][1] *= a1;
            acc[cm][nt][2] *= a0;
            acc[cm][nt][3] *= a1;
          }
        }
        const float m = st[nt].m;
        const float p00 = ex2_approx(sv[0][0] - m), p01 = ex2_approx(sv[0][1] - m);
        const float p10 = ex2_approx(sv[1][0] - m), p11 = ex2_approx(sv[1][1] - m);
        st[nt].l += (p00 + p01) + (p10 + p11);
        st[nt].z += (p00 * vz0.y + p01 * vz0.w) + (p10 * vz1.y + p11 * vz1.w);
        const float v00 = p00 * (vz0.x * kvs), v01 = p01 * (vz0.z * kvs);
        const float v10 = p10 * (vz1.x * kvs), v11 = p11 * (vz1.z * kvs);
        const __half2 h0 = __floats2half2_rn(v00, v01), h1 = __floats2half2_rn(v10, v11);
        const float2 f0 = __half22float2(h0), f1 = __half22float2(h1);
        float psum = (f0.x + f0.y) + (f1.x + f1.y);
        bph[nt][0] = h2_as_u32(h0);
        bph[nt][1] = h2_as_u32(h1);
        if constexpr (TGT && QS_TGT_PLO) {
          const __half2 l0 = __floats2half2_rn(v00 - f0.x, v01 - f0.y), l1 = __floats2half2_rn(v10 - f1.x, v11 - f1.y);
          const float2 g0 = __half22float2(l0), g1 = __half22float2(l1);
          psum += (g0.x + g0.y) + (g1.x + g1.y);
          bpl[nt][0] = h2_as_u32(l0);
          bpl[nt][1] = h2_as_u32(l1);
        }
        st[nt].ps += psum;
      }
      // ---- P.V: A = V^T codes [channels x tokens] of this token tile ----
      uint32_t vw[KS], vwl[KS];
      load_words<KS>(reinterpret_cast<const uint32_t*>(sp + C::PLANE_CHUNK), mt, lane, vw);
      if constexpr (TGT) load_words<KS>(reinterpret_cast<const uint32_t*>(sp + 3 * C::PLANE_CHUNK), mt, lane, vwl);
      if constexpr (C::PARK) {
        // per query tile: accumulators TMEM -> registers, rescale, the tile's MMAs, back to TMEM
        // (the same operations in the same order as the register-resident NT = 1 path)
        uint32_t va[KS][4];
#pragma unroll
        for (int cm = 0; cm < KS; ++cm) unpack_u4l4_raw(vw[cm], vwl[cm], va[cm]);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          float aw[32];
          tmem_ld32(tacc + nt * 32, aw);
          if (resc[nt]) {
#pragma unroll
            for (int cm = 0; cm < KS; ++cm) {
              aw[cm * 4 + 0] *= al0[nt];
              aw[cm * 4 + 1] *= al1[nt];
              aw[cm * 4 + 2] *= al0[nt];
              aw[cm * 4 + 3] *= al1[nt];
            }
          }
#pragma unroll
          for (int cm = 0; cm < KS; ++cm) {
            float (&a4)[4] = *reinterpret_cast<float(*)[4]>(aw + cm * 4);
            mma_nv(a4, va[cm], bph[nt][0], bph[nt][1]);
            if constexpr (QS_TGT_PLO) mma_nv(a4, va[cm], bpl[nt][0], bpl[nt][1]);
          }
          tmem_st32(tacc + nt * 32, aw);
        }
      } else {
#pragma unroll
        for (int cm = 0; cm < KS; ++cm) {
          uint32_t a[4];
          if constexpr (TGT) unpack_u4l4_raw(vw[cm], vwl[cm], a);
          else unpack_u4_raw(vw[cm], a);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) {
            mma_nv(acc[cm][nt], a, bph[nt][0], bph[nt][1]);
            if constexpr (TGT && QS_TGT_PLO) mma_nv(acc[cm][nt], a, bpl[nt][0], bpl[nt][1]);
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_b[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  }
  } else {
  // ======================= consumer warps =======================
  // Warp w owns the TPW consecutive 16-token tiles w*TPW .. w*TPW+TPW-1 of every chunk: their
  // Q.K^T chains interleave and share the query fragments' shared-memory loads, one online-softmax
  // update covers all of them, and the warp's per-chunk bookkeeping (barrier wait, shuffles,
  // release) is paid once per TPW tiles.
  constexpr int TP = C::TPW;
  const float sl2 = P.sm_scale_log2;
  // P' feeds P.V as f16 hi parts only (the lo columns stay zero): |error| <= 2^-12 |p'|, inside
  // the draft's fp16-level tolerance, and one split fewer per score
  const bool share_blk = TP == 1 || G >= 16 * TP;  // all of the warp's tiles in one (S,Z) block
  for (int i = 0, s = 0, ph = 0; i < nchunk; ++i) {
    const uint8_t* sp = stage_ptr(s);
    attn_wait(&full_b[s], ph);  // folded query fragments + biases (the fold waited for the whole stage)
    bool live[TP];
    int bl[TP];
#pragma unroll
    for (int k = 0; k < TP; ++k) {
      const int mt = warp * TP + k;
      live[k] = mt * 16 + i * QS_CHUNK_Q < tok_left && !(P.dbg & 1);  // tiles are whole: G is a multiple of 16
      bl[k] = (mt * 16) >> lgG;
    }
    if (live[0]) {  // live[k] implies live[k - 1]
      // ---- Q.K^T: A = K codes [tokens x channels], two accumulator chains per tile ----
      float d[TP][2][NT][4];
#pragma unroll
      for (int k = 0; k < TP; ++k)
#pragma unroll
        for (int j = 0; j < 2; ++j)
#pragma unroll
          for (int nt = 0; nt < NT; ++nt)
#pragma unroll
            for (int e = 0; e < 4; ++e) d[k][j][nt][e] = 0.f;
      // a dead second tile (partial last chunk) reads finite codes and is masked to -inf below
      uint32_t wu[TP][KS], wl[TP][KS];
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        load_words<KS>(reinterpret_cast<const uint32_t*>(sp), warp * TP + k, lane, wu[k]);
        if constexpr (TGT) load_words<KS>(reinterpret_cast<const uint32_t*>(sp + 2 * C::PLANE_CHUNK), warp * TP + k, lane, wl[k]);
      }
      const uint2* bq = reinterpret_cast<const uint2*>(sp + C::BQ_OFF) + lane;
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) {
          const uint2 b0 = bq[((size_t)bl[0] * KS * NT + ks * NT + nt) * 32];
#pragma unroll
          for (int k = 0; k < TP; ++k) {
            uint2 b = b0;
            if (k > 0 && !share_blk) b = bq[((size_t)bl[k] * KS * NT + ks * NT + nt) * 32];
            uint32_t a[4];
            if constexpr (TGT) unpack_u4l4_raw(wu[k][ks], wl[k][ks], a);
            else unpack_u4_raw(wu[k][ks], a);
            mma_nv(d[k][ks & 1][nt], a, b.x, b.y);
          }
        }
      }
      const float* bias = reinterpret_cast<const float*>(sp + C::BIAS_OFF);
      const float2* vps = reinterpret_cast<const float2*>(sp + C::VP_OFF);
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        float sv[2 * TP], p[2 * TP];
        float2 sz[TP][2];
#pragma unroll
        for (int k = 0; k < TP; ++k) {
          const int mt = warp * TP + k;
          const float2 bb = *reinterpret_cast<const float2*>(bias + (bl[k] * NQ + nt * 4 + t4) * 2);
          sz[k][0] = vps[mt * 16 + g];
          sz[k][1] = vps[mt * 16 + g + 8];
          const float r0 = (d[k][0][nt][0] + d[k][0][nt][1]) + (d[k][1][nt][0] + d[k][1][nt][1]);
          const float r1 = (d[k][0][nt][2] + d[k][0][nt][3]) + (d[k][1][nt][2] + d[k][1][nt][3]);
          sv[2 * k] = live[k] ? (r0 + bb.x) * sl2 : kNegInf;
          sv[2 * k + 1] = live[k] ? (TGT ? (r1 + bb.y) : fmaf(r1, 0.0625f, bb.y)) * sl2 : kNegInf;
        }
        const float alpha = softmax_update<2 * TP, (QS_LAZY_MAX_LOG2 > 0)>(st[nt], sv, p);
        if (alpha != 1.0f) rescale<KS, NT>(acc, nt, alpha);
#pragma unroll
        for (int k = 0; k < TP; ++k) {
          __half* prow = pw + k * C::PW_HALVES + (nt * 8 + 2 * t4) * PSTRIDE;
          if (k > 0 && !live[k]) {  // dead tile: p' = 0 feeds its (finite) codes
            prow[g] = prow[g + 8] = __float2half_rn(0.f);
            continue;
          }
          st[nt].l += p[2 * k] + p[2 * k + 1];
          st[nt].z += p[2 * k] * sz[k][0].y + p[2 * k + 1] * sz[k][1].y;
          const __half h0 = __float2half_rn(p[2 * k] * (sz[k][0].x * kvs));
          const __half h1 = __float2half_rn(p[2 * k + 1] * (sz[k][1].x * kvs));
          st[nt].ps += __half2float(h0) + __half2float(h1);
          prow[g] = h0;
          prow[g + 8] = h1;
        }
      }
      __syncwarp();
      // ---- P.V: A = V^T codes [channels x tokens] of each tile's token k-step ----
      uint32_t bpv[TP][NT][2];
#pragma unroll
      for (int k = 0; k < TP; ++k) get_pv_b<NT>(pw + k * C::PW_HALVES, g, t4, bpv[k]);
#pragma unroll
      for (int k = 0; k < TP; ++k) {
        uint32_t vw[KS], vwl[KS];
        load_words<KS>(reinterpret_cast<const uint32_t*>(sp + C::PLANE_CHUNK), warp * TP + k, lane, vw);
        if constexpr (TGT) load_words<KS>(reinterpret_cast<const uint32_t*>(sp + 3 * C::PLANE_CHUNK), warp * TP + k, lane, vwl);
#pragma unroll
        for (int cm = 0; cm < KS; ++cm) {
          uint32_t a[4];
          if constexpr (TGT) unpack_u4l4_raw(vw[cm], vwl[cm], a);
          else unpack_u4_raw(vw[cm], a);
#pragma unroll
          for (int nt = 0; nt < NT; ++nt) mma_nv(acc[cm][nt], a, bpv[k][nt][0], bpv[k][nt][1]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty_b[s]);
    if (++s == S) {
      s = 0;
      ph ^= 1;
    }
  }
  }
}

// Per-warp merge rows of the quantised path (query q = nt*8 + g holds the softmax state;
// accumulator columns are queries nt*8 + 2t + e).  P.V offsets: draft rows g carried
// (1024 + c) p' and rows g+8 (1024 + 16c) p'; target rows carried (1032 + 16 c_u + c_l) p'.
template <typename C, int HD, int NT, int MODE>
__device__ __forceinline__ void merge_rows_quant(float* mrg, const Softmax (&st)[NT], const float (&acc)[C::KS][NT][4],
                                                 bool offsets, uint32_t tacc = 0) {
  constexpr int KS = C::KS, NQ = C::NQ, MS = C::MS;
  constexpr bool TGT = MODE == MODE_QTARGET;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    float l = st[nt].l, z = st[nt].z, ps = st[nt].ps;
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
      z += __shfl_xor_sync(0xffffffffu, z, o);
      ps += __shfl_xor_sync(0xffffffffu, ps, o);
    }
    float* row = mrg + (warp * NQ + nt * 8 + g) * MS;
    if (t4 == 0) {
      row[0] = st[nt].m;
      row[1] = l;
      row[2] = z;
      row[3] = ps;
    }
  }
  __syncwarp();
  // (fp16 tails: plain values, no offsets)
  const float og = offsets ? (TGT ? 1032.f : 1024.f) : 0.f, og8 = offsets ? (TGT ? 1032.f : 64.f) : 0.f;
  const float sc8 = (offsets && !TGT) ? 0.0625f : 1.0f;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    float aw[32];
    if constexpr (C::PARK) {
      tmem_ld32(tacc + nt * 32, aw);  // parked accumulators (wide-query verify; TMEM address 0 is valid)
    } else {
#pragma unroll
      for (int cm = 0; cm < KS; ++cm)
#pragma unroll
        for (int e = 0; e < 4; ++e) aw[cm * 4 + e] = acc[cm][nt][e];
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      float* row = mrg + (warp * NQ + nt * 8 + 2 * t4 + e) * MS;
      const float z = row[2], ps = row[3];
#pragma unroll
      for (int cm = 0; cm < KS; ++cm) {
        row[4 + cm * 16 + g] = (aw[cm * 4 + e] - og * ps) + z;
        row[4 + cm * 16 + g + 8] = fmaf(aw[cm * 4 + e + 2], sc8, -og8 * ps) + z;
      }
    }
  }
}

// per-warp merge rows of the hi/lo column-pair layout (query q = nt*4 + t): the fp16
// regions, and the draft's quantised region with its P.V offsets (rows g carried
// (1024 + c) p', rows g+8 (1024 + 16c) p')
template <typename C, int HD, int NTO, int MODE>
__device__ __forceinline__ void merge_rows_fp(float* mrg, const Softmax (&st)[NTO], const float (&acc)[C::KS][NTO][4],
                                              bool offsets) {
  constexpr int KS = C::KS, NQ = C::NQ, MS = C::MS;
  constexpr bool TGT = MODE == MODE_QTARGET;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int nt = 0; nt < NTO; ++nt) {
    float l = st[nt].l, z = st[nt].z, ps = st[nt].ps;
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l += __shfl_xor_sync(0xffffffffu, l, o);
      z += __shfl_xor_sync(0xffffffffu, z, o);
      ps += __shfl_xor_sync(0xffffffffu, ps, o);
    }
    float* row = mrg + (warp * NQ + nt * 4 + t4) * MS;
    if (g == 0) {
      row[0] = st[nt].m;
      row[1] = l;
    }
    const float off_g = offsets ? (TGT ? 1032.f : 1024.f) * ps : 0.f;
    const float off_g8 = offsets ? (TGT ? 1032.f : 64.f) * ps : 0.f;
    const float sc8 = (offsets && !TGT) ? 0.0625f : 1.0f;
#pragma unroll
    for (int cm = 0; cm < KS; ++cm) {
      row[4 + cm * 16 + g] = ((acc[cm][nt][0] + acc[cm][nt][1]) - off_g) + z;
      row[4 + cm * 16 + g + 8] = fmaf(acc[cm][nt][2] + acc[cm][nt][3], sc8, -off_g8) + z;
    }
  }
}

// ---------------------------------------------------------------------------
// the kernel
// ---------------------------------------------------------------------------
template <int HD, int NT, int MODE, int QR>
__global__ void __launch_bounds__(AttnCfg<HD, NT, MODE, QR>::THREADS) __maxnreg__((AttnCfg<HD, NT, MODE, QR>::MAXREG))
    attn_kernel(const __grid_constant__ AttnParams P) {
  using C = AttnCfg<HD, NT, MODE, QR>;
  constexpr int KS = C::KS, NQ = C::NQ, NCW = C::NCW, NTH = C::THREADS;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* region = smem;
  uint32_t* bqf = reinterpret_cast<uint32_t*>(smem + C::REGION);      // [KS][NT][32][2]
  float* q_s = reinterpret_cast<float*>(bqf + C::BQF_WORDS);          // [NQ][HD]
  __half* pw_all = reinterpret_cast<__half*>(q_s + NQ * HD);           // [NCW][PW_HALVES]
  // tma[8] full[8] empty[8] tma_params[8] (the row-query kernels have no P transpose buffers)
  uint64_t* bars = reinterpret_cast<uint64_t*>(C::ROWQ ? reinterpret_cast<__half*>(q_s + NQ * HD) : pw_all + NCW * C::PW_WARP);
  int* ticket_s = reinterpret_cast<int*>(bars + 32);  // [0] split ticket, [2] TMEM base (PARK)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int seq = blockIdx.z;
  const int head = blockIdx.x / P.n_qgroups, qg = blockIdx.x % P.n_qgroups;
  const int split = blockIdx.y;
  const int n_main = P.n_main;
  const int n_split_tot = n_main + 2;
  const int nq = min(NQ, P.n_queries - qg * NQ);
  __half* pw = pw_all + min(warp, NCW - 1) * C::PW_WARP;

  if constexpr (C::QUANT && !C::ROWQ) {
    for (int i = tid; i < NCW * C::PW_WARP / 2; i += NTH) reinterpret_cast<uint32_t*>(pw_all)[i] = 0u;
  }
  if constexpr (C::QUANT) {
    // per-stage B fragment buffers: the unused query columns stay zero
    for (int s = 0; s < C::NSTAGE; ++s) {
      uint32_t* bq = reinterpret_cast<uint32_t*>(region + s * C::QSTAGE + C::BQ_OFF);
      for (int i = tid; i < C::BQ_WORDS + C::BIAS_FLOATS; i += NTH) bq[i] = 0u;  // fragments + biases
    }
  }
  if (tid == 0) {
    for (int i = 0; i < 8; ++i) {
      mbar_init(&bars[i], 1);         // TMA transactions
      mbar_init(&bars[8 + i], 1);     // producer (one warp per chunk) -> consumers
      mbar_init(&bars[16 + i], NCW);  // consumers -> producer
      mbar_init(&bars[24 + i], 1);    // TMA transactions of the (S, Z) params
    }
    fence_mbar_init();
  }

  // ---- region of this CTA (lengths are not written by the previous kernel: QKV linear) ----
  const int fp1_len = P.fp1_len ? P.fp1_len[seq] : 0;
  const int fp2_base = P.fp2_len ? P.fp2_len[seq] + P.row_offset : 0;
  int region_kind;  // 0 quant, 1 fp16 main, 2 fp1, 3 fp2
  int n_tok = 0, c_begin = 0, c_end = 0, causal = 0;
  const __half* fk = nullptr;
  const __half* fv = nullptr;
  if (split < n_main) {
    if constexpr (!C::QUANT) {
      region_kind = 1;
      if (P.main_is_fpcache) {
        n_tok = P.fp_len[seq] + P.row_offset + P.T;
        causal = 1;
      } else {
        n_tok = P.n_blocks[seq] * P.G;
      }
      const int nch = (n_tok + C::CF - 1) / C::CF;
      const int cps = P.main_is_fpcache ? P.fpcache_cps : (nch + n_main - 1) / n_main;
      c_begin = split * cps;
      c_end = min(nch, c_begin + cps);
      const size_t hoff = (size_t)seq * P.main_seq_stride + (size_t)head * P.main_head_stride;
      fk = reinterpret_cast<const __half*>(P.main_k) + hoff;
      fv = reinterpret_cast<const __half*>(P.main_v) + hoff;
    } else {
      region_kind = 0;
      n_tok = P.n_blocks[seq] * P.G;
      const int nch = (n_tok + QS_CHUNK_Q - 1) / QS_CHUNK_Q;
      const int cps = (nch + n_main - 1) / n_main;
      c_begin = split * cps;
      c_end = min(nch, c_begin + cps);
    }
  } else {
    const bool is1 = split == n_main;
    region_kind = is1 ? 2 : 3;
    n_tok = is1 ? fp1_len : fp2_base + P.T;
    causal = is1 ? 0 : 1;
    const size_t hoff = (size_t)seq * P.fp_seq_stride + (size_t)head * P.fp_rows * HD;
    const void* bk = is1 ? P.fp1_k : P.fp2_k;
    const void* bv = is1 ? P.fp1_v : P.fp2_v;
    fk = bk ? reinterpret_cast<const __half*>(bk) + hoff : nullptr;
    fv = bv ? reinterpret_cast<const __half*>(bv) + hoff : nullptr;
    c_begin = 0;
    c_end = fk ? (n_tok + C::CF - 1) / C::CF : 0;
  }
  // diagnostics (profiles/attn_micro.py): 4 = the fp tail CTAs skip their chunks, 8 = the main ones do
  if ((P.dbg & 4) && split >= n_main) c_end = c_begin;
  if ((P.dbg & 8) && split < n_main) c_end = c_begin;

  uint32_t tacc = 0;  // this consumer warp's parked accumulators (TMEM lane quarter + column block)
  if constexpr (C::PARK) {
    if (warp == 0) tmem_alloc(reinterpret_cast<uint32_t*>(ticket_s + 2), C::TMEM_COLS);
    tmem_fence_before();
  }
  __syncthreads();  // barriers initialised, fragment buffers zeroed, TMEM allocated
  if constexpr (C::PARK) {
    tmem_fence_after();
    if (warp < NCW) {
      tacc = reinterpret_cast<const uint32_t*>(ticket_s)[2] + ((uint32_t)(32 * (warp & 3)) << 16) +
             (uint32_t)((warp >> 2) * NT * 32);
      float z[32];
#pragma unroll
      for (int i = 0; i < 32; ++i) z[i] = 0.f;
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) tmem_st32(tacc + nt * 32, z);
    }
  }
  if constexpr (C::QUANT) {
    // PDL: the first ring stages of packed planes stream in before the grid dependency resolves
    if (region_kind == 0 && warp == NCW && lane == 0)
      for (int i = 0; i < C::NSTAGE && i < c_end - c_begin; ++i)
        quant_issue<C, HD, MODE>(P, region, bars, seq, head, P.n_blocks[seq], c_begin, i, c_end - c_begin);
  }
  pdl_wait();
  pdl_trigger();
  for (int i = tid; i < NQ * HD; i += NTH) {
    const int q = i / HD, c = i % HD;
    float v = 0.f;
    if (q < nq) {
      const int qgl = qg * NQ + q;
      const int t = qgl / P.r, j = qgl - t * P.r;
      v = P.q[((size_t)seq * P.T + t) * P.q_row_stride + (size_t)(head * P.r + j) * HD + c];
    }
    q_s[i] = v;
  }
  __syncthreads();

  constexpr int MS = C::MS;
  float* mrg = reinterpret_cast<float*>(region);  // [NCW][NQ][MS]: m, l, z, ps, acc[HD]  (after the regions)
  if (region_kind == 0) {
    if constexpr (C::QUANT) {
      Softmax st[NT];
      float acc[KS][NT][4];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        st[nt] = {kNegInf, 0.f, 0.f, 0.f};
#pragma unroll
        for (int a = 0; a < KS; ++a)
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[a][nt][e] = 0.f;
      }
      if (c_end > c_begin)
        quant_region<C, HD, NT, MODE>(region, bars, q_s, pw, nq, seq, head, n_tok, c_begin, c_end, P, st, acc, tacc);
      __syncthreads();
      if (warp < NCW) {
        if constexpr (C::ROWQ) merge_rows_quant<C, HD, NT, MODE>(mrg, st, acc, true, tacc);
        else merge_rows_fp<C, HD, NT, MODE>(mrg, st, acc, true);
      }
    }
  } else if constexpr (C::ROWQ) {
    Softmax st[NT];
    float acc[KS][NT][4];
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      st[nt] = {kNegInf, 0.f, 0.f, 0.f};
#pragma unroll
      for (int a = 0; a < KS; ++a)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[a][nt][e] = 0.f;
    }
    if (c_end > c_begin)
      fp16_region_q<C, HD, NT>(region, bqf, q_s, nq, fk, fv, n_tok, c_begin, c_end, causal, qg, P, st, acc, tacc);
    __syncthreads();
    if (warp < NCW) merge_rows_quant<C, HD, NT, MODE>(mrg, st, acc, false, tacc);
  } else {
    constexpr int NTO = C::NTO;
    Softmax st[NTO];
    float acc[KS][NTO][4];
#pragma unroll
    for (int nt = 0; nt < NTO; ++nt) {
      st[nt] = {kNegInf, 0.f, 0.f, 0.f};
#pragma unroll
      for (int a = 0; a < KS; ++a)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[a][nt][e] = 0.f;
    }
    if (c_end > c_begin) fp16_region<C, HD, NTO>(region, bqf, q_s, pw, nq, fk, fv, n_tok, c_begin, c_end, causal, qg, P, st, acc);
    __syncthreads();
    if (warp < NCW) merge_rows_fp<C, HD, NTO, MODE>(mrg, st, acc, false);
  }
  if constexpr (C::PARK) tmem_fence_before();
  __syncthreads();
  if constexpr (C::PARK) {
    if (warp == 0) {
      tmem_fence_after();
      tmem_dealloc(reinterpret_cast<const uint32_t*>(ticket_s)[2], C::TMEM_COLS);
    }
  }
  const size_t hidx = ((size_t)seq * P.Hkv + head) * P.n_qgroups + qg;
  float* part = P.partials + (hidx * n_split_tot + split) * (size_t)NQ * (HD + 2);
  for (int i = tid; i < nq * (HD + 2); i += NTH) {
    const int q = i / (HD + 2), c = i - q * (HD + 2);
    float mx = kNegInf;
#pragma unroll
    for (int w = 0; w < NCW; ++w) mx = fmaxf(mx, mrg[(w * NQ + q) * MS]);
    float v = 0.f;
    if (c == 0) {
      v = mx;
    } else if (mx != kNegInf) {
#pragma unroll
      for (int w = 0; w < NCW; ++w) {
        const float* row = mrg + (w * NQ + q) * MS;
        v += exp2f(row[0] - mx) * (c == 1 ? row[1] : row[4 + c - 2]);
      }
    }
    part[i] = v;
  }
  __syncthreads();  // every partial store before thread 0's release-acquire ticket (cumulative)
  if (tid == 0) *ticket_s = atom_add_acq_rel_gpu(&P.counters[hidx], 1);
  __syncthreads();
  if (*ticket_s != n_split_tot - 1) return;
  // ===================== last CTA of the head: merge splits in fixed order =====================
  const float* allp = P.partials + hidx * n_split_tot * (size_t)NQ * (HD + 2);
  // KV-head sharding: this layer's gather buffers (parity of the layers consumed so far)
  const qs_gather_args& GA = P.gather;
  const unsigned epoch0 = GA.world ? __ldcg(GA.epoch) : 0u;
  const int gpar = GA.world ? (int)((epoch0 / (unsigned)GA.arrivals) & 1u) : 0;
  // all lanes run every round (whole 16-channel groups are valid or not together) so the
  // optional f16 copy + 16-sums for the output projection can reduce with shuffles
  for (int base = 0; base < nq * HD; base += NTH) {
    const int i = base + tid;
    const bool valid = i < nq * HD;
    const int q = valid ? i / HD : 0, c = i % HD;
    float o = 0.f;
    if (valid) {
      // every split's (m, l, acc[c]) requested at once, 16 splits per round (one L2 round trip
      // per round instead of one per split); combined in split order
      float mx = kNegInf;
      for (int s0 = 0; s0 < n_split_tot; s0 += 16) {
        float mv[16];
#pragma unroll
        for (int j = 0; j < 16; ++j)
          mv[j] = s0 + j < n_split_tot ? __ldcg(allp + ((size_t)(s0 + j) * NQ + q) * (HD + 2)) : kNegInf;
#pragma unroll
        for (int j = 0; j < 16; ++j) mx = fmaxf(mx, mv[j]);
      }
      float num = 0.f, den = 0.f;
      if (mx != kNegInf) {
        for (int s0 = 0; s0 < n_split_tot; s0 += 16) {
          float mv[16], lv[16], av[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const bool ok = s0 + j < n_split_tot;
            const float* pr = allp + ((size_t)(s0 + j) * NQ + q) * (HD + 2);
            mv[j] = ok ? __ldcg(pr) : kNegInf;
            lv[j] = ok ? __ldcg(pr + 1) : 0.f;
            av[j] = ok ? __ldcg(pr + 2 + c) : 0.f;
          }
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            if (s0 + j < n_split_tot) {
              const float f = exp2f(mv[j] - mx);
              den += f * lv[j];
              num += f * av[j];
            }
          }
        }
      }
      o = den > 0.f ? num / den : 0.f;
    }
    const int qgl = qg * NQ + q;
    const int t = qgl / P.r, j = qgl - t * P.r;
    const size_t row = (size_t)seq * P.T + t;
    const size_t col = (size_t)(head * P.r + j) * HD + c;
    if (valid) P.out[row * P.q_row_stride + col] = o;
    if (P.out_h) {
      const __half h = __float2half_rn(o);
      float sm16 = __half2float(h);
#pragma unroll
      for (int off = 1; off < 16; off <<= 1) sm16 += __shfl_xor_sync(0xffffffffu, sm16, off);
      if (valid) {
        if (GA.world) {
          // fused all-gather: this head's row goes to every rank's gather buffer (P2P stores)
          const size_t gcol = (size_t)GA.q_col_offset + col;
          for (int rk = 0; rk < GA.world; ++rk) {
            reinterpret_cast<__half*>(GA.gh[rk])[gpar * GA.par_stride_h + row * P.ld_out_h + gcol] = h;
            if ((c & 15) == 0) GA.gs[rk][gpar * GA.par_stride_s + row * P.ld_out_s + gcol / 16] = sm16;
          }
        } else {
          reinterpret_cast<__half*>(P.out_h)[row * P.ld_out_h + col] = h;
          if ((c & 15) == 0) P.out_s[row * P.ld_out_s + col / 16] = sm16;
        }
      }
    }
  }
  if (tid == 0) P.counters[hidx] = 0;
  if (GA.world) {
    // signal every rank (release, system scope: the rows above are visible before the count),
    // then the CTA finishing this rank's last local merge waits for the whole layer
    __syncthreads();
    const int nloc = (int)(gridDim.x * gridDim.z);
    if (tid == 0) {
      __threadfence_system();
      for (int rk = 0; rk < GA.world; ++rk) red_release_sys_add(GA.flag[rk], 1u);
      *ticket_s = atomicAdd(GA.done, 1);
      if (*ticket_s == nloc - 1) {
        const unsigned target = epoch0 + (unsigned)GA.arrivals;
        while ((int)(ld_acquire_sys(GA.flag[GA.rank]) - target) < 0) __nanosleep(64);
      }
    }
    __syncthreads();
    if (*ticket_s != nloc - 1) return;
    // every rank's rows of this layer are in: hand the full row set to the output projection
    const int rows = P.B * P.T;
    const int nh = (int)(P.ld_out_h / 8), ns = (int)(P.ld_out_s / 4);  // uint4 / float4 per row
    const uint4* gh = reinterpret_cast<const uint4*>(reinterpret_cast<const __half*>(GA.gh[GA.rank]) + gpar * GA.par_stride_h);
    const float4* gs = reinterpret_cast<const float4*>(GA.gs[GA.rank] + gpar * GA.par_stride_s);
    for (int i = tid; i < rows * nh; i += NTH) reinterpret_cast<uint4*>(P.out_h)[i] = __ldcg(gh + i);
    for (int i = tid; i < rows * ns; i += NTH) reinterpret_cast<float4*>(P.out_s)[i] = __ldcg(gs + i);
    __syncthreads();
    if (tid == 0) {
      *GA.epoch = epoch0 + (unsigned)GA.arrivals;
      *GA.done = 0;
    }
  }
}

template <int HD, int NT, int MODE, int QR>
static cudaError_t launch_attn_t(const AttnParams& p, cudaStream_t stream) {
  using C = AttnCfg<HD, NT, MODE, QR>;
  auto kern = attn_kernel<HD, NT, MODE, QR>;
  static bool configured = false;
  if (!configured) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM);
    if (e != cudaSuccess) return e;
    configured = true;
  }
  dim3 grid(p.Hkv * p.n_qgroups, p.n_main + 2, p.B);
  return launch_pdl(kern, grid, dim3(C::THREADS), C::SMEM, stream, p);
}

// query rows stored per CTA for `per` query columns (quantised, one query tile)
static inline int attn_qr(int per) { return per <= 1 ? 1 : per <= 2 ? 2 : per <= 4 ? 4 : 8; }

template <int HD, int MODE>
static cudaError_t launch_attn_nt(const AttnParams& p, int nt, int per, cudaStream_t s) {
  if constexpr (MODE == MODE_FP16) {
    switch (nt) {
      case 1: return launch_attn_t<HD, 1, MODE, 8>(p, s);
      case 2: return launch_attn_t<HD, 2, MODE, 8>(p, s);
      case 3: return launch_attn_t<HD, 3, MODE, 8>(p, s);
      default: return cudaErrorInvalidValue;
    }
  } else if constexpr (MODE == MODE_QDRAFT) {
    switch (nt) {
      case 1:  // the fold computes only the live query slots (MHA: one)
        switch (attn_qr(per)) {
          case 1: return launch_attn_t<HD, 1, MODE, 1>(p, s);
          case 2: return launch_attn_t<HD, 1, MODE, 2>(p, s);
          default: return launch_attn_t<HD, 1, MODE, 8>(p, s);
        }
      case 2: return launch_attn_t<HD, 2, MODE, 8>(p, s);
      case 3: return launch_attn_t<HD, 3, MODE, 8>(p, s);
      default: return cudaErrorInvalidValue;
    }
  } else {
    if (nt == 2) return launch_attn_t<HD, 2, MODE, 8>(p, s);
    if (nt == 3) return launch_attn_t<HD, 3, MODE, 8>(p, s);
    if (nt != 1) return cudaErrorInvalidValue;
    switch (attn_qr(per)) {
      case 1: return launch_attn_t<HD, 1, MODE, 1>(p, s);
      case 2: return launch_attn_t<HD, 1, MODE, 2>(p, s);
      case 4: return launch_attn_t<HD, 1, MODE, 4>(p, s);
      default: return launch_attn_t<HD, 1, MODE, 8>(p, s);
    }
  }
}

template <int MODE>
static cudaError_t launch_attn_hd(const AttnParams& p, int nt, int per, cudaStream_t s) {
  switch (p.hd) {
    case 16: return launch_attn_nt<16, MODE>(p, nt, per, s);
    case 32: return launch_attn_nt<32, MODE>(p, nt, per, s);
    case 64: return launch_attn_nt<64, MODE>(p, nt, per, s);
    case 128: return launch_attn_nt<128, MODE>(p, nt, per, s);
    default: return cudaErrorInvalidValue;
  }
}

cudaError_t launch_attention(const AttnParams& p, int mode, cudaStream_t s) {
  const int per = (p.n_queries + p.n_qgroups - 1) / p.n_qgroups;
  const int nt = attention_nt(per, mode);
  switch (mode) {
    case MODE_QDRAFT: return launch_attn_hd<MODE_QDRAFT>(p, nt, per, s);
    case MODE_QTARGET: return launch_attn_hd<MODE_QTARGET>(p, nt, per, s);
    case MODE_FP16: return launch_attn_hd<MODE_FP16>(p, nt, per, s);
    default: return cudaErrorInvalidValue;
  }
}

template <int HD, int NT, int MODE, int QR>
static int occ_t() {
  using C = AttnCfg<HD, NT, MODE, QR>;
  auto kern = attn_kernel<HD, NT, MODE, QR>;
  if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM) != cudaSuccess) return -1;
  int n = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, kern, C::THREADS, C::SMEM) != cudaSuccess) return -1;
  return n;
}

template <int HD, int MODE>
static int occ_h(int per) {
  const int nt = attention_nt(per, MODE);
  if constexpr (MODE == MODE_QDRAFT) {
    if (nt == 1) return attn_qr(per) == 1 ? occ_t<HD, 1, MODE, 1>() : attn_qr(per) == 2 ? occ_t<HD, 1, MODE, 2>()
                                                                                        : occ_t<HD, 1, MODE, 8>();
    return nt == 2 ? occ_t<HD, 2, MODE, 8>() : occ_t<HD, 3, MODE, 8>();
  } else if constexpr (MODE != MODE_QTARGET) {
    return nt == 1 ? occ_t<HD, 1, MODE, 8>() : nt == 2 ? occ_t<HD, 2, MODE, 8>() : occ_t<HD, 3, MODE, 8>();
  } else {
    if (nt == 2) return occ_t<HD, 2, MODE, 8>();
    if (nt == 3) return occ_t<HD, 3, MODE, 8>();
    switch (attn_qr(per)) {
      case 1: return occ_t<HD, 1, MODE, 1>();
      case 2: return occ_t<HD, 1, MODE, 2>();
      case 4: return occ_t<HD, 1, MODE, 4>();
      default: return occ_t<HD, 1, MODE, 8>();
    }
  }
}

template <int MODE>
static int occ_m(int hd, int per) {
  switch (hd) {
    case 16: return occ_h<16, MODE>(per);
    case 32: return occ_h<32, MODE>(per);
    case 64: return occ_h<64, MODE>(per);
    case 128: return occ_h<128, MODE>(per);
    default: return -1;
  }
}

// resident CTAs per SM of the launch serving `per` query columns per CTA
int attention_occupancy(int hd, int per, int mode) {
  switch (mode) {
    case MODE_QDRAFT: return occ_m<MODE_QDRAFT>(hd, per);
    case MODE_QTARGET: return occ_m<MODE_QTARGET>(hd, per);
    case MODE_FP16: return occ_m<MODE_FP16>(hd, per);
    default: return -1;
  }
}

}  // namespace qs
