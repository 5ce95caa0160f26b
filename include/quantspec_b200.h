/*
 * quantspec_b200.h -- C ABI of the B200 (sm_100a) QuantSpec decode hot path.
 *
 * The reference (arXiv 2502.10424, /root/reference/pkg/src/quantspec) has no
 * FFI: its boundary is a duck-typed Python protocol.  Each entry point below
 * names the reference function / method whose work it replaces (Q/ =
 * pkg/src/quantspec/).  INTEGRATION.md shows the ctypes binding.
 *
 * Conventions
 *   - every call returns qs_status (0 = OK); qs_last_error() gives the text.
 *   - every call is stream-ordered on the caller's cudaStream_t (passed as
 *     void*), performs no allocation and no host synchronisation.
 *   - all buffers are caller-owned device pointers; sizes are element counts.
 *   - status codes map onto the reference exception taxonomy Q/errors.py:4-33.
 */
#ifndef QUANTSPEC_B200_H
#define QUANTSPEC_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QS_OK = 0,
  QS_ERR_DIMENSION = 1, /* DimensionError        Q/errors.py:8  */
  QS_ERR_CONFIG = 2,    /* ConfigError           Q/errors.py:12 */
  QS_ERR_DATA = 3,      /* DataError             Q/errors.py:16 */
  QS_ERR_INTEGRITY = 4, /* CacheIntegrityError   Q/errors.py:24 */
  QS_ERR_OVERFLOW = 5,  /* BufferOverflowError   Q/errors.py:28 */
  QS_ERR_CUDA = 6       /* CUDA launch / runtime failure          */
} qs_status;

/* attention modes (view kinds of Q/model.py:351-356) */
enum { QS_VIEW_DRAFT = 0, QS_VIEW_TARGET = 1, QS_VIEW_FP16 = 2 };

/* linear-layer epilogues (the per-layer dataflow of Q/model.py:377-397) */
enum {
  QS_EPI_STORE = 0,    /* y = x @ W                                  */
  QS_EPI_ADD = 1,      /* out += x @ W    (residual add)             */
  QS_EPI_QKV = 2,      /* q/k RoPE (Q/tensor.py:65-82), q store, k/v append (Q/cache.py:216-234) */
  QS_EPI_SILU_MUL = 3  /* silu(x@Wg) * (x@Wu)  (Q/model.py:397)      */
};
enum { QS_W_F16 = 0, QS_W_INT4 = 1 };

/* KV-head sharding (the paper's 2-GPU long-context runs): one
 * sequence's KV heads are split over `world` ranks and every rank needs every head's attention
 * row for the replicated output projection.  Instead of an all-gather after the attention kernel,
 * the merge epilogue of each (head, query group) stores its f16 row + 16-sums straight into every
 * rank's gather buffer (NVLink P2P through CUDA IPC mappings, or plain pointers in one process)
 * and bumps every rank's arrival counter (release, system scope); the CTA finishing a rank's last
 * local merge waits (acquire) until all `arrivals` of the layer are in, copies the full row set to
 * the output projection's input (out_h / out_s) and advances the epoch.  The gather buffers
 * alternate by layer parity (epoch / arrivals), so a rank one layer ahead never overwrites rows a
 * slower rank has not consumed.  world = 0: off. */
#define QS_MAX_RANKS 8
typedef struct {
  int world, rank;
  int q_col_offset;                 /* this rank's first column (query head * hd) of the full row */
  int arrivals;                     /* head merges per layer over all ranks                         */
  int64_t par_stride_h;             /* halves between the two parity buffers of gh[i]               */
  int64_t par_stride_s;             /* floats between the two parity buffers of gs[i]               */
  void* gh[QS_MAX_RANKS];           /* rank i's gather rows: half [2][rows][ld_out_h]               */
  float* gs[QS_MAX_RANKS];          /* rank i's 16-sums: f32 [2][rows][ld_out_s]                    */
  unsigned* flag[QS_MAX_RANKS];     /* rank i's arrival counter (monotonic, wraps)                  */
  unsigned* epoch;                  /* this rank: arrivals consumed so far (advanced by the waiter) */
  int* done;                        /* this rank: merges finished in the current launch (zeroed)    */
} qs_gather_args;

/* Split-K flash-decode over the hierarchical store for one layer.
 * Replaces draft_view/target_view (Q/cache.py:309-378) + _merged_attention
 * (Q/model.py:176-195) for T query rows at once (Q/specdec.py:270-273). */
typedef struct {
  int B, Hkv, hd, G, T, r; /* r = query heads per kv head (1 = MHA) */
  int n_queries;           /* T * r                                   */
  int n_qgroups;           /* query-column groups (grid.y split)      */
  int n_main;              /* main-region splits per head             */
  int row_offset;          /* provisional rows already appended this cycle */
  int main_is_fpcache;     /* 1: main region is an fp16 cache (causal tail) */
  int fpcache_cps;         /* chunks per split for the fp16 cache       */
  float sm_scale_log2;     /* log2(e) / sqrt(hd)                        */
  const float* q;          /* [B][T][q_row_stride]                     */
  float* out;              /* [B][T][q_row_stride]                     */
  int64_t q_row_stride;
  const int* n_blocks;     /* [B] quantised blocks                     */
  const int* fp1_len;      /* [B]                                      */
  const int* fp2_len;      /* [B] committed fp2 rows                   */
  const int* fp_len;       /* [B] fp16-cache rows                      */
  /* quantised planes, layer base (seq 0) */
  const uint8_t *ku, *kl, *vu, *vl;
  int64_t plane_seq_stride, plane_head_stride; /* bytes */
  const void *kp, *vp;                         /* float2 (S,Z) */
  int64_t kp_seq_stride, kp_head_stride, vp_seq_stride, vp_head_stride; /* float2 units */
  /* fp16 main region (sensitive-layer archive or fp16 cache) */
  const void *main_k, *main_v; /* half */
  int64_t main_seq_stride, main_head_stride; /* halves */
  /* fp1 / fp2 recent-token buffers (half) [seq][layer][2][kv_head][fp_rows][hd] */
  const void *fp1_k, *fp1_v, *fp2_k, *fp2_v;
  int64_t fp_seq_stride; /* halves */
  int fp_rows;           /* rows per (buffer, head): G + slack for the ragged batch's junk rows */
  float* partials;       /* scratch */
  int* counters;         /* [B*Hkv*n_qgroups] zero-initialised */
  int dbg;               /* 0; diagnostic bits (1: skip consumer math, 2: skip producer fold) */
  /* optional fused hand-off to the output projection (the qs_prep_act layout, no norm):
   * f16 copy [B*T][ld_out_h] and f32 sums of every 16 f16 values [B*T][ld_out_s]; NULL = off */
  void* out_h;
  int64_t ld_out_h;
  float* out_s;
  int64_t ld_out_s;
  /* KV-head sharding: fused all-gather of the rows into out_h / out_s (needs out_h, out_s) */
  qs_gather_args gather;
} qs_attn_args;

/* x @ W with fused epilogue.  Replaces the fp32 `h @ W` products of
 * decode_step (Q/model.py:379-397) and, for QS_W_INT4, the dequantised f32
 * copies of quantize_model_weights (Q/model.py:141-168).  Persistent kernels:
 * one CTA per SM owns whole 32-row tile pairs over the full K range, so the
 * result of one activation row never depends on how many rows share the launch. */
typedef struct {
  int wmode;          /* QS_W_F16 | QS_W_INT4                       */
  int epi;            /* QS_EPI_*                                    */
  int N, K;           /* output rows (d_out), reduction (d_in)       */
  int ncols;          /* activation rows (B*T), 1..48                */
  int wgroup;         /* INT4 group size along d_in                  */
  const void* w;      /* frag16 halves or frag4 u32                  */
  const void* wparams;/* INT4: float4 {S_g,Z_g,S_g8,Z_g8} per (mtile,group,g) */
  const void* xh;     /* half [ncols][ldxh]: f16 activations (qs_prep_act) */
  int64_t ldxh;       /* halves, multiple of 8, >= K + 64             */
  const float* xs;    /* [ncols][ldxs] sums of 16 consecutive f16 activations */
  int64_t ldxs;       /* floats, multiple of 4, >= K/16 + 4           */
  float* y;           /* [ncols][ldy] output (STORE/ADD) or SILU f32 copy (may be NULL) */
  int64_t ldy;
  void* yh;           /* SILU: half [ncols][ldyh] prepared input of the next layer */
  int64_t ldyh;
  float* ys;          /* SILU: [ncols][ldys] 16-sums of yh           */
  int64_t ldys;
  /* QKV epilogue */
  int Nq, Nk, hd, T;  /* q rows, k rows (= v rows), head dim, rows per sequence */
  float* q_out;       /* [ncols][Nq]                                 */
  void *k_dst, *v_dst;/* half, head-major rows                       */
  int64_t kv_seq_stride, kv_head_stride; /* halves */
  const int* row_base;/* [B] first free row (fp2_len or fp16-cache len) */
  int row_offset;
  int row_cap;        /* rows per head of k_dst / v_dst: a row >= row_cap is not written (flag 4) */
  const int* pos_base;/* [B] position of row_base (seq_len)         */
  const void* rope;   /* float2 [max_pos][hd/2] (cos, sin)           */
  int max_pos;        /* a position >= max_pos sets flag 8 (ConfigError) and is not rotated */
  int* flags;         /* optional device status word (bit 4 overflow, bit 8 position) */
  int dbg;            /* 0; diagnostic bits (1: consumers skip the MMA work; 2, INT4 only: ALU ops replace the MMAs) */
  /* optional (both weight modes): build the f16 activations (+ 16-sums) inside the kernel from
   * f32 rows xf [ncols][ldxf] (RMS-normalised with `gain` when non-NULL, Q/tensor.py:35-42)
   * instead of reading xh / xs -- replaces a qs_prep_act launch with bit-identical inputs (the
   * same device routine); one row (ncols = 1), K <= 4096 */
  const float* xf;
  int64_t ldxf;
  const float* gain;
  float eps;
} qs_linear_args;

/* KV store descriptor (device pointers + geometry), Q/cache.py:42-133 */
typedef struct {
  int B, L, Hkv, hd, G, max_blocks;
  int fp_rows;                /* rows per (buffer, head) of fp_k / fp_v (>= G) */
  uint8_t *ku, *kl, *vu, *vl; /* [B][L][Hkv][max_blocks][G*hd/2]          */
  void *kp, *vp;              /* float2 [B][L][Hkv][max_blocks][hd or G]   */
  void *fp_k, *fp_v;          /* half [B][L][2][Hkv][fp_rows][hd]          */
  void *arch_k, *arch_v;      /* half [B][n_sens][Hkv][max_blocks*G][hd]   */
  uint64_t sens_mask[2];      /* bit l set: layer l is sensitive (archives fp16) */
} qs_kv_store;

const char* qs_version(void);
qs_status qs_last_error(char* buf, size_t n);
qs_status qs_device_check(void);

/* ---- L0 quantisation entry points (Q/quant.py) ---- */
/* encode_plane_hierarchical Q/quant.py:251-276 (with encode_plane_asym :220-248) */
qs_status qs_encode_plane_hierarchical(const double* values, int64_t count, int group, int64_t row_len,
                                       uint8_t* upper_codes, uint8_t* lower_codes, float* upper_scales,
                                       float* upper_zeros, float* lower_scales, int* flags, void* stream);
/* quantize_group_sym_s4 Q/quant.py:83-91 (scale already rounded to f32) */
qs_status qs_quantize_sym_s4(const double* values, int64_t count, float scale, int8_t* codes, int* flags,
                             void* stream);
/* decode_plane_draft / decode_plane_target Q/quant.py:293-309 (target if lower_codes != NULL) */
qs_status qs_decode_plane(const uint8_t* upper_codes, const uint8_t* lower_codes, const float* scales,
                          const float* zeros, int64_t count, int group, int64_t row_len, double* out,
                          void* stream);
/* quantize_weights Q/quant.py:335-349: reference plane + frag4 device layout.
 * frag_params: per (16-row tile, group, g) float4 {S_g, Z_g - 1024 S_g, S_g8/16, Z_g8 - 64 S_g8} */
qs_status qs_quantize_weights(const float* w, int d_in, int d_out, int group, uint8_t* ref_codes,
                              float* scales, float* zeros, uint32_t* frag4, void* frag_params, int* flags,
                              void* stream);
/* fp16 weights into frag16 layout (no reference counterpart: storage format) */
qs_status qs_pack_weights_f16(const float* w, int d_in, int d_out, void* frag16, void* stream);
/* ---- L1 KV store (Q/cache.py) ---- */
/* _quantize_block Q/cache.py:283-303 for nblk consecutive blocks of one (seq, layer)
 * from head-major fp16 rows src[Hkv][src_rows][hd]; writes blocks dst_block.. */
qs_status qs_kv_quantize_blocks(const qs_kv_store* st, int seq, int layer, const void* src_k, const void* src_v,
                                int64_t src_head_stride, int nblk, int dst_block, int* flags, void* stream);
/* flush_if_full Q/cache.py:249-281, full-fp1 branch, for every sequence of the batch whose
 * device lengths say so (fp2_len[s] == G and fp1_len[s] == G): quantise fp1 of every layer into
 * block n_blocks[s], fp1 <- fp2, n_blocks[s] += 1, fp2_len[s] -= G.  Decided on the device, so a
 * captured decode cycle flushes without a host round trip; the host mirrors the same rule from the
 * per-cycle readback.  flags: bit 1 non-finite K/V (DataError, Q/quant.py:60-64), bit 4 arena full. */
qs_status qs_kv_flush(const qs_kv_store* st, int* n_blocks, const int* fp1_len, int* fp2_len, int* flags,
                      void* stream);
/* _decode_block / _quantized_region Q/cache.py:317-343: f32 view of blocks [0, nblk) */
qs_status qs_kv_dequant_view(const qs_kv_store* st, int seq, int layer, int nblk, int target, float* out_k,
                             float* out_v, void* stream);

/* ---- L2 forward pieces (Q/model.py) ---- */
qs_status qs_attn_decode(const qs_attn_args* a, int mode, void* stream);
int qs_attn_partials_floats(const qs_attn_args* a);
/* resident CTAs per SM of the attention kernel for (head_dim, query columns per CTA, mode);
 * the host sizes the split-K grid with it (fixed per view so results stay batch-invariant) */
int qs_attn_occupancy(int hd, int n_query_cols, int mode);
qs_status qs_linear(const qs_linear_args* a, void* stream);
/* rmsnorm Q/tensor.py:35-42 over rows [n][d] */
qs_status qs_rmsnorm(const float* x, const float* gain, float* out, int n, int d, float eps, void* stream);
/* linear-layer input prep: xh = f16(rmsnorm(x) * gain) (or f16(x) when gain is NULL),
 * xs = f32 sums of every 16 consecutive f16 values (INT4 zero-point term) */
qs_status qs_prep_act(const float* x, const float* gain, float eps, void* xh, int64_t ldxh, float* xs,
                      int64_t ldxs, int n, int d, void* stream);
/* embedding lookup (Q/model.py:375) for n = B*T rows; row c takes
 * tokens[(c / T) * tok_stride + c % T]; an id outside [0, vocab) sets flags bit 2 (DataError) */
qs_status qs_embed(const float* table, const int* tokens, int tok_stride, int T, float* out, int n, int d,
                   int vocab, int* flags, void* stream);
/* greedy selection np.argmax (first max), Q/specdec.py:209-212 */
qs_status qs_argmax(const float* logits, int n, int vocab, int* out_idx, int out_stride, void* stream);
/* greedy verification Q/specdec.py:276-299 for a ragged batch of B sequences.  Sequence b's
 * verify tokens are tok[b*tok_stride + 0..T-1] = (pending, d_0..d_{T-2}); tgt[b*T + i] is the
 * target argmax of its row i; gamma_step[b] <= T-1 of its drafts count (NULL: all T-1).
 * Per sequence: v = accepted prefix, next = tgt[v] (corrected or bonus); writes res[2b] = v,
 * res[2b+1] = next, tok[b*tok_stride] = next (the next cycle's pending token) and adds v+1
 * (the rows kept after rollback(gamma_step - v)) to fp2_len[b] and pos[b] (either may be NULL). */
qs_status qs_greedy_accept(int* tok, int tok_stride, const int* target, int T, const int* gamma_step, int B,
                           int* res, int* fp2_len, int* pos, void* stream);
/* device-side length bump (append bookkeeping of Q/cache.py:234) */
qs_status qs_add_int(int* p, int n, int delta, void* stream);

/* ---- KV-head sharding buffers (qs_gather_args): whole cudaMalloc allocations, so they can be
 * exported to the other ranks' processes as CUDA IPC handles (64 bytes) ---- */
qs_status qs_dev_alloc(size_t bytes, void** ptr); /* zero-filled */
qs_status qs_dev_free(void* ptr);
qs_status qs_ipc_handle(void* ptr, char* handle64);
qs_status qs_ipc_open(const char* handle64, void** ptr);
qs_status qs_ipc_close(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* QUANTSPEC_B200_H */
