// extern "C" boundary (include/quantspec_b200.h): argument validation that
// mirrors the reference's typed errors, then stream-ordered kernel launches.
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "qs_api_internal.h"
#include "qs_common.cuh"

namespace qs {
cudaError_t launch_encode_plane(const double* v, long long count, int group, long long row_len, uint8_t* up,
                                uint8_t* lo, float* s, float* z, float* sl, int* flags, cudaStream_t st);
cudaError_t launch_sym_s4(const double* e, long long n, float scale, int8_t* out, int* flags, cudaStream_t st);
cudaError_t launch_decode_plane(const uint8_t* up, const uint8_t* lo, const float* s, const float* z,
                                long long count, int group, long long row_len, double* out, cudaStream_t st);
cudaError_t launch_quantize_weights(const float* w, int d_in, int d_out, int group, uint8_t* ref, float* s,
                                    float* z, uint32_t* frag4, float4* fparams, int* flags, cudaStream_t st);
cudaError_t launch_pack_f16(const float* w, int d_in, int d_out, __half* out, cudaStream_t st);
cudaError_t launch_kv_quantize(const qs_kv_store& stt, int seq, int layer0, int nlayers, const __half* sk,
                               const __half* sv, long long layer_stride, long long head_stride, int nblk,
                               int dst_block, int* flags, cudaStream_t s);
cudaError_t launch_kv_dequant(const qs_kv_store& st, int seq, int layer, int nblk, int target, float* ok,
                              float* ov, cudaStream_t s);
cudaError_t launch_kv_flush(const qs_kv_store& st, int* n_blocks, int* fp1_len, int* fp2_len, int* flags,
                            cudaStream_t s);
cudaError_t launch_rmsnorm(const float* x, const float* gain, float* out, int n, int d, float eps, cudaStream_t s);
cudaError_t launch_embed(const float* table, const int* tok, int tok_stride, int T, float* out, int n, int d,
                         int vocab, int* flags, cudaStream_t s);
cudaError_t launch_argmax(const float* logits, int n, int vocab, int* out, int out_stride, cudaStream_t s);
cudaError_t launch_greedy_accept(int* tok, int tok_stride, const int* tgt, int T, const int* gs, int B, int* res,
                                 int* fp2_len, int* pos, cudaStream_t s);
cudaError_t launch_add_int(int* p, int n, int delta, cudaStream_t s);

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
}  // namespace qs

using namespace qs;

#define QS_FAIL(code, ...)      \
  do {                          \
    qs::set_error(__VA_ARGS__); \
    return code;                \
  } while (0)

static qs_status cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return QS_OK;
  qs::set_error("%s: %s", what, cudaGetErrorString(e));
  return QS_ERR_CUDA;
}

static inline cudaStream_t S(void* s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" {

const char* qs_version(void) { return "quantspec-b200 0.1 (sm_100a)"; }

qs_status qs_last_error(char* buf, size_t n) {
  if (buf && n) {
    strncpy(buf, qs::g_err, n - 1);
    buf[n - 1] = 0;
  }
  return QS_OK;
}

qs_status qs_device_check(void) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDevice");
  cudaDeviceProp p;
  e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return cuda_status(e, "cudaGetDeviceProperties");
  if (p.major != 10) QS_FAIL(QS_ERR_CUDA, "device %s is sm_%d%d; this library is built for sm_100a only", p.name, p.major, p.minor);
  return QS_OK;
}

qs_status qs_encode_plane_hierarchical(const double* values, int64_t count, int group, int64_t row_len,
                                       uint8_t* upper_codes, uint8_t* lower_codes, float* upper_scales,
                                       float* upper_zeros, float* lower_scales, int* flags, void* stream) {
  if (count <= 0) QS_FAIL(QS_ERR_DATA, "cannot quantize an empty group");
  if (group < 1) QS_FAIL(QS_ERR_CONFIG, "group size must be >= 1, got %d", group);
  if (row_len > 0 && row_len < count && count % row_len)
    QS_FAIL(QS_ERR_INTEGRITY, "plane of %lld codes is not a whole number of %lld-rows", (long long)count,
            (long long)row_len);
  return cuda_status(launch_encode_plane(values, count, group, row_len, upper_codes, lower_codes, upper_scales,
                                         upper_zeros, lower_scales, flags, S(stream)),
                     "encode_plane");
}

qs_status qs_quantize_sym_s4(const double* values, int64_t count, float scale, int8_t* codes, int* flags,
                             void* stream) {
  if (!(scale > 0.0f)) QS_FAIL(QS_ERR_CONFIG, "symmetric quantization needs a positive scale, got %g", (double)scale);
  if (count <= 0) QS_FAIL(QS_ERR_DATA, "cannot quantize an empty group");
  return cuda_status(launch_sym_s4(values, count, scale, codes, flags, S(stream)), "quantize_sym_s4");
}

qs_status qs_decode_plane(const uint8_t* upper_codes, const uint8_t* lower_codes, const float* scales,
                          const float* zeros, int64_t count, int group, int64_t row_len, double* out,
                          void* stream) {
  if (count <= 0 || group < 1) QS_FAIL(QS_ERR_CONFIG, "bad plane geometry");
  return cuda_status(
      launch_decode_plane(upper_codes, lower_codes, scales, zeros, count, group, row_len, out, S(stream)),
      "decode_plane");
}

qs_status qs_quantize_weights(const float* w, int d_in, int d_out, int group, uint8_t* ref_codes, float* scales,
                              float* zeros, uint32_t* frag4, void* frag_params, int* flags, void* stream) {
  if (d_in < 1 || d_out < 1) QS_FAIL(QS_ERR_CONFIG, "weight quantization expects a non-empty 2-D matrix");
  if (group < 1) QS_FAIL(QS_ERR_CONFIG, "group size must be >= 1, got %d", group);
  int g = group < d_in ? group : d_in;
  if ((frag4 || frag_params) && (d_in % 16 || d_out % 16 || g % 16))
    QS_FAIL(QS_ERR_CONFIG, "INT4 device layout needs d_in, d_out and the group size to be multiples of 16 (%d, %d, %d)",
            d_in, d_out, g);
  return cuda_status(launch_quantize_weights(w, d_in, d_out, group, ref_codes, scales, zeros, frag4,
                                             reinterpret_cast<float4*>(frag_params), flags, S(stream)),
                     "quantize_weights");
}

qs_status qs_pack_weights_f16(const float* w, int d_in, int d_out, void* frag16, void* stream) {
  if (d_in % 16 || d_out % 16) QS_FAIL(QS_ERR_CONFIG, "fp16 device layout needs d_in, d_out multiples of 16");
  return cuda_status(launch_pack_f16(w, d_in, d_out, reinterpret_cast<__half*>(frag16), S(stream)), "pack_f16");
}

static qs_status check_store(const qs_kv_store* st) {
  if (!st) QS_FAIL(QS_ERR_CONFIG, "null store");
  if (st->hd != 16 && st->hd != 32 && st->hd != 64 && st->hd != 128)
    QS_FAIL(QS_ERR_CONFIG, "head_dim %d not supported on the device path (16/32/64/128)", st->hd);
  if (st->G % 16 || st->G > 128 || 128 % st->G)
    QS_FAIL(QS_ERR_CONFIG, "group size %d not supported on the device path (16, 32, 64, 128)", st->G);
  int kvd = st->Hkv * st->hd;
  if (!(st->G % st->hd == 0 || kvd <= st->G))
    QS_FAIL(QS_ERR_CONFIG, "value groups of %d channels would split a %d-channel head", st->G, st->hd);
  return QS_OK;
}

qs_status qs_kv_quantize_blocks(const qs_kv_store* st, int seq, int layer, const void* src_k, const void* src_v,
                                int64_t src_head_stride, int nblk, int dst_block, int* flags, void* stream) {
  qs_status r = check_store(st);
  if (r) return r;
  if (nblk <= 0) return QS_OK;
  if (dst_block + nblk > st->max_blocks)
    QS_FAIL(QS_ERR_OVERFLOW, "quantised arena full (%d + %d > %d blocks)", dst_block, nblk, st->max_blocks);
  return cuda_status(launch_kv_quantize(*st, seq, layer, 1, reinterpret_cast<const __half*>(src_k),
                                        reinterpret_cast<const __half*>(src_v), 0, src_head_stride, nblk,
                                        dst_block, flags, S(stream)),
                     "kv_quantize");
}

qs_status qs_kv_flush(const qs_kv_store* st, int* n_blocks, const int* fp1_len, int* fp2_len, int* flags,
                      void* stream) {
  qs_status r = check_store(st);
  if (r) return r;
  if (!n_blocks || !fp1_len || !fp2_len) QS_FAIL(QS_ERR_CONFIG, "flush needs the device length arrays");
  if (st->fp_rows < st->G) QS_FAIL(QS_ERR_CONFIG, "fp buffers of %d rows cannot hold a group of %d", st->fp_rows, st->G);
  return cuda_status(launch_kv_flush(*st, n_blocks, const_cast<int*>(fp1_len), fp2_len, flags, S(stream)),
                     "kv_flush");
}

qs_status qs_kv_dequant_view(const qs_kv_store* st, int seq, int layer, int nblk, int target, float* out_k,
                             float* out_v, void* stream) {
  qs_status r = check_store(st);
  if (r) return r;
  return cuda_status(launch_kv_dequant(*st, seq, layer, nblk, target, out_k, out_v, S(stream)), "kv_dequant");
}

int qs_attn_partials_floats(const qs_attn_args* a) {
  int per = (a->n_queries + a->n_qgroups - 1) / a->n_qgroups;
  int nq = 0;
  for (int m = 0; m < 3; ++m) {  // one scratch layout serves every view
    int v = qs::attention_queries_per_cta(per, m);
    if (v > nq) nq = v;
  }
  return a->B * a->Hkv * a->n_qgroups * (a->n_main + 2) * nq * (a->hd + 2);
}

int qs_attn_occupancy(int hd, int n_query_cols, int mode) { return qs::attention_occupancy(hd, n_query_cols, mode); }

qs_status qs_attn_decode(const qs_attn_args* a, int mode, void* stream) {
  if (!a) QS_FAIL(QS_ERR_CONFIG, "null args");
  if (a->hd != 16 && a->hd != 32 && a->hd != 64 && a->hd != 128) QS_FAIL(QS_ERR_CONFIG, "head_dim %d unsupported", a->hd);
  if (a->T < 1 || a->r < 1 || a->n_queries != a->T * a->r) QS_FAIL(QS_ERR_DIMENSION, "bad query geometry");
  int per = (a->n_queries + a->n_qgroups - 1) / a->n_qgroups;
  const int per_max = mode == QS_VIEW_TARGET ? 24 : 12;  // target: up to three 8-query MMA tiles (TMEM-parked)
  if (per > per_max) QS_FAIL(QS_ERR_CONFIG, "at most %d query columns per CTA (got %d); raise n_qgroups", per_max, per);
  if (a->n_main < 1) QS_FAIL(QS_ERR_CONFIG, "need at least one main split");
  if (mode != QS_VIEW_FP16 && (a->G % 16 || a->G > 128 || 128 % a->G)) QS_FAIL(QS_ERR_CONFIG, "group size %d unsupported", a->G);
  if ((a->fp1_k || a->fp2_k) && a->fp_rows < a->G)
    QS_FAIL(QS_ERR_CONFIG, "fp buffers of %d rows cannot hold a group of %d", a->fp_rows, a->G);
  if (mode != QS_VIEW_FP16 && !(a->G % a->hd == 0 || a->Hkv * a->hd <= a->G))
    QS_FAIL(QS_ERR_CONFIG, "value groups of %d channels would split a %d-channel head", a->G, a->hd);
  if (a->gather.world) {
    const qs_gather_args& g = a->gather;
    if (g.world < 1 || g.world > QS_MAX_RANKS || g.rank < 0 || g.rank >= g.world)
      QS_FAIL(QS_ERR_CONFIG, "gather: rank %d of world %d", g.rank, g.world);
    if (!a->out_h || !a->out_s || !g.epoch || !g.done) QS_FAIL(QS_ERR_CONFIG, "gather needs out_h, out_s, epoch, done");
    for (int i = 0; i < g.world; ++i)
      if (!g.gh[i] || !g.gs[i] || !g.flag[i]) QS_FAIL(QS_ERR_CONFIG, "gather: rank %d buffers missing", i);
    if (g.arrivals != g.world * a->B * a->Hkv * a->n_qgroups)
      QS_FAIL(QS_ERR_CONFIG, "gather: %d arrivals per layer, expected world*B*Hkv*n_qgroups", g.arrivals);
  }
  return cuda_status(launch_attention(*a, mode, S(stream)), "attn_decode");
}

qs_status qs_linear(const qs_linear_args* a, void* stream) {
  if (!a) QS_FAIL(QS_ERR_CONFIG, "null args");
  if (a->K % 16 || a->N % 16) QS_FAIL(QS_ERR_DIMENSION, "linear dims must be multiples of 16 (N=%d K=%d)", a->N, a->K);
  if (a->ncols < 1 || a->ncols > QS_MAX_COLS)
    QS_FAIL(QS_ERR_DIMENSION, "1..%d activation rows supported (got %d)", QS_MAX_COLS, a->ncols);
  if (a->wmode == QS_W_INT4 && a->ncols > 16) QS_FAIL(QS_ERR_DIMENSION, "INT4 (draft) linear: at most 16 rows");
  if (a->epi == QS_EPI_SILU_MUL && a->N % 32) QS_FAIL(QS_ERR_DIMENSION, "gate/up interleave needs N multiple of 32");
  if (a->wmode == QS_W_INT4 && a->wgroup != 16 && a->wgroup != 32 && a->wgroup != 64 && a->wgroup != 128)
    QS_FAIL(QS_ERR_CONFIG, "INT4 group %d unsupported on the device path (16/32/64/128)", a->wgroup);
  if (a->xf) {
    if (a->ncols != 1 || a->K > 4096 || a->ldxf % 4 || a->ldxf < a->K)
      QS_FAIL(QS_ERR_CONFIG, "in-kernel activation prep needs one row, K <= 4096, 16-byte rows");
  } else if (a->ldxh % 8 || a->ldxh < a->K + 64 ||
             (a->wmode == QS_W_INT4 && (a->ldxs % 4 || a->ldxs < a->K / 16 + 4))) {
    QS_FAIL(QS_ERR_CONFIG, "activation buffers need padded, 16-byte aligned rows");
  }
  return cuda_status(launch_linear(*a, S(stream)), "linear");
}

qs_status qs_prep_act(const float* x, const float* gain, float eps, void* xh, int64_t ldxh, float* xs, int64_t ldxs,
                      int n, int d, void* stream) {
  if (n < 1 || d < 16 || d % 16) QS_FAIL(QS_ERR_DIMENSION, "prep_act needs rows of a multiple of 16 (d=%d)", d);
  return cuda_status(qs::launch_prep_act(x, gain, eps, xh, ldxh, xs, ldxs, n, d, S(stream)), "prep_act");
}

qs_status qs_rmsnorm(const float* x, const float* gain, float* out, int n, int d, float eps, void* stream) {
  if (n < 1 || d < 1) QS_FAIL(QS_ERR_DIMENSION, "empty rmsnorm");
  return cuda_status(launch_rmsnorm(x, gain, out, n, d, eps, S(stream)), "rmsnorm");
}

qs_status qs_embed(const float* table, const int* tokens, int tok_stride, int T, float* out, int n, int d,
                   int vocab, int* flags, void* stream) {
  if (T < 1 || tok_stride < T || n < 1 || n % T) QS_FAIL(QS_ERR_DIMENSION, "embed: bad row geometry");
  return cuda_status(launch_embed(table, tokens, tok_stride, T, out, n, d, vocab, flags, S(stream)), "embed");
}

qs_status qs_argmax(const float* logits, int n, int vocab, int* out_idx, int out_stride, void* stream) {
  if (vocab < 1) QS_FAIL(QS_ERR_CONFIG, "empty vocab");
  return cuda_status(launch_argmax(logits, n, vocab, out_idx, out_stride, S(stream)), "argmax");
}

qs_status qs_greedy_accept(int* tok, int tok_stride, const int* target, int T, const int* gamma_step, int B,
                           int* res, int* fp2_len, int* pos, void* stream) {
  if (T < 1 || B < 1 || tok_stride < T) QS_FAIL(QS_ERR_CONFIG, "greedy_accept: bad geometry");
  return cuda_status(launch_greedy_accept(tok, tok_stride, target, T, gamma_step, B, res, fp2_len, pos, S(stream)),
                     "greedy_accept");
}

qs_status qs_add_int(int* p, int n, int delta, void* stream) {
  return cuda_status(launch_add_int(p, n, delta, S(stream)), "add_int");
}

qs_status qs_dev_alloc(size_t bytes, void** ptr) {
  if (!ptr) QS_FAIL(QS_ERR_CONFIG, "null out pointer");
  *ptr = nullptr;
  cudaError_t e = cudaMalloc(ptr, bytes);
  if (e == cudaSuccess) e = cudaMemset(*ptr, 0, bytes);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  return cuda_status(e, "dev_alloc");
}

qs_status qs_dev_free(void* ptr) { return cuda_status(cudaFree(ptr), "dev_free"); }

qs_status qs_ipc_handle(void* ptr, char* handle64) {
  if (!ptr || !handle64) QS_FAIL(QS_ERR_CONFIG, "null pointer");
  cudaIpcMemHandle_t h;
  cudaError_t e = cudaIpcGetMemHandle(&h, ptr);
  if (e == cudaSuccess) memcpy(handle64, &h, sizeof(h) < 64 ? sizeof(h) : 64);
  return cuda_status(e, "ipc_handle");
}

qs_status qs_ipc_open(const char* handle64, void** ptr) {
  if (!ptr || !handle64) QS_FAIL(QS_ERR_CONFIG, "null pointer");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h) < 64 ? sizeof(h) : 64);
  return cuda_status(cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess), "ipc_open");
}

qs_status qs_ipc_close(void* ptr) { return cuda_status(cudaIpcCloseMemHandle(ptr), "ipc_close"); }

}  // extern "C"
