// Device data layout of the hierarchical KV store and packed weights.
// Shared by the CUDA kernels (qs_*.cu); the Python host mirror restates the
// same formulas in paper_2502_10424_b200/layout.py.
//
// Quantised arena, per plane P in {KU, KL, VU, VL} (uint8):
//   P[seq][layer][kv_head][block][G*hd/2]
// Within one (head, block) the codes are stored as frag4 words (qs_common.cuh):
//   keys   (A = K[token][channel]):  word((mt, ks), lane) with mt = token/16, ks = channel/16
//   values (A = V^T[channel][token]): word((ks, cm), lane) with ks = token/16, cm = channel/16
//   index(outer, inner, lane) = ((outer*(NI/VEC) + inner/VEC)*32 + lane)*VEC + inner%VEC
//   NI = hd/16 (inner tiles per outer tile), VEC = min(NI, 4)
// KL/VL hold the lower codes offset-binary (c_l + 8), so one select-lop3
// rebuilds the exact 8-bit target code 16*c_u + c_l + 8.
//
// Key params  (float2 S,Z):  KP[seq][layer][kv_head][block][hd]   (one group per channel)
// Value params(float2 S,Z):  VP[seq][layer][kv_head][block][G]    (the group holding this head)
// fp buffers (half):         FP[seq][layer][2][kv_head][G][hd]     (0 = fp1, 1 = fp2)
// fp16 cache (half):         K/V[seq][layer][kv_head][cap][hd]
#pragma once
#include <stdint.h>

#define QS_CHUNK_Q 128  // tokens per quantised attention chunk
#define QS_CHUNK_F 64   // tokens per fp16 attention chunk

static inline __host__ __device__ int qs_vec(int ni) { return ni >= 4 ? 4 : ni; }

static inline __host__ __device__ int qs_frag_index(int outer, int inner, int lane, int ni) {
  int vec = qs_vec(ni);
  return ((outer * (ni / vec) + inner / vec) * 32 + lane) * vec + (inner % vec);
}

// position of element (row, col) of a 16x16 A tile inside the frag4 word of a lane
static inline __host__ __device__ void qs_frag_pos(int row, int col, int* lane, int* nib) {
  int g = row & 7, jlo = row >> 3;
  int jhi = col >> 3, rem = col & 7;
  int t = rem >> 1, h = rem & 1;
  *lane = g * 4 + t;
  *nib = (jlo + 2 * jhi) + 4 * h;
}

// position of element (row, col) of a 16x16 A tile inside the 8-half register
// quad of a lane (fp16 weights): halves [a0.lo a0.hi a1.lo a1.hi a2.lo a2.hi a3.lo a3.hi]
static inline __host__ __device__ void qs_frag16_pos(int row, int col, int* lane, int* slot) {
  int g = row & 7, jlo = row >> 3;
  int jhi = col >> 3, rem = col & 7;
  int t = rem >> 1, h = rem & 1;
  *lane = g * 4 + t;
  *slot = 2 * (jlo + 2 * jhi) + h;
}
