// Shared device helpers for the QuantSpec B200 kernels (sm_100a only).
//
// Fragment conventions (mma.sync.m16n8k16, f16 x f16 -> f32), used by every
// kernel that dequantises in registers:
//   A (16x16, row-major): lane (g = lane>>2, t = lane&3) holds
//     a0 = (row g,   cols 2t,2t+1)   a1 = (row g+8, cols 2t,2t+1)
//     a2 = (row g,   cols 2t+8,2t+9) a3 = (row g+8, cols 2t+8,2t+9)
//   B (16x8):  b0 = (rows 2t,2t+1, col g)  b1 = (rows 2t+8,2t+9, col g)
//   D (16x8):  d0,d1 = (row g, cols 2t,2t+1)  d2,d3 = (row g+8, cols 2t,2t+1)
//
// Packed 4-bit A fragment ("frag4"): one u32 per lane per 16x16 tile.  Nibble
// p (bits 4p..4p+3) holds A element
//     j = p & 3, h = p >> 2:  row = g + 8*(j&1),  col = 2t + 8*(j>>1) + h
// so a_j = lop3(x >> 4*(j&~1)..) style extraction yields (lo=nibble j, hi=nibble j+4)
// directly as an f16x2 pair with the 0x6400 magic exponent.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef __CUDA_ARCH__
#define QS_HOST_ONLY 1
#endif

namespace qs {

constexpr int kWarp = 32;

// ---------------------------------------------------------------------------
// tensor-core MMA (legacy warp-level path; per-column independent, so the
// result for one query column does not depend on how many columns ride along)
// ---------------------------------------------------------------------------
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t lop3_and_or(uint32_t x, uint32_t mask, uint32_t magic) {
  uint32_t r;
  // (x & mask) | magic
  asm("lop3.b32 %0, %1, %2, %3, 0xEA;\n" : "=r"(r) : "r"(x), "r"(mask), "r"(magic));
  return r;
}

__device__ __forceinline__ uint32_t lop3_select(uint32_t a, uint32_t b, uint32_t mask) {
  // (a & mask) | (b & ~mask)
  uint32_t r;
  asm("lop3.b32 %0, %1, %2, %3, 0xE4;\n" : "=r"(r) : "r"(a), "r"(b), "r"(mask));
  return r;
}

__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
  uint32_t r;
  asm("prmt.b32 %0, %1, %2, %3;\n" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
  return r;
}

__device__ __forceinline__ uint32_t h2_as_u32(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u32_as_h2(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }

// 8 unsigned nibbles -> four exact f16x2 A registers (values 0..15).
__device__ __forceinline__ void unpack_u4(uint32_t x, uint32_t (&a)[4]) {
  const uint32_t MAGIC = 0x64006400u;  // f16 1024.0 in both halves
  const __half2 k1024 = __halves2half2(__ushort_as_half(0x6400), __ushort_as_half(0x6400));
  const __half2 k1_16 = __halves2half2(__ushort_as_half(0x2C00), __ushort_as_half(0x2C00));  // 1/16
  const __half2 km64 = __halves2half2(__ushort_as_half(0xD400), __ushort_as_half(0xD400));   // -64
  uint32_t t = x >> 8;
  a[0] = h2_as_u32(__hsub2(u32_as_h2(lop3_and_or(x, 0x000F000Fu, MAGIC)), k1024));
  a[1] = h2_as_u32(__hfma2(u32_as_h2(lop3_and_or(x, 0x00F000F0u, MAGIC)), k1_16, km64));
  a[2] = h2_as_u32(__hsub2(u32_as_h2(lop3_and_or(t, 0x000F000Fu, MAGIC)), k1024));
  a[3] = h2_as_u32(__hfma2(u32_as_h2(lop3_and_or(t, 0x00F000F0u, MAGIC)), k1_16, km64));
}

// Upper nibbles x (c_u in 0..15) and lower nibbles y stored offset-binary
// (c_l + 8 in 0..15) -> four f16x2 registers holding the exact combined code
// 16*c_u + c_l (0..240 for codes produced by the encoder).
__device__ __forceinline__ void unpack_u4l4(uint32_t x, uint32_t y, uint32_t (&a)[4]) {
  const __half2 k1032 = __halves2half2(__ushort_as_half(0x6408), __ushort_as_half(0x6408));  // 1032
  uint32_t ev = lop3_select(x << 4, y, 0xF0F0F0F0u);         // bytes: codes at nibble pos 0,2,4,6
  uint32_t od = lop3_select(x, y >> 4, 0xF0F0F0F0u);         // bytes: codes at nibble pos 1,3,5,7
  const uint32_t M = 0x64646464u;
  a[0] = h2_as_u32(__hsub2(u32_as_h2(prmt(ev, M, 0x4240u)), k1032));  // pos0 (ev.b0), pos4 (ev.b2)
  a[1] = h2_as_u32(__hsub2(u32_as_h2(prmt(od, M, 0x4240u)), k1032));  // pos1, pos5
  a[2] = h2_as_u32(__hsub2(u32_as_h2(prmt(ev, M, 0x4341u)), k1032));  // pos2, pos6
  a[3] = h2_as_u32(__hsub2(u32_as_h2(prmt(od, M, 0x4341u)), k1032));  // pos3, pos7
}

// Offset forms for the attention kernels: no per-element subtraction; the
// constant offsets are folded into per-block score biases / per-column sums.
//   unpack_u4_raw:   a0,a2 = 1024 + c (rows g),  a1,a3 = 1024 + 16 c (rows g+8)
//   unpack_u4l4_raw: all = 1032 + (16 c_u + c_l)
__device__ __forceinline__ void unpack_u4_raw(uint32_t x, uint32_t (&a)[4]) {
  const uint32_t MAGIC = 0x64006400u;
  uint32_t t = x >> 8;
  a[0] = lop3_and_or(x, 0x000F000Fu, MAGIC);
  a[1] = lop3_and_or(x, 0x00F000F0u, MAGIC);
  a[2] = lop3_and_or(t, 0x000F000Fu, MAGIC);
  a[3] = lop3_and_or(t, 0x00F000F0u, MAGIC);
}
__device__ __forceinline__ void unpack_u4l4_raw(uint32_t x, uint32_t y, uint32_t (&a)[4]) {
  uint32_t ev = lop3_select(x << 4, y, 0xF0F0F0F0u);
  uint32_t od = lop3_select(x, y >> 4, 0xF0F0F0F0u);
  const uint32_t M = 0x64646464u;
  a[0] = prmt(ev, M, 0x4240u);
  a[1] = prmt(od, M, 0x4240u);
  a[2] = prmt(ev, M, 0x4341u);
  a[3] = prmt(od, M, 0x4341u);
}

// 2^x on the SFU alone (ex2.approx.ftz: one MUFU, 2 ulp; exp2f adds the denormal-range fix-up
// around it).  ex2(-inf) = +0.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(y) : "f"(x));
  return y;
}

// split an f32 into f16 hi + f16 lo (hi + lo reproduces ~22 bits)
__device__ __forceinline__ void split_hl(float v, __half& hi, __half& lo) {
  hi = __float2half_rn(v);
  lo = __float2half_rn(v - __half2float(hi));
}

// ---------------------------------------------------------------------------
// ldmatrix / cp.async / bulk copy / mbarrier
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void ldmatrix_x4(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], uint32_t addr) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred = true) {
  int sz = pred ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::);
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes));
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity));
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// blocking wait with a suspend-time hint: the warp sleeps in hardware until the
// phase completes instead of spinning (keeps issue slots for the warps doing work)
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity), "r"(0x100000u));
  } while (!ok);
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
// ticket counter with release-acquire semantics at GPU scope (replaces fence.sc + relaxed atomic)
__device__ __forceinline__ int atom_add_acq_rel_gpu(int* p, int v) {
  int old;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;\n" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}

// ---------------------------------------------------------------------------
// Tensor memory (tcgen05): accumulator parking for the wide-query verify consumers.  One warp
// allocates / frees; warp w may touch TMEM lanes [32 (w % 4), 32 (w % 4) + 32) only.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tmem_alloc(uint32_t* smem_dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(smem_dst)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(taddr), "r"(ncols) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
// 32 consecutive 32-bit columns of this thread's lane <-> 32 registers.  The waits name the
// registers as in/out operands: uses of loaded values cannot be hoisted above wait::ld, and the
// source registers of an in-flight st stay allocated until wait::st.
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, float (&v)[32]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]), "=f"(v[6]), "=f"(v[7]), "=f"(v[8]), "=f"(v[9]), "=f"(v[10]), "=f"(v[11]), "=f"(v[12]), "=f"(v[13]), "=f"(v[14]), "=f"(v[15]), "=f"(v[16]), "=f"(v[17]), "=f"(v[18]), "=f"(v[19]), "=f"(v[20]), "=f"(v[21]), "=f"(v[22]), "=f"(v[23]), "=f"(v[24]), "=f"(v[25]), "=f"(v[26]), "=f"(v[27]), "=f"(v[28]), "=f"(v[29]), "=f"(v[30]), "=f"(v[31])
               : "r"(taddr)
               : "memory");
}
__device__ __forceinline__ void tmem_wait_ld32(float (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]), "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]), "+f"(v[12]), "+f"(v[13]), "+f"(v[14]), "+f"(v[15]), "+f"(v[16]), "+f"(v[17]), "+f"(v[18]), "+f"(v[19]), "+f"(v[20]), "+f"(v[21]), "+f"(v[22]), "+f"(v[23]), "+f"(v[24]), "+f"(v[25]), "+f"(v[26]), "+f"(v[27]), "+f"(v[28]), "+f"(v[29]), "+f"(v[30]), "+f"(v[31]) :: "memory");
}
__device__ __forceinline__ void tmem_st32_issue(uint32_t taddr, const float (&v)[32]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "f"(v[4]), "f"(v[5]), "f"(v[6]), "f"(v[7]), "f"(v[8]), "f"(v[9]), "f"(v[10]), "f"(v[11]), "f"(v[12]), "f"(v[13]), "f"(v[14]), "f"(v[15]), "f"(v[16]), "f"(v[17]), "f"(v[18]), "f"(v[19]), "f"(v[20]), "f"(v[21]), "f"(v[22]), "f"(v[23]), "f"(v[24]), "f"(v[25]), "f"(v[26]), "f"(v[27]), "f"(v[28]), "f"(v[29]), "f"(v[30]), "f"(v[31])
               : "memory");
}
__device__ __forceinline__ void tmem_wait_st32(float (&v)[32]) {
  asm volatile("tcgen05.wait::st.sync.aligned;\n" : "+f"(v[0]), "+f"(v[1]), "+f"(v[2]), "+f"(v[3]), "+f"(v[4]), "+f"(v[5]), "+f"(v[6]), "+f"(v[7]), "+f"(v[8]), "+f"(v[9]), "+f"(v[10]), "+f"(v[11]), "+f"(v[12]), "+f"(v[13]), "+f"(v[14]), "+f"(v[15]), "+f"(v[16]), "+f"(v[17]), "+f"(v[18]), "+f"(v[19]), "+f"(v[20]), "+f"(v[21]), "+f"(v[22]), "+f"(v[23]), "+f"(v[24]), "+f"(v[25]), "+f"(v[26]), "+f"(v[27]), "+f"(v[28]), "+f"(v[29]), "+f"(v[30]), "+f"(v[31]) :: "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  tmem_ld32_issue(taddr, v);
  tmem_wait_ld32(v);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, float (&v)[32]) {
  tmem_st32_issue(taddr, v);
  tmem_wait_st32(v);
}

// cross-GPU (system-scope) signalling for the fused all-gather of KV-head-sharded attention
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys_add(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// TMA-engine 1-D bulk copy global -> shared, completion counted on an mbarrier.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// bulk prefetch of [src, src + bytes) into L2 (no shared memory, no barrier): keeps DRAM requests
// in flight beyond what a shared-memory ring can hold; the ring's later TMA copy then hits L2.
// bytes: a multiple of 16, src 16-byte aligned.
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
}

__device__ __forceinline__ uint4 ldg_nc_v4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// ---------------------------------------------------------------------------
// programmatic dependent launch (PDL).  Every hot-loop kernel is launched with
// programmatic stream serialisation: its CTAs may start while the previous
// kernel is still running.  Protocol (keeps the overlap window one kernel deep):
//   1. before pdl_wait(): only shared-memory setup and reads of data no kernel
//      on the decode path writes (weights, quantised blocks below n_blocks);
//   2. pdl_wait() in every thread (returns once the previous grid completed and
//      its memory is visible);
//   3. pdl_trigger() right after: lets the next kernel's CTAs be scheduled.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }

bool pdl_enabled();  // QS_PDL=0 in the environment disables it (A/B measurements)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, static_cast<Args&&>(args)...);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
template <typename T>
__device__ __forceinline__ T warp_max(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// INT4 weight params: slot of row g of group grp is g ^ i4_param_swz(grp).  One param load of
// the W4A16 consumer reads, per quarter warp, rows {2q, 2q+1} of four groups 512 B (CW = 1) or
// 256 B (CW = 2) apart -- the same banks without the swizzle (4-way conflict); the even XOR mask
// 2 f(grp & 7), f = 0 2 1 3 2 0 3 1, makes those groups' slots distinct for CW = 1, 2 and 4.
__host__ __device__ __forceinline__ int i4_param_swz(int grp) {
  const int i = grp & 7;
  return 2 * (((i >> 1) ^ ((i & 1) << 1)) & 3);
}

}  // namespace qs
