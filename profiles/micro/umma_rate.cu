// tcgen05.mma (UMMA, kind::f16, f32 accumulate in TMEM) correctness + issue rate on sm_100a, for the
// decode-attention shapes: M = 128 (tokens or channels of a chunk), small N (query columns), K = 16.
// Compared against the legacy mma.sync rate of profiles/micro/hmma_lat.cu (HMMA.16816: one per
// ~2 cycles per SM = 2048 MAC/cycle/SM).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu && ./umma_rate
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// SWIZZLE_NONE K-major canonical layout: 8-row x 16-byte core matrices; element (r, k) of a
// rows x K tile at ((r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2) bytes
__host__ __device__ inline uint32_t kmajor_off(int r, int k, int K) {
  const int LBO = 128, SBO = (K / 8) * 128;
  return (r / 8) * SBO + (k / 8) * LBO + (r % 8) * 16 + (k % 8) * 2;
}
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, int K) {
  const uint64_t lbo = 128, sbo = (uint64_t)(K / 8) * 128;
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // descriptor version (sm100)
  // base_offset 0, lbo_mode 0, layout_type 0 = SWIZZLE_NONE
  return d;
}
__host__ __device__ inline uint32_t make_idesc(int M, int N) {
  uint32_t d = 0;
  d |= 1u << 4;                      // D format F32
  // A/B format F16 (0), no negate, both K-major
  d |= (uint32_t)(N >> 3) << 17;     // N / 8
  d |= (uint32_t)(M >> 4) << 24;     // M / 16
  return d;
}

template <int N, int K, int NACC, bool ATMEM>
__global__ void umma_kernel(const __half* A, const __half* B, float* D, long long* cycles, int iters) {
  constexpr int M = 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sa = smem;
  uint8_t* sb = smem + M * K * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sb + N * K * 2);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < M * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sa + kmajor_off(r, k, K)) = A[i];
  }
  for (int i = tid; i < N * K; i += blockDim.x) {
    const int r = i / K, k = i % K;
    *reinterpret_cast<__half*>(sb + kmajor_off(r, k, K)) = B[i];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n");
  }
  constexpr uint32_t ACOL = ATMEM ? K / 2 : 0;  // A in tensor memory: K f16 = K/2 columns per row
  constexpr uint32_t NC0 = N * NACC + ACOL < 32 ? 32 : N * NACC + ACOL;
  constexpr uint32_t NCOL = NC0 <= 32 ? 32 : NC0 <= 64 ? 64 : NC0 <= 128 ? 128 : NC0 <= 256 ? 256 : 512;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tslot)), "r"(NCOL));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("fence.proxy.async.shared::cta;\n");  // generic-proxy smem writes -> visible to the tensor core
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  const uint32_t tmem = *tslot;
  const uint32_t ta = tmem + (uint32_t)(N * NACC);  // A operand columns (ATMEM)
  if constexpr (ATMEM) {
    // row 32w + lane of A -> TMEM lane 32w + lane, k pairs -> consecutive columns
    if (warp < 4) {
      const int row = 32 * warp + (tid & 31);
      uint32_t r[K / 2];
#pragma unroll
      for (int c = 0; c < K / 2; ++c) {
        __half2 h = __halves2half2(A[row * K + 2 * c], A[row * K + 2 * c + 1]);
        r[c] = *reinterpret_cast<uint32_t*>(&h);
      }
#pragma unroll
      for (int c = 0; c < K / 2; c += 8)
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(ta + ((uint32_t)(32 * warp) << 16) + c),
                     "r"(r[c]), "r"(r[c + 1]), "r"(r[c + 2]), "r"(r[c + 3]), "r"(r[c + 4]), "r"(r[c + 5]), "r"(r[c + 6]), "r"(r[c + 7]));
      asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
  }
  const uint64_t da = make_desc(smem_u32(sa), K), db = make_desc(smem_u32(sb), K);
  const uint32_t id = make_idesc(M, N);
  long long t0 = 0, t1 = 0;
  if (tid == 0) {
    t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int ks = 0; ks < K / 16; ++ks) {
        // advance both descriptors by one 16-wide k step = two core matrices (2 * LBO bytes)
        const uint64_t step = (uint64_t)(ks * 2 * 128) >> 4;
        const uint32_t acc = (it >= NACC || ks > 0) ? 1u : 0u;
        if constexpr (ATMEM)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem + (uint32_t)((it % NACC) * N)),
              "r"(ta + (uint32_t)(ks * 8)), "l"(db + step), "r"(id), "r"(acc));
        else
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + (uint32_t)((it % NACC) * N)),
              "l"(da + step), "l"(db + step), "r"(id), "r"(acc));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
    uint32_t ok = 0;
    while (!ok) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(ok) : "r"(smem_u32(bar)));
    }
    t1 = clock64();
    cycles[blockIdx.x] = t1 - t0;
  }
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n");
  // D row m -> TMEM lane m: warp w reads lanes 32w.., one column per load (x1)
  if (warp < 4) {
    for (int n = 0; n < N; ++n) {
      uint32_t v;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(tmem + ((uint32_t)(32 * warp) << 16) + n));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n");
      if (blockIdx.x == 0) D[(32 * warp + (tid & 31)) * N + n] = __uint_as_float(v);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(NCOL));
}

template <int N, int K, int NACC = 1, bool ATMEM = false>
void run(int nblocks, int iters) {
  constexpr int M = 128;
  std::vector<__half> a(M * K), b(N * K);
  std::vector<float> af(M * K), bf(N * K);
  srand(1);
  for (int i = 0; i < M * K; ++i) { float v = (rand() % 17 - 8) / 8.f; a[i] = __float2half(v); af[i] = v; }
  for (int i = 0; i < N * K; ++i) { float v = (rand() % 13 - 6) / 4.f; b[i] = __float2half(v); bf[i] = v; }
  __half *dA, *dB; float* dD; long long* dc;
  cudaMalloc(&dA, M * K * 2); cudaMalloc(&dB, N * K * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8 * 1024);
  cudaMemcpy(dA, a.data(), M * K * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, b.data(), N * K * 2, cudaMemcpyHostToDevice);
  const int smem = M * K * 2 + N * K * 2 + 64;
  auto kern = umma_kernel<N, K, NACC, ATMEM>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // correctness: one pass (iters = 1) -> D = A . B^T
  kern<<<1, 128, smem>>>(dA, dB, dD, dc, 1);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("N=%d K=%d: %s\n", N, K, cudaGetErrorString(e)); exit(1); }
  std::vector<float> d(M * N);
  cudaMemcpy(d.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < K; ++k) ref += (double)af[m * K + k] * bf[n * K + k];
      maxerr = fmax(maxerr, fabs(ref - d[m * N + n]));
    }
  kern<<<nblocks, 128, smem>>>(dA, dB, dD, dc, iters);
  cudaDeviceSynchronize();
  std::vector<long long> c(nblocks);
  cudaMemcpy(c.data(), dc, 8 * nblocks, cudaMemcpyDeviceToHost);
  double mean = 0;
  for (long long x : c) mean += (double)x / nblocks;
  const double per = mean / (iters * (K / 16));
  printf("UMMA m128n%dk16 A in %s (K=%d per pass, %d independent accumulators) blocks=%d: max|err| %.3g, %.2f cycles per UMMA, %.0f MAC/cycle/SM (HMMA.16816: ~2048)\n",
         N, ATMEM ? "TMEM" : "SMEM", K, NACC, nblocks, maxerr, per, 128.0 * N * 16 / per);
  cudaFree(dA); cudaFree(dB); cudaFree(dD); cudaFree(dc);
}

int main() {
  run<16, 16>(1, 4096);
  run<16, 64>(1, 1024);
  run<32, 64>(1, 1024);
  run<48, 64>(1, 1024);
  run<64, 64>(1, 1024);
  run<128, 64>(1, 1024);
  run<256, 64>(1, 512);
  run<48, 64>(148, 1024);
  run<16, 64, 4>(1, 1024);
  run<32, 64, 4>(1, 1024);
  run<48, 64, 4>(1, 1024);
  run<48, 64, 8>(1, 1024);
  run<64, 64, 4>(1, 1024);
  run<128, 64, 2>(1, 1024);
  run<16, 64, 4, true>(1, 1024);
  run<48, 64, 1, true>(1, 1024);
  run<48, 64, 4, true>(1, 1024);
  run<64, 64, 4, true>(1, 1024);
  run<128, 64, 2, true>(1, 1024);
  return 0;
}
