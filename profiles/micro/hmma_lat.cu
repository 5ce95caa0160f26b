// Latency / throughput of legacy mma.sync m16n8k16 (HMMA.16816.F32) on sm_100a.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_lat hmma_lat.cu && ./hmma_lat
#include <cstdio>
#include <cstdint>
template <int CH>
__global__ void k(float* out, long long* cyc, int iters) {
  uint32_t a[4] = {0x3c003c00u ^ threadIdx.x, 0x3c003c00u, 0x3c003c00u, 0x3c003c00u}, b0 = 0x3c003c00u, b1 = 0x3c003c00u;
  float d[CH][4] = {};
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                   : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  float s = 0;
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int CH>
void run(int warps) {
  float* o; long long* c; cudaMalloc(&o, 4 << 20); cudaMalloc(&c, 8 * 1024);
  int iters = 4096;
  k<CH><<<1, 32 * warps>>>(o, c, iters);
  cudaDeviceSynchronize();
  k<CH><<<1, 32 * warps>>>(o, c, iters);
  long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("chains %d warps/SM %2d: %.2f cycles per HMMA per warp, %.2f cycles per HMMA per SM\n", CH, warps,
         (double)h / (iters * CH), (double)h / (iters * CH * warps));
  cudaFree(o); cudaFree(c);
}
int main() {
  run<1>(1); run<2>(1); run<4>(1); run<8>(1);
  run<1>(4); run<2>(4); run<4>(4); run<8>(4);
  run<2>(16); run<4>(16); run<8>(16); run<2>(32);
  return 0;
}
