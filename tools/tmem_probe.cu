// TMEM probe: can tcgen05.ld.32x32b.xN start at a column that is not a
// multiple of N, and how fast are pipelined narrow loads?  Decides whether the
// column-pass ring can live in tensor memory.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void st1(uint32_t addr, uint32_t v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(addr), "r"(v));
}
__device__ __forceinline__ void ld16(uint32_t addr, uint32_t* v) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(addr));
}
__device__ __forceinline__ void ld4(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
               : "r"(addr));
}
__device__ __forceinline__ void ld1(uint32_t addr, uint32_t& v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(addr));
}
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;"); }

__global__ void probe(int start16, int start4, uint32_t* out) {
  __shared__ uint32_t base_s;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = base_s;
  const uint32_t la = base + ((uint32_t)(warp * 32) << 16);
  for (int c = 0; c < 512; ++c) st1(la + c, (uint32_t)(threadIdx.x * 1000 + c));
  wait_st();
  uint32_t v[16];
  ld16(la + start16, v);
  wait_ld();
  int bad16 = 0;
  for (int j = 0; j < 16; ++j) bad16 += (v[j] != (uint32_t)(threadIdx.x * 1000 + start16 + j));
  uint32_t w[4];
  ld4(la + start4, w);
  wait_ld();
  int bad4 = 0;
  for (int j = 0; j < 4; ++j) bad4 += (w[j] != (uint32_t)(threadIdx.x * 1000 + start4 + j));
  // pipelined x1 loads: 8 independent loads per wait
  long long t0 = clock64();
  uint32_t acc = 0;
  for (int it = 0; it < 256; ++it) {
    uint32_t a[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) ld1(la + ((it * 8 + j * 61) & 511), a[j]);
    wait_ld();
#pragma unroll
    for (int j = 0; j < 8; ++j) acc += a[j];
  }
  long long t1 = clock64();
  // pipelined x16: 4 loads per wait
  uint32_t b[64];
  for (int it = 0; it < 64; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j) ld16(la + ((it * 16 + j * 112) & 495), b + 16 * j);
    wait_ld();
#pragma unroll
    for (int j = 0; j < 64; ++j) acc += b[j];
  }
  long long t2 = clock64();
  if (lane == 0) {
    out[warp * 8 + 0] = bad16;
    out[warp * 8 + 1] = bad4;
    out[warp * 8 + 2] = (uint32_t)(t1 - t0);
    out[warp * 8 + 3] = (uint32_t)(t2 - t1);
    out[warp * 8 + 4] = acc;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
  uint32_t* d;
  cudaMalloc(&d, 4096);
  int cases[][2] = {{0, 0}, {16, 4}, {3, 1}, {5, 2}, {77, 13}, {495, 507}};
  for (auto& cs : cases) {
    cudaMemset(d, 0xff, 4096);
    probe<<<1, 128>>>(cs[0], cs[1], d);
    cudaError_t e = cudaDeviceSynchronize();
    uint32_t h[32];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("{\"start16\": %d, \"start4\": %d, \"err\": \"%s\", \"bad16\": [%u,%u,%u,%u], \"bad4\": [%u,%u,%u,%u], "
           "\"x1_cycles_per_8\": %.1f, \"x16_cycles_per_4\": %.1f}\n",
           cs[0], cs[1], cudaGetErrorString(e), h[0], h[8], h[16], h[24], h[1], h[9], h[17], h[25], h[2] / 256.0,
           h[3] / 64.0);
    if (e != cudaSuccess) return 1;
  }
  return 0;
}
