// Throughput microbenchmarks that decide the filter's arithmetic/storage design
// on B200 (sm_100a): FP64 add/FMA, fp32<->fp64 and int<->fp32 conversions,
// shared-memory load bandwidth, tcgen05.ld (TMEM) load bandwidth, HBM copy.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o microbench microbench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 4096;

__global__ void k_dadd(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    x0 += a; x1 += b; x2 += a; x3 += b; x4 += a; x5 += b; x6 += a; x7 += b;
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[0] = x0;
}

__global__ void k_dfma(double* out, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345) out[0] = x0;
}

__global__ void k_ffma(float* out, float a, float b) {
  float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
    x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 1.2345f) out[0] = x0;
}

__global__ void k_iadd3(int* out, int a, int b) {
  int x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  int c0 = a * threadIdx.x, c1 = c0 + b, c2 = c1 + b, c3 = c2 + b, c4 = c3 + b, c5 = c4 + b, c6 = c5 + b, c7 = c6 + b;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    x0 = x0 + c0 - i; x1 = x1 + c1 - i; x2 = x2 + c2 - i; x3 = x3 + c3 - i;
    x4 = x4 + c4 - i; x5 = x5 + c5 - i; x6 = x6 + c6 - i; x7 = x7 + c7 - i;
  }
  if (x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7 == 12345) out[0] = x0;
}

// fp32 -> fp64 conversion: 8 independent conversions per iteration, results summed in fp64
// would add DADDs, so fold them with integer xor of the high words instead.
__global__ void k_f2f_up(int* out, float a) {
  float f0 = threadIdx.x * a, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3, f4 = f0 + 4, f5 = f0 + 5, f6 = f0 + 6, f7 = f0 + 7;
  int acc = 0;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    acc ^= __double2hiint((double)f0) ^ __double2hiint((double)f1) ^ __double2hiint((double)f2) ^ __double2hiint((double)f3)
         ^ __double2hiint((double)f4) ^ __double2hiint((double)f5) ^ __double2hiint((double)f6) ^ __double2hiint((double)f7);
    f0 = __int_as_float(__float_as_int(f0) ^ acc & 1); f1 = __int_as_float(__float_as_int(f1) ^ acc & 2);
    f2 = __int_as_float(__float_as_int(f2) ^ acc & 4); f3 = __int_as_float(__float_as_int(f3) ^ acc & 8);
    f4 = __int_as_float(__float_as_int(f4) ^ acc & 16); f5 = __int_as_float(__float_as_int(f5) ^ acc & 32);
    f6 = __int_as_float(__float_as_int(f6) ^ acc & 64); f7 = __int_as_float(__float_as_int(f7) ^ acc & 128);
  }
  if (acc == 12345) out[0] = acc;
}

__global__ void k_f2f_down(int* out, double a) {
  double d0 = threadIdx.x * a, d1 = d0 + 1, d2 = d0 + 2, d3 = d0 + 3, d4 = d0 + 4, d5 = d0 + 5, d6 = d0 + 6, d7 = d0 + 7;
  int acc = 0;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    acc ^= __float_as_int((float)d0) ^ __float_as_int((float)d1) ^ __float_as_int((float)d2) ^ __float_as_int((float)d3)
         ^ __float_as_int((float)d4) ^ __float_as_int((float)d5) ^ __float_as_int((float)d6) ^ __float_as_int((float)d7);
    d0 = __hiloint2double(__double2hiint(d0), acc & 1); d1 = __hiloint2double(__double2hiint(d1), acc & 2);
    d2 = __hiloint2double(__double2hiint(d2), acc & 4); d3 = __hiloint2double(__double2hiint(d3), acc & 8);
    d4 = __hiloint2double(__double2hiint(d4), acc & 16); d5 = __hiloint2double(__double2hiint(d5), acc & 32);
    d6 = __hiloint2double(__double2hiint(d6), acc & 64); d7 = __hiloint2double(__double2hiint(d7), acc & 128);
  }
  if (acc == 12345) out[0] = acc;
}

__global__ void k_i2f(int* out, int a) {
  int i0 = threadIdx.x * a, i1 = i0 + 1, i2 = i0 + 2, i3 = i0 + 3, i4 = i0 + 4, i5 = i0 + 5, i6 = i0 + 6, i7 = i0 + 7;
  int acc = 0;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    acc ^= __float_as_int((float)i0) ^ __float_as_int((float)i1) ^ __float_as_int((float)i2) ^ __float_as_int((float)i3)
         ^ __float_as_int((float)i4) ^ __float_as_int((float)i5) ^ __float_as_int((float)i6) ^ __float_as_int((float)i7);
    i0 ^= acc & 1; i1 ^= acc & 2; i2 ^= acc & 4; i3 ^= acc & 8; i4 ^= acc & 16; i5 ^= acc & 32; i6 ^= acc & 64; i7 ^= acc & 128;
  }
  if (acc == 12345) out[0] = acc;
}

__global__ void k_f2i(int* out, float a) {
  float f0 = threadIdx.x * a, f1 = f0 + 1, f2 = f0 + 2, f3 = f0 + 3, f4 = f0 + 4, f5 = f0 + 5, f6 = f0 + 6, f7 = f0 + 7;
  int acc = 0;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    acc ^= __float2int_rn(f0) ^ __float2int_rn(f1) ^ __float2int_rn(f2) ^ __float2int_rn(f3)
         ^ __float2int_rn(f4) ^ __float2int_rn(f5) ^ __float2int_rn(f6) ^ __float2int_rn(f7);
    f0 = __int_as_float(__float_as_int(f0) ^ acc & 1); f1 = __int_as_float(__float_as_int(f1) ^ acc & 2);
    f2 = __int_as_float(__float_as_int(f2) ^ acc & 4); f3 = __int_as_float(__float_as_int(f3) ^ acc & 8);
    f4 = __int_as_float(__float_as_int(f4) ^ acc & 16); f5 = __int_as_float(__float_as_int(f5) ^ acc & 32);
    f6 = __int_as_float(__float_as_int(f6) ^ acc & 64); f7 = __int_as_float(__float_as_int(f7) ^ acc & 128);
  }
  if (acc == 12345) out[0] = acc;
}

// Shared-memory load bandwidth: each thread reads lagged words of a ring (conflict-free).
template <int VEC>
__global__ void k_lds(int* out, int lagmix) {
  extern __shared__ int4 smem4[];
  int* s = reinterpret_cast<int*>(smem4);
  const int n = 16384;  // 64 KB
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = i * 7;
  __syncthreads();
  int acc = 0;
  int base = threadIdx.x * VEC;
#pragma unroll 4
  for (int i = 0; i < ITERS; ++i) {
    int off = (base + (i * 8 + (acc & lagmix)) * 32 * VEC) & (n - 1);
    if (VEC == 1) {
      acc += s[off] + s[(off + 1024) & (n - 1)] + s[(off + 2048) & (n - 1)] + s[(off + 3072) & (n - 1)];
    } else {
      int4 a = smem4[off >> 2], b = smem4[((off + 1024) & (n - 1)) >> 2];
      int4 c = smem4[((off + 2048) & (n - 1)) >> 2], d = smem4[((off + 3072) & (n - 1)) >> 2];
      acc += a.x ^ a.y ^ a.z ^ a.w ^ b.x ^ b.y ^ b.z ^ b.w ^ c.x ^ c.y ^ c.z ^ c.w ^ d.x ^ d.y ^ d.z ^ d.w;
    }
  }
  if (acc == 12345) out[0] = acc;
}

// TMEM: allocate 512 columns, store, then each thread streams tcgen05.ld.32x32b.xN from its lane.
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t addr, uint32_t* v);
template <>
__device__ __forceinline__ void tmem_ld<1>(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v[0]) : "r"(addr));
}
template <>
__device__ __forceinline__ void tmem_ld<4>(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]) : "r"(addr));
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t addr, uint32_t* v) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                 "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
               : "r"(addr));
}

template <int N>
__global__ void k_tmem(int* out, int lagmix) {
  __shared__ uint32_t tmem_base_s;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;"
                 :: "r"((uint32_t)__cvta_generic_to_shared(&tmem_base_s)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t base = tmem_base_s;
  const uint32_t lane_addr = base + ((uint32_t)((warp & 3) * 32) << 16);
  // initialise all 512 columns of this warp's 32 lanes (warps 4..7 alias 0..3; harmless)
  for (int c = 0; c < 512; ++c) {
    uint32_t v = c * 3 + threadIdx.x;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" :: "r"(lane_addr + c), "r"(v));
  }
  asm volatile("tcgen05.wait::st.sync.aligned;");
  uint32_t acc = 0;
  uint32_t v[N];
  for (int i = 0; i < ITERS; ++i) {
    uint32_t col = ((uint32_t)(i * 37) + (acc & lagmix)) & (512 - 4 * N);
    tmem_ld<N>(lane_addr + col, v);
    tmem_ld<N>(lane_addr + ((col + 128) & (512 - 4 * N)), v + 0);
    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
    for (int j = 0; j < N; ++j) acc ^= v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" :: "r"(base));
  }
  if (acc == 12345u) out[0] = acc;
}

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) b[i] = a[i];
}

__global__ void k_clock(long long* out, int spin) {
  long long t0 = clock64();
  volatile int x = 0;
  for (int i = 0; i < spin; ++i) x = x + 1;
  if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
}

int main() {
  int dev = 0;
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, dev));
  int sms = prop.multiProcessorCount;
  int l2 = prop.l2CacheSize;
  int smem_optin = 0;
  CK(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"smem_optin\": %d, \"clock_khz_attr\": %d}\n",
         prop.name, sms, l2, smem_optin, clk_khz);
  int* d_out; CK(cudaMalloc(&d_out, 1 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;

  // measure SM clock: cycles / wall time for a spin kernel
  long long* d_clk; CK(cudaMalloc(&d_clk, sizeof(long long) * sms));
  k_clock<<<sms, 32>>>(d_clk, 1 << 20);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  k_clock<<<sms, 32>>>(d_clk, 1 << 22);
  cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1);
  long long cyc; CK(cudaMemcpy(&cyc, d_clk, sizeof(long long), cudaMemcpyDeviceToHost));
  double ghz = cyc / (ms * 1e6);
  printf("{\"test\": \"clock\", \"ghz_est\": %.3f}\n", ghz);

  auto run = [&](const char* name, auto launch, double ops_per_thread, int blocks, int threads) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    double ops = ops_per_thread * blocks * (double)threads * 5;
    double per_clk_sm = ops / (ms * 1e-3) / (ghz * 1e9) / sms;
    printf("{\"test\": \"%s\", \"ms\": %.3f, \"lane_ops_per_clk_per_sm\": %.2f, \"err\": \"%s\"}\n",
           name, ms, per_clk_sm, cudaGetErrorString(err));
  };
  const int B = sms * 8, T = 256;
  const double O = 8.0 * ITERS;
  run("dadd", [&] { k_dadd<<<B, T>>>((double*)d_out, 1.0, 2.0); }, O, B, T);
  run("dfma", [&] { k_dfma<<<B, T>>>((double*)d_out, 1.0000001, 1e-9); }, O, B, T);
  run("ffma", [&] { k_ffma<<<B, T>>>((float*)d_out, 1.0000001f, 1e-9f); }, O, B, T);
  run("iadd3", [&] { k_iadd3<<<B, T>>>(d_out, 3, 5); }, O, B, T);
  run("f2f_f32_to_f64", [&] { k_f2f_up<<<B, T>>>(d_out, 1.5f); }, O, B, T);
  run("f2f_f64_to_f32", [&] { k_f2f_down<<<B, T>>>(d_out, 1.5); }, O, B, T);
  run("i2f_s32_to_f32", [&] { k_i2f<<<B, T>>>(d_out, 3); }, O, B, T);
  run("f2i_f32_to_s32", [&] { k_f2i<<<B, T>>>(d_out, 1.5f); }, O, B, T);
  // lds: ops counted as 32-bit words read
  CK(cudaFuncSetAttribute(k_lds<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  CK(cudaFuncSetAttribute(k_lds<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536));
  run("lds32_words", [&] { k_lds<1><<<sms * 2, 512, 65536>>>(d_out, 0); }, 4.0 * ITERS, sms * 2, 512);
  run("lds128_words", [&] { k_lds<4><<<sms * 2, 512, 65536>>>(d_out, 0); }, 16.0 * ITERS, sms * 2, 512);
  // tmem: words per thread = 2 * N per iteration
  run("tmem_ld_x1_words", [&] { k_tmem<1><<<sms, 128>>>(d_out, 0); }, 2.0 * 1 * ITERS, sms, 128);
  run("tmem_ld_x4_words", [&] { k_tmem<4><<<sms, 128>>>(d_out, 0); }, 2.0 * 4 * ITERS, sms, 128);
  run("tmem_ld_x16_words", [&] { k_tmem<16><<<sms, 128>>>(d_out, 0); }, 2.0 * 16 * ITERS, sms, 128);
  run("tmem_ld_x4_words_8w", [&] { k_tmem<4><<<sms, 256>>>(d_out, 0); }, 2.0 * 4 * ITERS, sms, 256);
  run("tmem_ld_x16_words_8w", [&] { k_tmem<16><<<sms, 256>>>(d_out, 0); }, 2.0 * 16 * ITERS, sms, 256);

  // HBM copy
  size_t nbytes = (size_t)2 << 30;
  float4 *a, *b;
  CK(cudaMalloc(&a, nbytes)); CK(cudaMalloc(&b, nbytes));
  cudaMemset(a, 0, nbytes);
  size_t n4 = nbytes / 16;
  k_copy<<<sms * 8, 512>>>(a, b, n4);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k_copy<<<sms * 8, 512>>>(a, b, n4);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  printf("{\"test\": \"hbm_copy\", \"gbs\": %.1f}\n", 2.0 * nbytes * 5 / (ms * 1e-3) / 1e9);
  CK(cudaGetLastError());
  return 0;
}
