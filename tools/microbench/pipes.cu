// Pipe-throughput microbenchmarks for the B200 design decisions in DESIGN.md:
// FP64 add/mul/fma, FP32 add/fma (reg + imm), packed FP32x2, int<->float
// conversions, integer ALU, and an HBM copy. Prints one line per probe:
//   name  Gop/s  ops/clk/SM (at the measured SM clock)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

constexpr int ITERS = 2048;
constexpr int CH = 8;   // independent chains per thread

__global__ void k_dadd(double* out, double s) {
  double a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __dadd_rn(a[i], s);
  }
  double r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678) out[0] = r;
}
__global__ void k_dmul(double* out, double s) {
  double a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __dmul_rn(a[i], s);
  }
  double r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678) out[0] = r;
}
__global__ void k_dfma(double* out, double s) {
  double a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __fma_rn(a[i], s, s);
  }
  double r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678) out[0] = r;
}
__global__ void k_fadd(float* out, float s) {
  float a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __fadd_rn(a[i], s);
  }
  float r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678f) out[0] = r;
}
__global__ void k_ffma(float* out, float s, float t) {
  float a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __fmaf_rn(a[i], s, t);
  }
  float r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678f) out[0] = r;
}
__global__ void k_ffma_imm(float* out) {
  float a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __fmaf_rn(a[i], 0.999f, 0.25f);
  }
  float r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678f) out[0] = r;
}
__device__ __forceinline__ unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d;
}
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d;
}
__global__ void k_fadd2(unsigned long long* out, unsigned long long s) {
  unsigned long long a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = fadd2(a[i], s);
  }
  unsigned long long r = 0; for (int i = 0; i < CH; ++i) r ^= a[i];
  if (r == 12345) out[0] = r;
}
__global__ void k_ffma2(unsigned long long* out, unsigned long long s) {
  unsigned long long a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = ffma2(a[i], s, s);
  }
  unsigned long long r = 0; for (int i = 0; i < CH; ++i) r ^= a[i];
  if (r == 12345) out[0] = r;
}
__global__ void k_iadd(int* out, int s) {
  int a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = (a[i] + s) ^ it;
  }
  int r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345) out[0] = r;
}
__global__ void k_i2f(float* out, int s) {
  float a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = 0.f;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __int2float_rn(__float_as_int(a[i]) + s);
  }
  float r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678f) out[0] = r;
}
__global__ void k_i2d(double* out, int s) {
  double a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = 0.0;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __int2double_rn(__double2loint(a[i]) + s);
  }
  double r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345.678) out[0] = r;
}
__global__ void k_f2i(int* out, float s) {
  int a[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) a[i] = i;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = __float2int_rd(__int_as_float(a[i]) * s);
  }
  int r = 0; for (int i = 0; i < CH; ++i) r += a[i];
  if (r == 12345) out[0] = r;
}
__global__ void k_copy(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (; i < n; i += stride) dst[i] = src[i];
}

template <typename F>
static float time_it(F launch, int reps = 5) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch(); cudaDeviceSynchronize();
  float best = 1e30f;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(a); launch(); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
  }
  return best;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  int sms = p.multiProcessorCount;
  printf("device %s sms %d clock_attr %d MHz\n", p.name, sms, clk_khz / 1000);
  void* buf; CK(cudaMalloc(&buf, 1 << 20));
  const int threads = 256, blocks = sms * 8;
  const double ops = (double)blocks * threads * ITERS * CH;
  auto report = [&](const char* name, float ms, double mult) {
    double gops = ops * mult / (ms * 1e-3) / 1e9;
    printf("%-10s %10.1f Gop/s  %7.2f op/clk/SM @1965MHz  (%.3f ms)\n", name, gops,
           gops * 1e9 / (sms * 1965e6), ms);
  };
  report("dadd", time_it([&] { k_dadd<<<blocks, threads>>>((double*)buf, 1.0000001); }), 1);
  report("dmul", time_it([&] { k_dmul<<<blocks, threads>>>((double*)buf, 1.0000001); }), 1);
  report("dfma", time_it([&] { k_dfma<<<blocks, threads>>>((double*)buf, 0.999999); }), 1);
  report("fadd", time_it([&] { k_fadd<<<blocks, threads>>>((float*)buf, 1.0001f); }), 1);
  report("ffma", time_it([&] { k_ffma<<<blocks, threads>>>((float*)buf, 0.999f, 0.25f); }), 1);
  report("ffma_imm", time_it([&] { k_ffma_imm<<<blocks, threads>>>((float*)buf); }), 1);
  report("fadd2(x2)", time_it([&] { k_fadd2<<<blocks, threads>>>((unsigned long long*)buf, 0x3f8000003f800000ull); }), 2);
  report("ffma2(x2)", time_it([&] { k_ffma2<<<blocks, threads>>>((unsigned long long*)buf, 0x3f7ff0003f7ff000ull); }), 2);
  report("iadd+lop", time_it([&] { k_iadd<<<blocks, threads>>>((int*)buf, 7); }), 2);
  report("i2f", time_it([&] { k_i2f<<<blocks, threads>>>((float*)buf, 1); }), 1);
  report("i2d", time_it([&] { k_i2d<<<blocks, threads>>>((double*)buf, 1); }), 1);
  report("f2i.rd", time_it([&] { k_f2i<<<blocks, threads>>>((int*)buf, 1.0001f); }), 1);
  size_t n = (size_t)1 << 30;  // 1 GiB each way
  void *s, *d; CK(cudaMalloc(&s, n)); CK(cudaMalloc(&d, n));
  cudaMemset(s, 1, n);
  for (int bpsm : {4, 8, 16}) {
    float ms = time_it([&] { k_copy<<<sms * bpsm, 512>>>((const int4*)s, (int4*)d, n / 16); });
    printf("copy int4 grid=%d*%d: %.1f GB/s (r+w)\n", sms, bpsm, 2.0 * n / (ms * 1e-3) / 1e9);
  }
  return 0;
}
