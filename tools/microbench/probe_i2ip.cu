// Semantics + throughput probe for cvt.pack.sat.u8.s32.b32 (SASS I2IP),
// FRND (cvt.rmi.f32.f32) and PRMT on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void sem(unsigned *o) {
  unsigned d;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(0x11), "r"(0x22), "r"(0xAABBCCDD));
  o[0] = d;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(-5), "r"(300), "r"(0));
  o[1] = d;
  asm("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(0x33), "r"(0x44), "r"(0x1122));
  o[2] = d;
}
__global__ void thr_i2ip(unsigned *o, int s) {
  unsigned a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { unsigned d; asm volatile("cvt.pack.sat.u8.s32.b32 %0, %1, %2, %3;" : "=r"(d) : "r"(a[i]), "r"(s), "r"(a[i])); a[i] = d + it; }
  }
  unsigned r = 0; for (int i = 0; i < 8; ++i) r ^= a[i]; if (r == 12345) o[0] = r;
}
__global__ void thr_frnd(float *o, float s) {
  float a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i * 0.3f;
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { float d; asm volatile("cvt.rmi.f32.f32 %0, %1;" : "=f"(d) : "f"(a[i] * s)); a[i] = d + 0.5f; }
  }
  float r = 0; for (int i = 0; i < 8; ++i) r += a[i]; if (r == 1.2345f) o[0] = r;
}
__global__ void thr_prmt(unsigned *o, unsigned s) {
  unsigned a[8]; for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __byte_perm(a[i], s, 0x5140 + it);
  }
  unsigned r = 0; for (int i = 0; i < 8; ++i) r ^= a[i]; if (r == 12345) o[0] = r;
}
__global__ void thr_lds(unsigned *o, int s) {
  __shared__ unsigned long long t[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) t[i] = i;
  __syncthreads();
  unsigned long long acc = 0; unsigned idx = threadIdx.x * 7;
  for (int it = 0; it < 2048; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { unsigned long long v = t[(idx + i * 37) & 511]; acc += v; idx += (unsigned)v & 1; }
  }
  if (acc == 12345) o[0] = (unsigned)acc;
}
template <typename F> float tm(F f) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b); f(); cudaDeviceSynchronize();
  float best = 1e9; for (int r = 0; r < 5; ++r) { cudaEventRecord(a); f(); cudaEventRecord(b); cudaEventSynchronize(b); float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms; }
  return best;
}
int main() {
  unsigned *o; cudaMalloc(&o, 1 << 20); unsigned h[3];
  sem<<<1, 1>>>(o); cudaMemcpy(h, o, 12, cudaMemcpyDeviceToHost);
  printf("cvt.pack.sat.u8 (a=0x11,b=0x22,c=0xAABBCCDD) -> %08x\n", h[0]);
  printf("cvt.pack.sat.u8 (a=-5,b=300,c=0) -> %08x\n", h[1]);
  printf("cvt.pack.sat.u8 (a=0x33,b=0x44,c=0x1122) -> %08x\n", h[2]);
  int sms = 148, blocks = sms * 8, threads = 256; double ops = (double)blocks * threads * 2048 * 8;
  float ms = tm([&] { thr_i2ip<<<blocks, threads>>>(o, 3); });
  printf("I2IP   %.1f op/clk/SM\n", ops / (ms * 1e-3) / (sms * 1.965e9));
  ms = tm([&] { thr_frnd<<<blocks, threads>>>((float *)o, 1.0001f); });
  printf("FRND+FMUL+FADD %.1f iter/clk/SM\n", ops / (ms * 1e-3) / (sms * 1.965e9));
  ms = tm([&] { thr_prmt<<<blocks, threads>>>(o, 7); });
  printf("PRMT+IADD  %.1f iter/clk/SM\n", ops / (ms * 1e-3) / (sms * 1.965e9));
  ms = tm([&] { thr_lds<<<blocks, threads>>>(o, 7); });
  printf("LDS.64 random  %.1f loads/clk/SM\n", ops / (ms * 1e-3) / (sms * 1.965e9));
  return 0;
}
