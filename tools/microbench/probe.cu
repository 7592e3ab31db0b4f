// check ptx f32x2 syntax
__global__ void k(float2* p, float a){
  float2 v = p[threadIdx.x];
  unsigned long long x = *reinterpret_cast<unsigned long long*>(&v);
  unsigned long long y;
  asm("add.rn.f32x2 %0, %1, %1;" : "=l"(y) : "l"(x));
  asm("fma.rn.f32x2 %0, %1, %1, %1;" : "=l"(y) : "l"(y));
  asm("mul.rn.f32x2 %0, %1, %1;" : "=l"(y) : "l"(y));
  p[threadIdx.x] = *reinterpret_cast<float2*>(&y);
}
