// Issue-rate probes for the render kernel's integer / packed-FP32 mix
// (DESIGN.md §3.4): per-SMSP throughput of the ALU-pipe ops (PRMT, LOP3,
// LEA.HI, SHF, IADD3, I2IP), the FMA-pipe ops (IMAD, FFMA, FADD2, FFMA2),
// and 1:1 mixes of the two pipes (does the scheduler reach 1 instr/clk
// when both pipes are fed?).  Prints warp-instructions per clock per SMSP.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipes2 pipes2.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);      \
            return 1;                                                                           \
        }                                                                                       \
    } while (0)

constexpr int ITERS = 1024;
constexpr int CH = 8;

#define OP_PRMT(a, b) asm volatile("prmt.b32 %0, %0, %1, 0x5410;" : "+r"(a) : "r"(b))
#define OP_LOP3(a, b) asm volatile("lop3.b32 %0, %0, %1, %0, 0x96;" : "+r"(a) : "r"(b))
#define OP_SHF(a, b) asm volatile("shf.l.wrap.b32 %0, %0, %1, 7;" : "+r"(a) : "r"(b))
#define OP_IADD3(a, b) asm volatile("add.u32 %0, %0, %1;" : "+r"(a) : "r"(b))
#define OP_IMAD(a, b) asm volatile("mad.lo.u32 %0, %0, %1, %1;" : "+r"(a) : "r"(b))
#define OP_I2IP(a, b) asm volatile("cvt.pack.sat.u8.s32.b32 %0, %0, %1, %0;" : "+r"(a) : "r"(b))
#define OP_LEAHI(a, b) asm volatile("{.reg .s32 t; shr.s32 t, %0, 20; add.s32 %0, t, %1;}" : "+r"(a) : "r"(b))
#define OP_FFMA(a, b) asm volatile("fma.rn.f32 %0, %0, %1, %1;" : "+r"(a) : "r"(b))
#define OP_FADD(a, b) asm volatile("add.rn.f32 %0, %0, %1;" : "+r"(a) : "r"(b))

template <int KIND>
__global__ void k_int(uint32_t *out, uint32_t s) {
    uint32_t a[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) a[i] = threadIdx.x + i * 77u;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (KIND == 0) OP_PRMT(a[i], s);
            if (KIND == 1) OP_LOP3(a[i], s);
            if (KIND == 2) OP_SHF(a[i], s);
            if (KIND == 3) OP_IADD3(a[i], s);
            if (KIND == 4) OP_IMAD(a[i], s);
            if (KIND == 5) OP_I2IP(a[i], s);
            if (KIND == 6) OP_LEAHI(a[i], s);
            if (KIND == 7) OP_FFMA(a[i], s);
            if (KIND == 8) OP_FADD(a[i], s);
            // mixes: one FMA-pipe op + one ALU-pipe op per chain step
            if (KIND == 9) { if (i & 1) OP_IMAD(a[i], s); else OP_PRMT(a[i], s); }
            if (KIND == 10) { if (i & 1) OP_FFMA(a[i], s); else OP_LOP3(a[i], s); }
            if (KIND == 11) { if (i & 1) OP_IMAD(a[i], s); else OP_LEAHI(a[i], s); }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r ^= a[i];
    if (r == 0x12345678u) out[0] = r;
}

typedef unsigned long long u64;
template <int KIND>
__global__ void k_f2(u64 *out, u64 s, uint32_t t) {
    u64 a[CH];
    uint32_t b[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        a[i] = (u64)(threadIdx.x + i) * 0x3f8000003f800000ull;
        b[i] = threadIdx.x * 3u + i;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            if (KIND == 0) asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(s));
            if (KIND == 1) asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(a[i]) : "l"(s));
            if (KIND == 2) {  // FADD2 + PRMT
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(s));
                OP_PRMT(b[i], t);
            }
            if (KIND == 3) {  // FADD2 + 2 PRMT
                asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(a[i]) : "l"(s));
                OP_PRMT(b[i], t);
                OP_LOP3(b[i], t);
            }
        }
    }
    u64 r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i) r ^= a[i] ^ b[i];
    if (r == 0x12345678ull) out[0] = r;
}

int main() {
    cudaDeviceProp p;
    CK(cudaGetDeviceProperties(&p, 0));
    const int sms = p.multiProcessorCount;
    uint32_t *o;
    CK(cudaMalloc(&o, 64));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    const double mhz = 1965.0;
    const int threads = 512, blocks = sms * 4;  // 64 warps / SM
    auto run = [&](const char *name, auto launch, double instr_per_thread) {
        launch();
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0));
        for (int r = 0; r < 5; ++r) launch();
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        const double warp_instr = 5.0 * blocks * (threads / 32) * instr_per_thread;
        const double per_clk_smsp = warp_instr / (ms * 1e-3 * mhz * 1e6) / (sms * 4);
        printf("%-14s %6.3f warp-instr/clk/SMSP @%.0f MHz (%.3f ms)\n", name, per_clk_smsp, mhz, ms);
        return 0;
    };
    const double n1 = (double)ITERS * CH;
#define RI(K, NAME) run(NAME, [&] { k_int<K><<<blocks, threads>>>(o, 0x01020304u); }, n1)
    RI(0, "PRMT");
    RI(1, "LOP3");
    RI(2, "SHF");
    RI(3, "IADD");
    RI(4, "IMAD");
    RI(5, "I2IP");
    RI(6, "SHR+IADD");
    RI(7, "FFMA");
    RI(8, "FADD");
    RI(9, "IMAD|PRMT");
    RI(10, "FFMA|LOP3");
    RI(11, "IMAD|SHR+ADD");
    u64 *o2 = reinterpret_cast<u64 *>(o);
    const u64 s2 = 0x3f8000013f800001ull;
#define RF(K, NAME, M) run(NAME, [&] { k_f2<K><<<blocks, threads>>>(o2, s2, 0x01020304u); }, n1 *(M))
    RF(0, "FADD2", 1);
    RF(1, "FFMA2", 1);
    RF(2, "FADD2+PRMT", 2);
    RF(3, "FADD2+PRMT+LOP3", 3);
    CK(cudaGetLastError());
    return 0;
}
