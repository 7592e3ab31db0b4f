// Probe of the tcgen05 kind::i8 path the render kernel's IDCT screen uses:
// K-major SWIZZLE_NONE shared-memory operands (core matrices of 8 rows x
// 16 B), M=128 rows, N = 16/32 outputs, K = 64 bytes (two K=32 steps),
// signed / unsigned operand formats from the instruction descriptor, int32
// accumulation in TMEM read back with tcgen05.ld.32x32b.  Checks D = A B^T
// against the host and prints PASS/FAIL per configuration.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o tc_i8_probe tc_i8_probe.cu
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// canonical K-major no-swizzle byte offset of (row r, byte k) in a tile
// with LBO = 128 B (K-adjacent core matrices) and SBO = 512 B (8-row groups)
__host__ __device__ inline int kmaj_off(int r, int k) { return (r >> 3) * 512 + (k >> 4) * 128 + (r & 7) * 16 + (k & 15); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3fff);
    d |= (uint64_t)((128 >> 4) & 0x3fff) << 16;   // LBO
    d |= (uint64_t)((512 >> 4) & 0x3fff) << 32;   // SBO
    d |= (uint64_t)1 << 46;                       // version (sm100)
    return d;                                     // base offset 0, layout SWIZZLE_NONE (0)
}
__host__ __device__ inline uint32_t idesc_i8(int n, bool a_signed, bool b_signed) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | ((b_signed ? 1u : 0u) << 10) | ((uint32_t)(n >> 3) << 17) |
           ((uint32_t)(128 >> 4) << 24);
}

template <int N>
__global__ void probe(const int8_t *A, const int8_t *B, int32_t *D, uint32_t idesc) {
    __shared__ __align__(1024) uint8_t sa[128 * 64];
    __shared__ __align__(1024) uint8_t sb[64 * 64];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 128 * 64; i += blockDim.x) sa[kmaj_off(i / 64, i % 64)] = (uint8_t)A[i];
    for (int i = tid; i < N * 64; i += blockDim.x) sb[kmaj_off(i / 64, i % 64)] = (uint8_t)B[i];
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = tbase;
    if (tid == 0) {
        for (int k = 0; k < 2; ++k) {
            const uint64_t da = sdesc(smem_u32(sa) + k * 256), db = sdesc(smem_u32(sb) + k * 256);
            const uint32_t acc = k > 0;
            asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                         "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                         "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            smem_u32(&mbar)));
    }
    // wait phase 0
    asm volatile("{\n.reg .pred P;\nW: mbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}" ::"r"(
        smem_u32(&mbar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    // lane = row; warp w reads lanes 32w..32w+31
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                       "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
                       "=r"(v[15])
                     : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        for (int j = 0; j < 16; ++j) D[tid * N + c0 + j] = (int32_t)v[j];
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
}

template <int N>
int run(bool as, bool bs) {
    int8_t *hA = new int8_t[128 * 64], *hB = new int8_t[N * 64];
    int32_t *hD = new int32_t[128 * N];
    srand(1 + N + 2 * as + 4 * bs);
    for (int i = 0; i < 128 * 64; ++i) hA[i] = (int8_t)(rand() & 0xff);
    for (int i = 0; i < N * 64; ++i) hB[i] = (int8_t)(rand() & 0xff);
    int8_t *dA, *dB;
    int32_t *dD;
    CK(cudaMalloc(&dA, 128 * 64));
    CK(cudaMalloc(&dB, N * 64));
    CK(cudaMalloc(&dD, 128 * N * 4));
    CK(cudaMemcpy(dA, hA, 128 * 64, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(dB, hB, N * 64, cudaMemcpyHostToDevice));
    probe<N><<<1, 128>>>(dA, dB, dD, idesc_i8(N, as, bs));
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(hD, dD, 128 * N * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            int64_t s = 0;
            for (int k = 0; k < 64; ++k) {
                const int a = as ? (int)hA[m * 64 + k] : (int)(uint8_t)hA[m * 64 + k];
                const int b = bs ? (int)hB[n * 64 + k] : (int)(uint8_t)hB[n * 64 + k];
                s += a * b;
            }
            if ((int32_t)s != hD[m * N + n]) {
                if (bad < 4) printf("  mismatch m=%d n=%d got %d want %lld\n", m, n, hD[m * N + n], (long long)s);
                ++bad;
            }
        }
    printf("N=%d A %s B %s: %s (%d bad)\n", N, as ? "s8" : "u8", bs ? "s8" : "u8", bad ? "FAIL" : "PASS", bad);
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dD);
    return bad != 0;
}

int main() {
    int f = 0;
    f |= run<32>(true, false);
    f |= run<32>(true, true);
    f |= run<32>(false, false);
    f |= run<16>(true, false);
    f |= run<64>(true, true);
    printf(f ? "SOME FAILED\n" : "ALL PASS\n");
    return f;
}
