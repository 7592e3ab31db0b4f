// Latency of one render-kernel "unit" on the tensor cores: n_mma dependent /
// independent kind::i8 MMAs (M=128, N, K=32 each) + commit + mbarrier wait,
// timed by the issuing thread with clock64 (1 CTA, 128 threads; 200 reps).
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_1311_5304_b200/csrc/hj_tc.cuh"
using namespace hj;

template <int N, int NMMA, int CHAINS>
__global__ void lat(long long *out) {
    __shared__ __align__(1024) uint8_t sa[128 * 64];
    __shared__ __align__(1024) uint8_t sb[3 * 64 * 64];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x;
    for (int i = tid; i < 128 * 64; i += blockDim.x) sa[i] = (uint8_t)i;
    for (int i = tid; i < 3 * 64 * 64; i += blockDim.x) sb[i] = (uint8_t)(i * 7);
    if (tid == 0) { tc::mbar_init(&mbar, 1); asm volatile("fence.mbarrier_init.release.cluster;"); }
    if (tid < 32) tc::tmem_alloc<256>(&tbase);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tm = tbase;
    long long tot = 0, best = 1ll << 60;
    for (int rep = 0; rep < 200; ++rep) {
        if (tid == 0) {
            const long long t0 = clock64();
            for (int m = 0; m < NMMA; ++m) {
                const int ch = m % CHAINS, ks = (m / CHAINS) & 1;
                tc::mma_i8(tm + (ch * N) % 256, tc::sdesc(tc::smem_u32(sa) + ks * 256),
                           tc::sdesc(tc::smem_u32(sb) + (N > 64 ? 0 : (ch % 3) * 4096) + ks * 256), tc::idesc_i8(N, true, false),
                           (m / CHAINS) > 0);
            }
            tc::commit(&mbar);
            tc::mbar_wait(&mbar, rep & 1);
            const long long dt = clock64() - t0;
            tot += dt;
            best = dt < best ? dt : best;
        }
        __syncthreads();
    }
    if (tid == 0) { out[0] = tot / 200; out[1] = best; }
    tc::fence_before();
    __syncthreads();
    if (tid < 32) tc::tmem_free<256>(tm);
}

template <int N, int NMMA, int CHAINS>
void run(const char *name) {
    long long *d, h[2];
    cudaMalloc(&d, 16);
    lat<N, NMMA, CHAINS><<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("%-34s N=%3d mmas=%2d chains=%d: mean %lld clk, best %lld clk (%s)\n", name, N, NMMA, CHAINS, h[0], h[1],
           cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<32, 1, 1>("single MMA");
    run<32, 6, 3>("Y unit (3 limbs x 2 k)");
    run<16, 12, 6>("chroma unit (2 comps x 3 x 2 k)");
    run<64, 6, 3>("Y full tile N=64");
    run<16, 6, 3>("N=16 x 6");
    run<128, 2, 1>("N=128 x2");
    run<32, 24, 6>("24 MMAs N=32");
    run<96, 2, 1>("N=96 limb-stacked x2 (Y half)");
    run<96, 4, 2>("N=96 x4 (two halves)");
    run<192, 2, 1>("N=192 x2");
    return 0;
}
