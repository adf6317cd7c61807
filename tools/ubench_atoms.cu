// Microbenchmark: shared-memory atomic (ATOMS.ADD) cost by lane-address pattern on B200.
// Each warp issues `iters` ATOMS over a 4096-word table; the pattern decides which lanes share
// an address or a bank.  Reports time per warp-ATOMS (SM cycles) so the insert kernel's lane
// map can be chosen from measurements instead of guesses.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_atoms tools/ubench_atoms.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void red_s(unsigned a, unsigned v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// pattern: address (word index) of lane l at iteration it
template <int P>
__device__ __forceinline__ unsigned addr_of(unsigned l, unsigned it, unsigned w) {
    const unsigned b = (it * 97u + w * 131u) & 1023u;
    if (P == 0) return b + l;                 // 32 distinct words, 32 distinct banks
    if (P == 1) return b + (l >> 1);          // pairs of lanes share a word (16 words, 16 banks)
    if (P == 2) return b + (l >> 2);          // 4 lanes per word
    if (P == 3) return b + 32 * (l & 1) + (l >> 1);   // 32 distinct words, 2 per bank
    if (P == 4) return b + 32 * (l & 3) + (l >> 2);   // 32 distinct words, 4 per bank
    if (P == 5) return b;                     // all lanes one word
    if (P == 6) return b + 33 * (l >> 2) + 4 * (l & 3);  // k_pnn_lin-like: 8 rows x 4 chunk cols, distinct
    if (P == 7) return b + (l >> 3);          // 8 lanes per word
    return 0;
}

template <int P, int ACTIVE>
__global__ void __launch_bounds__(128) kern(int iters, unsigned* sink) {
    __shared__ unsigned s[4096 + 2048];
    for (int i = threadIdx.x; i < 4096 + 2048; i += blockDim.x) s[i] = 0;
    __syncthreads();
    const unsigned base = (unsigned)__cvta_generic_to_shared(s);
    const unsigned l = threadIdx.x & 31, w = threadIdx.x >> 5;
    const bool act = ACTIVE >= 32 || (l % (32 / ACTIVE)) == 0;
    // addresses precomputed (8 sets), so the loop is ATOMS-bound rather than issue-bound
    unsigned ad[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) ad[q] = base + 4 * addr_of<P>(l, q, w);
    for (int it = 0; it < iters; it += 8) {
        if (ACTIVE >= 32) {
#pragma unroll
            for (int q = 0; q < 8; ++q) red_s(ad[q], l + q);
            continue;
        }
        {
            const unsigned a = addr_of<P>(l, it, w);
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p red.shared.add.u32 [%0], %1;\n\t}"
                         ::"r"(base + 4 * a), "r"(1u), "r"((unsigned)act) : "memory");
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) sink[blockIdx.x] = s[l];
}

template <int P, int ACTIVE>
void run(const char* name, unsigned* sink, int blocks, int iters, int sms, int clk_khz) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<P, ACTIVE><<<blocks, 128>>>(iters, sink);
    cudaEventRecord(a);
    kern<P, ACTIVE><<<blocks, 128>>>(iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    const double warp_ops = (double)blocks * 4 * (ACTIVE >= 32 ? iters : iters / 8);
    const double cyc = ms * 1e-3 * clk_khz * 1e3 * sms / warp_ops;
    printf("%-28s active %2d  %8.3f ms  %6.2f SM-cycles per warp-ATOMS  %7.1f G lane-ops/s\n", name,
           ACTIVE, ms, cyc, warp_ops * ACTIVE / ms / 1e6);
}

int main() {
    unsigned* sink;
    cudaMalloc(&sink, sizeof(unsigned) << 20);
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int blocks = sms * 8, iters = 4096;
    run<0, 32>("distinct words+banks", sink, blocks, iters, sms, clk);
    run<1, 32>("2 lanes/word", sink, blocks, iters, sms, clk);
    run<2, 32>("4 lanes/word", sink, blocks, iters, sms, clk);
    run<7, 32>("8 lanes/word", sink, blocks, iters, sms, clk);
    run<5, 32>("32 lanes/word", sink, blocks, iters, sms, clk);
    run<3, 32>("2 words/bank", sink, blocks, iters, sms, clk);
    run<4, 32>("4 words/bank", sink, blocks, iters, sms, clk);
    run<6, 32>("8x4 stride33", sink, blocks, iters, sms, clk);
    run<0, 8>("distinct, 8 active", sink, blocks, iters, sms, clk);
    run<2, 8>("4 lanes/word, 8 active", sink, blocks, iters, sms, clk);
    run<0, 16>("distinct, 16 active", sink, blocks, iters, sms, clk);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s, SMs %d, clock %d kHz\n", cudaGetErrorString(e), sms, clk);
    return e == cudaSuccess ? 0 : 1;
}
