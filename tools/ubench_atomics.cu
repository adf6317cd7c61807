// Microbenchmark: lane-atomic throughput on B200 for the insert kernel's design choices.
//   red64_spread   : RED.E.ADD.64 to pseudo-random addresses in a 1 MiB window (L2-resident)
//   red64_run      : RED.64 where 4 consecutive lanes share an address (run-like)
//   atoms32_spread : shared-memory atomicAdd (u32) to pseudo-random slots of a 16 KiB table
//   atoms32_run    : shared atomics, 4 lanes per address
//   sts32_spread   : plain shared stores, same pattern (LSU reference)
//   red64_256MiB   : RED.64 spread over 256 MiB (DRAM read-modify-write)
//   red64_warp64w  : a warp's lanes within 64 words of a random per-warp base, 256 MiB window
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_atomics tools/ubench_atomics.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash32(unsigned x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

template <int MODE>
__global__ void __launch_bounds__(256) kern(unsigned long long* g, int iters, unsigned long long* sink) {
    __shared__ unsigned s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = 0;
    __syncthreads();
    unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
    unsigned lane = threadIdx.x & 31;
    unsigned long long acc = 0;
    for (int it = 0; it < iters; ++it) {
        unsigned key = (MODE == 1 || MODE == 3) ? hash32((t >> 2) * 977u + it) : hash32(t * 131u + it);
        if (MODE == 0 || MODE == 1) atomicAdd(&g[key & ((1u << 17) - 1)], 1ull);
        if (MODE == 2 || MODE == 3) atomicAdd(&s[key & 4095], 1u);
        if (MODE == 4) s[key & 4095] = key;
        if (MODE == 5) atomicAdd(&g[(key % 30000u) * 7u % (1u << 17)], 1ull);  // hot 30k-address set
        if (MODE == 6) atomicAdd(&g[(t >> 3) % 30000u], 1ull);                  // 8 lanes/address
        if (MODE == 7) atomicAdd(&g[key & ((1u << 25) - 1)], 1ull);             // 256 MiB window
        if (MODE == 8)  // warp-local: lanes within 64 words of a per-warp random base (sector sharing)
            atomicAdd(&g[((hash32((t >> 5) * 31u + it) & ((1u << 25) - 1)) + (hash32(t + it) & 63u)) & ((1u << 25) - 1)], 1ull);
        if (MODE == 9)  // a warp's lanes on 32 consecutive words (8 sectors) at a random base, 1 MiB window
            atomicAdd(&g[((hash32((t >> 5) * 31u + it) << 5) + lane) & ((1u << 17) - 1)], 1ull);
        if (MODE == 10)  // the same in a 256 MiB window
            atomicAdd(&g[((hash32((t >> 5) * 31u + it) << 5) + lane) & ((1u << 25) - 1)], 1ull);
        if (MODE == 11)  // 2 lanes per word, 16 consecutive words (4 sectors), 1 MiB window
            atomicAdd(&g[((hash32((t >> 5) * 31u + it) << 5) + (lane >> 1)) & ((1u << 17) - 1)], 1ull);
        // 2 GiB window (every sector misses L2): RED alone, RED after an L2 prefetch issued PF
        // iterations earlier, plain loads, prefetches alone
        constexpr unsigned W28 = (1u << 28) - 1;
        if (MODE == 12) atomicAdd(&g[hash32(t * 131u + it) & W28], 1ull);
        if (MODE == 13 || MODE == 15 || MODE == 16) {
            constexpr int PF = MODE == 13 ? 8 : (MODE == 15 ? 2 : 32);
            asm volatile("prefetch.global.L2 [%0];" ::"l"(&g[hash32(t * 131u + it + PF) & W28]));
            atomicAdd(&g[hash32(t * 131u + it) & W28], 1ull);
        }
        if (MODE == 14) acc += g[hash32(t * 131u + it) & W28];
        // float2 (red.global.add.v2.f32, the trilinear splat's atomic): one lane per sector in a
        // 1 MiB window; a warp on 32 consecutive pairs (8 sectors); 4 lanes per sector, sectors apart
        if (MODE == 18) atomicAdd(reinterpret_cast<float2*>(g) + (hash32(t * 131u + it) & ((1u << 17) - 1)), make_float2(1.f, 1.f));
        if (MODE == 19) atomicAdd(reinterpret_cast<float2*>(g) + (((hash32((t >> 5) * 31u + it) << 5) + lane) & ((1u << 17) - 1)), make_float2(1.f, 1.f));
        if (MODE == 20) atomicAdd(reinterpret_cast<float2*>(g) + (hash32(t * 131u + it) & W28), make_float2(1.f, 1.f));
        if (MODE == 17) asm volatile("prefetch.global.L2 [%0];" ::"l"(&g[hash32(t * 131u + it) & W28]));
    }
    __syncthreads();
    if (MODE == 14 && acc == 0x123456789ull) sink[t] = acc;
    if (MODE >= 2 && MODE < 12 && threadIdx.x == 0) sink[blockIdx.x] = s[lane];
}

template <int MODE>
float run(const char* name, unsigned long long* g, unsigned long long* sink, int blocks, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    kern<MODE><<<blocks, 256>>>(g, iters, sink);
    cudaEventRecord(a);
    kern<MODE><<<blocks, 256>>>(g, iters, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * 256 * iters;
    printf("%-16s %8.3f ms  %8.1f G lane-ops/s\n", name, ms, ops / ms / 1e6);
    return ms;
}

int main() {
    unsigned long long *g, *sink;
    cudaMalloc(&g, sizeof(unsigned long long) << 28);
    cudaMalloc(&sink, sizeof(unsigned long long) << 20);
    cudaMemset(g, 0, sizeof(unsigned long long) << 28);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int blocks = sms * 8, iters = 512;
    run<0>("red64_spread", g, sink, blocks, iters);
    run<1>("red64_run4", g, sink, blocks, iters);
    run<2>("atoms32_spread", g, sink, blocks, iters);
    run<3>("atoms32_run4", g, sink, blocks, iters);
    run<4>("sts32_spread", g, sink, blocks, iters);
    run<5>("red64_hot30k", g, sink, blocks, iters);
    run<6>("red64_same8", g, sink, blocks, iters);
    run<7>("red64_256MiB", g, sink, blocks, iters);
    run<8>("red64_warp64w", g, sink, blocks, iters);
    run<9>("red64_coal_1MiB", g, sink, blocks, iters);
    run<10>("red64_coal_256M", g, sink, blocks, iters);
    run<11>("red64_pair_1MiB", g, sink, blocks, iters);
    run<12>("red64_2GiB", g, sink, blocks, iters);
    run<15>("red64_2GiB_pf2", g, sink, blocks, iters);
    run<13>("red64_2GiB_pf8", g, sink, blocks, iters);
    run<16>("red64_2GiB_pf32", g, sink, blocks, iters);
    run<14>("ld64_2GiB", g, sink, blocks, iters);
    run<17>("pf_2GiB", g, sink, blocks, iters);
    run<18>("redf2_spread_1M", g, sink, blocks, iters);
    run<19>("redf2_coal_1M", g, sink, blocks, iters);
    run<20>("redf2_2GiB", g, sink, blocks, iters);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s, SMs %d\n", cudaGetErrorString(e), sms);
    return e == cudaSuccess ? 0 : 1;
}
