// Minimal TMA probe: load one (130 x 18) u64 box with cp.async.bulk.tensor.3d and report the sum.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>
#include <cstdlib>
typedef unsigned long long ull;
template <int VARIANT>
__global__ void k(const __grid_constant__ CUtensorMap tmap, ull* out, int x, int y, int z) {
    extern __shared__ __align__(128) unsigned char sm[];
    __shared__ __align__(8) ull bar;
    unsigned b = (unsigned)__cvta_generic_to_shared(&bar), d = (unsigned)__cvta_generic_to_shared(sm);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(b), "r"(1) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(130 * 18 * 8) : "memory");
        if (VARIANT == 0)
            asm volatile("cp.async.bulk.tensor.3d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                         ::"r"(d), "l"(&tmap), "r"(b), "r"(x), "r"(y), "r"(z) : "memory");
        else
            asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                         ::"r"(d), "l"(&tmap), "r"(b), "r"(x), "r"(y), "r"(z) : "memory");
    }
    asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(b), "r"(0) : "memory");
    ull s = 0;
    const ull* v = reinterpret_cast<const ull*>(sm);
    for (int i = threadIdx.x; i < 130 * 18; i += blockDim.x) s += v[i];
    atomicAdd(out, s);
}
int main(int argc, char** argv) {
    const int variant_sel = atoi(argv[1]), xs = atoi(argv[2]), ys = atoi(argv[3]), zs = atoi(argv[4]);
    const int nx = 500, ny = 267, nz = 40;
    std::vector<ull> h((size_t)nx * ny * nz);
    for (size_t i = 0; i < h.size(); ++i) h[i] = i % 7;
    ull *d, *o;
    cudaMalloc(&d, h.size() * 8);
    cudaMalloc(&o, 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
    using Encode = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    CUtensorMap m;
    cuuint64_t dims[3] = {nx, ny, nz}, str[2] = {nx * 8ull, (cuuint64_t)nx * ny * 8};
    cuuint32_t box[3] = {130, 18, 1}, es[3] = {1, 1, 1};
    CUresult r = ((Encode)fn)(&m, CU_TENSOR_MAP_DATA_TYPE_UINT64, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d (query %d)\n", (int)r, (int)q);
    {
        int variant = variant_sel, c = 0, x = xs, y = ys, z = zs;
        {
            cudaMemset(o, 0, 8);
            if (variant == 0) k<0><<<1, 128, 130 * 18 * 8>>>(m, o, x, y, z);
            else k<1><<<1, 128, 130 * 18 * 8>>>(m, o, x, y, z);
            cudaError_t e = cudaDeviceSynchronize();
            ull got = 0;
            cudaMemcpy(&got, o, 8, cudaMemcpyDeviceToHost);
            ull want = 0;
            for (int yy = y; yy < y + 18; ++yy)
                for (int xx = x; xx < x + 130; ++xx)
                    if (xx >= 0 && yy >= 0 && z >= 0 && xx < nx && yy < ny && z < nz) want += h[((size_t)z * ny + yy) * nx + xx];
            printf("variant %d (%d,%d,%d): %s got %llu want %llu\n", variant, x, y, z, cudaGetErrorString(e), got, want);
            if (e != cudaSuccess) return 1;
        }
    }
    return 0;
}
