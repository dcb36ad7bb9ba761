// tma_probe.cu -- minimal 3-D TMA load probe (development aid).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap map, float* out, int bw, int bh, int c0,
                      int c1, int c2)
{
    extern __shared__ __align__(128) unsigned char smem[];
    __shared__ uint64_t bar;
    const uint32_t b = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                     "r"(bw * bh * 4));
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
            "l"(reinterpret_cast<uint64_t>(&map)), "r"(c0), "r"(c1), "r"(c2), "r"(b)
            : "memory");
    }
    uint32_t ok = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n"
            " selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(b)
            : "memory");
    } while (!ok);
    const float* s = reinterpret_cast<const float*>(smem);
    for (int e = threadIdx.x; e < bw * bh; e += blockDim.x) out[e] = s[e];
}

int main(int argc, char** argv)
{
    const int Nu = 64, Nr = 64, Nv = 3, bw = 28, bh = 57;
    std::vector<float> h((size_t)Nu * Nr * Nv);
    for (size_t q = 0; q < h.size(); ++q) h[q] = (float)q;
    float *d, *o;
    cudaMalloc(&d, h.size() * 4);
    cudaMalloc(&o, bw * bh * 4);
    cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult qr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &qr);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fp;
    CUtensorMap map;
    memset(&map, 0, sizeof map);
    cuuint64_t dims[3] = {(cuuint64_t)Nu, (cuuint64_t)Nr, (cuuint64_t)Nv};
    cuuint64_t str[2] = {(cuuint64_t)Nu * 4, (cuuint64_t)Nu * 4 * Nr};
    cuuint32_t box[3] = {bw, bh, 1}, es[3] = {1, 1, 1};
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, d, dims, str, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d (query %d)\n", (int)r, (int)qr);
    int cs[1][3] = {{atoi(argv[1]), atoi(argv[2]), atoi(argv[3])}};
    for (auto& c : cs) {
        probe<<<1, 128, bw * bh * 4 + 128>>>(map, o, bw, bh, c[0], c[1], c[2]);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> got(bw * bh);
        cudaMemcpy(got.data(), o, got.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int y = 0; y < bh; ++y)
            for (int x = 0; x < bw; ++x) {
                int u = c[0] + x, v = c[1] + y;
                float ref = (u >= 0 && u < Nu && v >= 0 && v < Nr) ? h[((size_t)c[2] * Nr + v) * Nu + u] : 0.f;
                bad += got[y * bw + x] != ref;
            }
        printf("coords (%d,%d,%d): %s, %d mismatches\n", c[0], c[1], c[2], cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
