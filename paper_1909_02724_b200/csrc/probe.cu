// probe.cu -- libifdk_probe.so: the shared-memory gather micro-benchmark behind the BP
// roofline ("measure it on the box with a shared-memory gather micro-benchmark
// at the clock the BP actually runs").  Not part of the FDK path; bench.py calls it once.
//
// Every warp issues conflict-free LDS.64 (the BP kernel's tap load: 32 lanes x 8 B = two
// 128-byte wavefronts) back to back, 8 independent loads in flight per thread, with the
// BP kernel's occupancy (2 CTAs x 256 threads per SM).  The result is the shared-memory
// crossbar bandwidth in bytes/s over the whole GPU.
#include <cuda_runtime.h>

#include <cstdint>

namespace {

constexpr int kThreads = 256, kWords = 8192;  // 64 KB of float2 per CTA

__global__ void __launch_bounds__(kThreads, 2) smem_gather(float* out, int iters, uint32_t stride)
{
    __shared__ float2 buf[kWords / 2];
    for (int q = threadIdx.x; q < kWords / 2; q += kThreads)
        buf[q] = make_float2((float)q, 1.f);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // lane l reads float2 slot base + l: 32 consecutive 8-byte slots, no bank conflict
    uint32_t base = (uint32_t)(warp * 512);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f, a4 = 0.f, a5 = 0.f, a6 = 0.f, a7 = 0.f;
    for (int it = 0; it < iters; ++it) {
        // stride arrives at run time (256 slots): the compiler cannot prove two iterations'
        // addresses equal, so no load is merged away
        const uint32_t b = (base + (uint32_t)it * stride) & (kWords / 2 - 1) & ~31u;
        float2 v0 = buf[(b + lane) & (kWords / 2 - 1)];
        float2 v1 = buf[(b + 32 + lane) & (kWords / 2 - 1)];
        float2 v2 = buf[(b + 64 + lane) & (kWords / 2 - 1)];
        float2 v3 = buf[(b + 96 + lane) & (kWords / 2 - 1)];
        float2 v4 = buf[(b + 128 + lane) & (kWords / 2 - 1)];
        float2 v5 = buf[(b + 160 + lane) & (kWords / 2 - 1)];
        float2 v6 = buf[(b + 192 + lane) & (kWords / 2 - 1)];
        float2 v7 = buf[(b + 224 + lane) & (kWords / 2 - 1)];
        a0 += v0.x + v0.y; a1 += v1.x + v1.y; a2 += v2.x + v2.y; a3 += v3.x + v3.y;
        a4 += v4.x + v4.y; a5 += v5.x + v5.y; a6 += v6.x + v6.y; a7 += v7.x + v7.y;
    }
    const float s = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
    if (s == -1.f) out[blockIdx.x] = s;  // never true; keeps the loads alive
}

}  // namespace

// Shared-memory gather bandwidth (bytes/s, whole GPU) on the current device, and the kernel
// time in ms.  Returns 0 on success, the cudaError_t otherwise.
extern "C" int ifdk_probe_smem_bandwidth(double* bytes_per_s, double* ms_out)
{
    int dev = 0, sms = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (e != cudaSuccess) return (int)e;
    float* out = nullptr;
    if ((e = cudaMalloc(&out, sizeof(float) * 4096)) != cudaSuccess) return (int)e;
    const int grid = sms * 2, iters = 1 << 15;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    smem_gather<<<grid, kThreads>>>(out, 256, 256u);  // warm-up (clocks up)
    for (int w = 0; w < 3; ++w) smem_gather<<<grid, kThreads>>>(out, iters, 256u);
    cudaEventRecord(a);
    smem_gather<<<grid, kThreads>>>(out, iters, 256u);
    cudaEventRecord(b);
    e = cudaEventSynchronize(b);
    float ms = 0.f;
    if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    if (e != cudaSuccess) return (int)e;
    const double bytes = (double)grid * kThreads * iters * 8.0 * 8.0;  // 8 LDS.64 per iteration
    *bytes_per_s = bytes / (ms * 1e-3);
    *ms_out = ms;
    return 0;
}
