// probe_mc.cu -- can this box build an NVLS multicast object over ONE device and reduce into
// it with multimem.red?  (feasibility probe for the fused projection-split reduce)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

#define CK(x) do { CUresult r = (x); if (r != CUDA_SUCCESS) { const char* s; cuGetErrorString(r, &s); \
    printf("FAIL %s: %s\n", #x, s); return 1; } } while (0)

__global__ void red_kernel(float* mc, int n)
{
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        float v = 1.0f + (float)(i & 7);
        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(mc + i), "f"(v) : "memory");
    }
}

int main()
{
    CK(cuInit(0));
    CUdevice dev;
    CK(cuDeviceGet(&dev, 0));
    int mc = 0;
    CK(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    printf("MULTICAST_SUPPORTED=%d\n", mc);
    cudaSetDevice(0);
    cudaFree(0);
    if (!mc) return 0;
    const size_t n = 1 << 20;
    CUmulticastObjectProp prop = {};
    prop.numDevices = 1;
    prop.size = n * 4;
    size_t gran = 0;
    CUmemGenericAllocationHandle mch;
    CUmemAllocationHandleType types[3] = {CU_MEM_HANDLE_TYPE_NONE, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR,
                                          CU_MEM_HANDLE_TYPE_FABRIC};
    bool made = false;
    for (auto ht : types) {
        prop.handleTypes = ht;
        prop.size = n * 4;
        if (cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED) != CUDA_SUCCESS) {
            printf("handle type %d: granularity query failed\n", (int)ht);
            continue;
        }
        prop.size = (n * 4 + gran - 1) / gran * gran;
        CUresult r = cuMulticastCreate(&mch, &prop);
        const char* es; cuGetErrorString(r, &es);
        printf("handle type %d: granularity=%zu size=%zu create: %s\n", (int)ht, gran, prop.size, es);
        if (r == CUDA_SUCCESS) { made = true; break; }
    }
    if (!made) return 0;
    CK(cuMulticastAddDevice(mch, dev));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = 0;
    ap.requestedHandleTypes = (CUmemAllocationHandleType)prop.handleTypes;
    CUmemGenericAllocationHandle mh;
    CK(cuMemCreate(&mh, prop.size, &ap, 0));
    CK(cuMulticastBindMem(mch, 0, mh, 0, prop.size, 0));
    CUdeviceptr uc, mcp;
    CK(cuMemAddressReserve(&uc, prop.size, gran, 0, 0));
    CK(cuMemMap(uc, prop.size, 0, mh, 0));
    CK(cuMemAddressReserve(&mcp, prop.size, gran, 0, 0));
    CK(cuMemMap(mcp, prop.size, 0, mch, 0));
    CUmemAccessDesc ad = {};
    ad.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ad.location.id = 0;
    ad.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CK(cuMemSetAccess(uc, prop.size, &ad, 1));
    CK(cuMemSetAccess(mcp, prop.size, &ad, 1));
    cudaMemset((void*)uc, 0, n * 4);
    for (int rep = 0; rep < 3; ++rep) red_kernel<<<n / 256, 256>>>((float*)mcp, n);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<float> h(n);
    cudaMemcpy(h.data(), (void*)uc, n * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (size_t i = 0; i < n; ++i) if (h[i] != 3.f * (1.0f + (float)(i & 7))) ++bad;
    printf("multimem.red over 1-device multicast: %s (bad=%d)\n", bad ? "WRONG" : "OK", bad);
    // timing
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int rep = 0; rep < 20; ++rep) red_kernel<<<n / 256, 256>>>((float*)mcp, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("multimem.red: %.1f GB/s (4 B per element)\n", 20.0 * n * 4 / (ms * 1e6));
    return 0;
}
