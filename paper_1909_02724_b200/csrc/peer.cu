// peer.cu -- the plumbing of the fused row-band exchange of the k-slab split:
// peer-mapped device memory (CUDA IPC: one process per GPU, mapped over NVLink by the driver)
// and device-side signals that order the peers' stores into that memory.
//
// Ordering argument (CUDA C++ Programming Guide, "Memory Fence Functions"):
//  * A producer kernel stores rows into a peer's buffer, then every thread executes
//    __threadfence_system() ("all writes to all memory made by the calling thread before the
//    call are observed by all threads in the device, host threads, and all threads in peer
//    devices as occurring before all writes to all memory made by the calling thread after
//    the call"), a __syncthreads(), and thread 0 takes a ticket (atomicAdd on a device word);
//    the CTA that takes the last ticket fences again and increments each destination's flag
//    with a system-scope atomic -- the guide's "last block" reduction pattern at system scope.
//  * The consumer spins on the flag with ld.acquire.sys until it reaches the target, fences,
//    and exits; the back-projection is stream-ordered after it on the consumer's GPU.
//  * Buffer reuse (write-after-read): the consumer signals "released" with a kernel
//    stream-ordered after the back-projection that read the buffer; a kernel completes only
//    after all its loads have returned, so no later store can be observed by them.
#include <cstring>
#include <mutex>

#include "ifdk_internal.h"

namespace ifdk {
namespace {

__global__ void signal_kernel(PeerFlags f)
{
    const int i = threadIdx.x;
    __threadfence_system();
    if (i < f.n) atomicAdd_system(f.flag[i], 1u);
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p)
{
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Thread w waits for word w; a peer that never signals (a dead rank) traps after the timeout
// instead of hanging the GPU.
__global__ void wait_kernel(const unsigned* flags, int n, unsigned target,
                            unsigned long long timeout_ns)
{
    const int w = threadIdx.x;
    if (w < n) {
        const unsigned long long t0 = globaltimer();
        unsigned spins = 0;
        while ((int)(ld_acquire_sys(flags + w) - target) < 0) {
            if (++spins > 64) __nanosleep(200);
            if ((spins & 1023) == 0 && globaltimer() - t0 > timeout_ns) __trap();
        }
    }
    __threadfence_system();
    __syncthreads();
}

}  // namespace

ifdk_status launch_signal(const PeerFlags& f, cudaStream_t st)
{
    if (f.n == 0) return IFDK_OK;
    signal_kernel<<<1, 32, 0, st>>>(f);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "signal_kernel launch");
    count_launch();
    return IFDK_OK;
}

}  // namespace ifdk

using namespace ifdk;

static const unsigned long long kWaitTimeoutNs = 300ull * 1000 * 1000 * 1000;

extern "C" ifdk_status ifdk_peer_alloc(size_t bytes, void** dev_ptr, unsigned char handle[64])
{
    if (!dev_ptr || !handle || bytes == 0) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL or empty");
    *dev_ptr = nullptr;
    cudaError_t e = cudaMalloc(dev_ptr, bytes);  // a whole allocation: its IPC handle maps offset 0
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(peer buffer)");
    cudaIpcMemHandle_t h;
    e = cudaIpcGetMemHandle(&h, *dev_ptr);
    if (e != cudaSuccess) {
        cudaFree(*dev_ptr);
        *dev_ptr = nullptr;
        return cuda_fail(e, "cudaIpcGetMemHandle");
    }
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    std::memcpy(handle, &h, 64);
    return IFDK_OK;
}

extern "C" ifdk_status ifdk_peer_open(const unsigned char handle[64], void** dev_ptr)
{
    if (!dev_ptr || !handle) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    cudaError_t e = cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcOpenMemHandle");
    return IFDK_OK;
}

extern "C" ifdk_status ifdk_peer_close(void* dev_ptr)
{
    if (!dev_ptr) return IFDK_OK;
    cudaError_t e = cudaIpcCloseMemHandle(dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaIpcCloseMemHandle");
    return IFDK_OK;
}

extern "C" ifdk_status ifdk_peer_free(void* dev_ptr)
{
    if (!dev_ptr) return IFDK_OK;
    cudaError_t e = cudaFree(dev_ptr);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFree(peer buffer)");
    return IFDK_OK;
}

extern "C" ifdk_status ifdk_signal(int n_flags, unsigned int* const* flags, void* stream)
{
    if (n_flags < 0 || n_flags > kMaxFilterDest || (n_flags > 0 && !flags))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "need 0 <= n_flags <= 16 and flags");
    PeerFlags f{};
    f.n = n_flags;
    for (int i = 0; i < n_flags; ++i) {
        if (!flags[i]) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL flag");
        f.flag[i] = flags[i];
    }
    return launch_signal(f, (cudaStream_t)stream);
}

// Under lazy module loading (the CUDA 12 default) a kernel is loaded at its first launch, and
// loading waits for the context to be idle: a wait kernel spinning for a signal that a
// not-yet-loaded kernel (a peer's scatter, this GPU's own next filter) will send would never
// finish.  So every kernel of the exchange pipeline is loaded before the first wait kernel
// is launched on a device.
static void preload_once()
{
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) {
        cudaGetLastError();
        return;
    }
    std::lock_guard<std::mutex> lk(mu);
    if (done[dev]) return;
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(signal_kernel)) != cudaSuccess ||
        cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(wait_kernel)) != cudaSuccess)
        cudaGetLastError();
    preload_filter_kernels();
    preload_bp_kernels();
    done[dev] = true;
}

extern "C" ifdk_status ifdk_wait(const unsigned int* flags_dev, int n, unsigned int target,
                                 unsigned int timeout_ms, void* stream)
{
    if (!flags_dev || n < 1 || n > 1024)
        return fail(IFDK_ERR_INVALID_ARGUMENT, "need flags and 1 <= n <= 1024");
    preload_once();
    const unsigned long long ns =
        timeout_ms ? 1000000ull * timeout_ms : kWaitTimeoutNs;
    wait_kernel<<<1, ((n + 31) / 32) * 32, 0, (cudaStream_t)stream>>>(flags_dev, n, target, ns);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "wait_kernel launch");
    count_launch();
    return IFDK_OK;
}
