// api.cu -- the extern "C" entry points of libifdk (see include/ifdk.h for the contract).
#include <cstdio>
#include <cstring>
#include <string>
#include <utility>
#include <vector>
#include <algorithm>

#include "ifdk_internal.h"

namespace ifdk {

static thread_local std::string t_last_error;
static thread_local int t_launches = 0;

ifdk_status fail(ifdk_status st, const std::string& msg)
{
    t_last_error = msg;
    return st;
}

ifdk_status cuda_fail(cudaError_t e, const char* what)
{
    t_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? IFDK_ERR_OUT_OF_MEMORY : IFDK_ERR_CUDA;
}

void count_launch(int n) { t_launches += n; }

static ifdk_status need_device()
{
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        cudaGetLastError();
        return fail(IFDK_ERR_CUDA, "no CUDA device (libifdk has no CPU fallback)");
    }
    return IFDK_OK;
}

static ifdk_status check_band(const ifdk_geometry* g, long n_views, int v0, int n_rows)
{
    if (n_views < 0) return fail(IFDK_ERR_SHAPE, "n_views < 0");
    if (n_rows < 1 || v0 < 0 || (long)v0 + n_rows > g->Nv)
        return fail(IFDK_ERR_SHAPE, "row band v0..v0+n_rows-1 outside [0, Nv)");
    return IFDK_OK;
}

cudaError_t scratch_alloc(ifdk_geometry* g, void** ptr, size_t bytes, cudaStream_t st)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev >= 32) return cudaErrorInvalidDevice;
    cudaMemPool_t pool;
    {
        std::lock_guard<std::mutex> lk(g->mu);
        auto& D = g->dev[dev];
        if (!D.pool) {
            // The default pool returns its memory to the driver at every synchronisation, so a
            // 40 GiB scratch set would be remapped on every call; this one keeps it.
            cudaMemPoolProps props{};
            props.allocType = cudaMemAllocationTypePinned;
            props.handleTypes = cudaMemHandleTypeNone;
            props.location.type = cudaMemLocationTypeDevice;
            props.location.id = dev;
            if ((e = cudaMemPoolCreate(&D.pool, &props)) != cudaSuccess) return e;
            uint64_t keep = ~0ull;
            cudaMemPoolSetAttribute(D.pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        pool = D.pool;
    }
    return cudaMallocFromPoolAsync(ptr, bytes, pool, st);
}

}  // namespace ifdk

using namespace ifdk;

// Views per batch of ifdk_reconstruct / ifdk_reconstruct_host (a multiple of the BP kernel's
// two-level summation batch, so batching does not change a single bit of the result).
static const long kViewBatch = 256;

extern "C" ifdk_status ifdk_filter(const ifdk_geometry* g, const float* raw_dev,
                                   float* filtered_dev, long n_views, int v0, int n_rows,
                                   void* stream)
{
    t_launches = 0;
    if (!g || !raw_dev || !filtered_dev) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    ifdk_status s = check_band(g, n_views, v0, n_rows);
    if (s != IFDK_OK) return s;
    if ((s = need_device()) != IFDK_OK) return s;
    return launch_filter(const_cast<ifdk_geometry*>(g), raw_dev, filtered_dev, n_views, v0,
                         n_rows, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_filter_scatter(const ifdk_geometry* g, const float* raw_dev,
                                           long n_views, int v0, int n_rows, int n_dest,
                                           const ifdk_band_dest* dests, int n_flags,
                                           unsigned int* const* flags, unsigned int* ticket_dev,
                                           void* stream)
{
    t_launches = 0;
    if (!g || !raw_dev || !dests) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_dest < 1 || n_dest > kMaxFilterDest)
        return fail(IFDK_ERR_INVALID_ARGUMENT, "n_dest must be 1..16");
    if (n_flags < 0 || n_flags > kMaxFilterDest || (n_flags > 0 && (!flags || !ticket_dev)))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "need 0 <= n_flags <= 16, flags and a ticket");
    PeerFlags pf{};
    pf.n = n_flags;
    pf.ticket = ticket_dev;
    for (int f = 0; f < n_flags; ++f) {
        if (!flags[f]) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL flag");
        pf.flag[f] = flags[f];
    }
    for (int d = 0; d < n_dest; ++d)
        if (!dests[d].base || dests[d].v_lo < 0 || dests[d].v_hi >= g->Nv ||
            dests[d].v_hi < dests[d].v_lo)
            return fail(IFDK_ERR_INVALID_ARGUMENT, "destination band NULL, empty or outside [0, Nv)");
    ifdk_status s = check_band(g, n_views, v0, n_rows);
    if (s != IFDK_OK) return s;
    if ((s = need_device()) != IFDK_OK) return s;
    return launch_filter(const_cast<ifdk_geometry*>(g), raw_dev, nullptr, n_views, v0, n_rows,
                         (cudaStream_t)stream, n_dest, dests, n_flags > 0 ? &pf : nullptr);
}

extern "C" ifdk_status ifdk_backproject(const ifdk_geometry* g, const float* filtered_dev,
                                        long s0, long n_views, int v0, int n_rows, float* vol_dev,
                                        int k0, int nk, int accumulate, void* stream)
{
    t_launches = 0;
    if (!g || !vol_dev || (!filtered_dev && n_views > 0))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (accumulate != 0 && accumulate != 1)
        return fail(IFDK_ERR_INVALID_ARGUMENT, "accumulate must be 0 or 1");
    ifdk_status s = check_band(g, n_views, v0, n_rows);
    if (s != IFDK_OK) return s;
    if (k0 < 0 || nk < 1 || (long)k0 + nk > g->Nz)
        return fail(IFDK_ERR_SHAPE, "slab k0..k0+nk-1 outside [0, Nz)");
    for (long t = 0; t < n_views; ++t) {
        int lo, hi;
        band_rows(g, k0, nk, s0 + t, &lo, &hi);
        if (lo <= hi && (lo < v0 || hi > v0 + n_rows - 1)) {
            char buf[200];
            snprintf(buf, sizeof buf,
                     "view %ld needs detector rows %d..%d but the band holds %d..%d", s0 + t, lo,
                     hi, v0, v0 + n_rows - 1);
            return fail(IFDK_ERR_SHAPE, buf);
        }
    }
    if ((s = need_device()) != IFDK_OK) return s;
    return launch_backproject(g, filtered_dev, s0, n_views, v0, n_rows, vol_dev, k0, nk,
                              accumulate, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_backproject_reduce(const ifdk_geometry* g, const float* filtered_dev,
                                               long s0, long n_views, int v0, int n_rows,
                                               int k0, int nk, int n_dest, float* const* dest,
                                               const int* dest_k0, int mode, void* stream)
{
    t_launches = 0;
    if (!g || !dest || !dest_k0 || (!filtered_dev && n_views > 0))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (mode != 0 && mode != 1) return fail(IFDK_ERR_INVALID_ARGUMENT, "mode must be 0 or 1");
    if (n_dest < 1 || n_dest > kMaxRedDest)
        return fail(IFDK_ERR_INVALID_ARGUMENT, "n_dest must be 1..16");
    ifdk_status s = check_band(g, n_views, v0, n_rows);
    if (s != IFDK_OK) return s;
    if (k0 < 0 || nk < 1 || (long)k0 + nk > g->Nz)
        return fail(IFDK_ERR_SHAPE, "slab k0..k0+nk-1 outside [0, Nz)");
    // destination slabs: strictly increasing starts, the first at or below k0 (each slab runs
    // to the next one's start, the last through k0+nk-1)
    RedDest red;
    red.mode = mode;
    red.n = n_dest;
    for (int d = 0; d < n_dest; ++d) {
        if (!dest[d]) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL destination slab");
        if (d > 0 && dest_k0[d] <= dest_k0[d - 1])
            return fail(IFDK_ERR_SHAPE, "destination slab starts must increase");
        red.k0[d] = dest_k0[d];
        red.base[d] = dest[d];
    }
    if (dest_k0[0] > k0) return fail(IFDK_ERR_SHAPE, "destination slabs do not cover k0");
    for (long t = 0; t < n_views; ++t) {
        int lo, hi;
        band_rows(g, k0, nk, s0 + t, &lo, &hi);
        if (lo <= hi && (lo < v0 || hi > v0 + n_rows - 1))
            return fail(IFDK_ERR_SHAPE, "the row band does not cover the slab's rows");
    }
    if ((s = need_device()) != IFDK_OK) return s;
    return launch_backproject(g, filtered_dev, s0, n_views, v0, n_rows, nullptr, k0, nk, 1,
                              (cudaStream_t)stream, &red);
}

extern "C" ifdk_status ifdk_forward_project(const ifdk_geometry* g, const float* vol_dev, int k0,
                                            int nk, long s0, long n_views, float* proj_dev,
                                            int v0, int n_rows, int accumulate, void* stream)
{
    t_launches = 0;
    if (!g || !vol_dev || (!proj_dev && n_views > 0))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (accumulate != 0 && accumulate != 1)
        return fail(IFDK_ERR_INVALID_ARGUMENT, "accumulate must be 0 or 1");
    ifdk_status s = check_band(g, n_views, v0, n_rows);
    if (s != IFDK_OK) return s;
    if (k0 < 0 || nk < 1 || (long)k0 + nk > g->Nz)
        return fail(IFDK_ERR_SHAPE, "slab k0..k0+nk-1 outside [0, Nz)");
    for (long t = 0; t < n_views; ++t) {
        int lo, hi;
        band_rows(g, k0, nk, s0 + t, &lo, &hi);
        if (lo <= hi && (lo < v0 || hi > v0 + n_rows - 1)) {
            char buf[200];
            snprintf(buf, sizeof buf,
                     "view %ld reaches detector rows %d..%d but the band holds %d..%d", s0 + t,
                     lo, hi, v0, v0 + n_rows - 1);
            return fail(IFDK_ERR_SHAPE, buf);
        }
    }
    if ((s = need_device()) != IFDK_OK) return s;
    return launch_forward_project(g, vol_dev, k0, nk, s0, n_views, proj_dev, v0, n_rows,
                                  accumulate, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_sart_ratio(const float* b_dev, const float* ax_dev, const float* R_dev,
                                       float* out_dev, long n, void* stream)
{
    t_launches = 0;
    if (n < 0) return fail(IFDK_ERR_SHAPE, "n < 0");
    if (n > 0 && (!b_dev || !ax_dev || !R_dev || !out_dev))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    return launch_sart_ratio(b_dev, ax_dev, R_dev, out_dev, n, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_sart_update(float* x_dev, const float* c_dev, const float* C_dev,
                                        float lambda, long n, int nonneg, void* stream)
{
    t_launches = 0;
    if (n < 0) return fail(IFDK_ERR_SHAPE, "n < 0");
    if (n > 0 && (!x_dev || !c_dev || !C_dev))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (!(lambda > 0.f && lambda < 2.f))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "relaxation lambda must lie in (0, 2)");
    if (nonneg != 0 && nonneg != 1) return fail(IFDK_ERR_INVALID_ARGUMENT, "nonneg must be 0 or 1");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    return launch_sart_update(x_dev, c_dev, C_dev, lambda, n, nonneg, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_mlem_ratio(const float* b_dev, const float* ax_dev, float* out_dev,
                                       long n, void* stream)
{
    t_launches = 0;
    if (n < 0) return fail(IFDK_ERR_SHAPE, "n < 0");
    if (n > 0 && (!b_dev || !ax_dev || !out_dev))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    return launch_mlem_ratio(b_dev, ax_dev, out_dev, n, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_mlem_update(float* x_dev, const float* c_dev, const float* C_dev,
                                        long n, void* stream)
{
    t_launches = 0;
    if (n < 0) return fail(IFDK_ERR_SHAPE, "n < 0");
    if (n > 0 && (!x_dev || !c_dev || !C_dev))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    return launch_mlem_update(x_dev, c_dev, C_dev, n, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_fill(float* x_dev, float value, long n, void* stream)
{
    t_launches = 0;
    if (n < 0) return fail(IFDK_ERR_SHAPE, "n < 0");
    if (n > 0 && !x_dev) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    return launch_fill(x_dev, value, n, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_backproject_alg2(const ifdk_geometry* g, const float* filtered_dev,
                                             long s0, long n_views, float* vol_dev, int k0, int nk,
                                             int accumulate, int texture, void* stream)
{
    t_launches = 0;
    if (!g || !vol_dev || (!filtered_dev && n_views > 0))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if ((accumulate != 0 && accumulate != 1) || (texture != 0 && texture != 1))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "accumulate and texture must be 0 or 1");
    if (n_views < 0) return fail(IFDK_ERR_SHAPE, "n_views < 0");
    if (k0 < 0 || nk < 1 || (long)k0 + nk > g->Nz)
        return fail(IFDK_ERR_SHAPE, "slab k0..k0+nk-1 outside [0, Nz)");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    if (n_views == 0) return launch_backproject(g, filtered_dev, s0, 0, 0, g->Nv, vol_dev, k0, nk,
                                                accumulate, (cudaStream_t)stream);
    return launch_backproject_alg2(g, filtered_dev, s0, n_views, vol_dev, k0, nk, accumulate,
                                   texture, (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_backproject_alg4(const ifdk_geometry* g, const float* filtered_dev,
                                             long s0, long n_views, float* vol_dev, int accumulate,
                                             int texture, void* stream)
{
    t_launches = 0;
    if (!g || !vol_dev || (!filtered_dev && n_views > 0))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if ((accumulate != 0 && accumulate != 1) || (texture != 0 && texture != 1))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "accumulate and texture must be 0 or 1");
    if (n_views < 0) return fail(IFDK_ERR_SHAPE, "n_views < 0");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    if (n_views == 0) return launch_backproject(g, filtered_dev, s0, 0, 0, g->Nv, vol_dev, 0,
                                                g->Nz, accumulate, (cudaStream_t)stream);
    return launch_backproject_alg4(g, filtered_dev, s0, n_views, vol_dev, accumulate, texture,
                                   (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_reconstruct(const ifdk_geometry* g, const float* raw_dev,
                                        long n_views, float* vol_dev, void* stream)
{
    t_launches = 0;
    if (!g || !raw_dev || !vol_dev) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_views < 0) return fail(IFDK_ERR_SHAPE, "n_views < 0");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t view_elems = (size_t)g->Nv * g->Nu;
    const long batch = n_views < kViewBatch ? (n_views > 0 ? n_views : 1) : kViewBatch;
    ifdk_geometry* gm = const_cast<ifdk_geometry*>(g);
    // Batch b + 1 is filtered on a side stream into the other of two scratch buffers while
    // batch b is back-projected on `st` (the paper's filter / back-projection overlap, P:790-833,
    // on one GPU): the filter kernels fill the SM slots the back-projection leaves free.
    float* Q[2] = {nullptr, nullptr};
    const long nbatch = (n_views + batch - 1) / batch;
    cudaError_t e = scratch_alloc(gm, (void**)&Q[0], sizeof(float) * view_elems * batch, st);
    if (e == cudaSuccess && nbatch > 1)
        e = scratch_alloc(gm, (void**)&Q[1], sizeof(float) * view_elems * batch, st);
    if (e != cudaSuccess) {
        if (Q[0]) cudaFreeAsync(Q[0], st);
        return fail(IFDK_ERR_OUT_OF_MEMORY, "cudaMallocAsync(filtered scratch)");
    }
    if (n_views == 0) s = launch_backproject(g, Q[0], 0, 0, 0, g->Nv, vol_dev, 0, g->Nz, 0, st);
    if (s == IFDK_OK && nbatch == 1) {  // nothing to overlap: no side stream (latency)
        s = launch_filter(gm, raw_dev, Q[0], n_views, 0, g->Nv, st);
        if (s == IFDK_OK) s = launch_backproject(g, Q[0], 0, n_views, 0, g->Nv, vol_dev, 0, g->Nz, 0, st);
        cudaFreeAsync(Q[0], st);
        return s;
    }
    cudaStream_t fs = nullptr;
    cudaEvent_t ev[5] = {};  // start, filtered[2], consumed[2]
    if (s == IFDK_OK && n_views > 0) {
        if ((e = cudaStreamCreateWithFlags(&fs, cudaStreamNonBlocking)) != cudaSuccess)
            s = cuda_fail(e, "cudaStreamCreate");
        for (int q = 0; q < 5 && s == IFDK_OK; ++q)
            if ((e = cudaEventCreateWithFlags(&ev[q], cudaEventDisableTiming)) != cudaSuccess)
                s = cuda_fail(e, "cudaEventCreate");
    }
    if (s == IFDK_OK && n_views > 0) {
        cudaEventRecord(ev[0], st);  // the caller's earlier work and the scratch allocations
        cudaStreamWaitEvent(fs, ev[0], 0);
        auto filter = [&](long b) {
            const int q = (int)(b & 1);
            const long b0 = b * batch;
            const long nb = (n_views - b0) < batch ? (n_views - b0) : batch;
            if (b >= 2) cudaStreamWaitEvent(fs, ev[3 + q], 0);  // BP of batch b - 2 read Q[q]
            ifdk_status r = launch_filter(gm, raw_dev + b0 * view_elems, Q[q], nb, 0, g->Nv, fs);
            cudaEventRecord(ev[1 + q], fs);
            return r;
        };
        s = filter(0);
        for (long b = 0; b < nbatch && s == IFDK_OK; ++b) {
            const int q = (int)(b & 1);
            const long b0 = b * batch;
            const long nb = (n_views - b0) < batch ? (n_views - b0) : batch;
            if (b + 1 < nbatch && (s = filter(b + 1)) != IFDK_OK) break;
            cudaStreamWaitEvent(st, ev[1 + q], 0);
            s = launch_backproject(g, Q[q], b0, nb, 0, g->Nv, vol_dev, 0, g->Nz, b0 > 0 ? 1 : 0, st);
            cudaEventRecord(ev[3 + q], st);
        }
        // every filter launch joined before the scratch returns to the pool on `st`
        cudaEventRecord(ev[0], fs);
        cudaStreamWaitEvent(st, ev[0], 0);
    }
    for (int q = 0; q < 5; ++q)
        if (ev[q]) cudaEventDestroy(ev[q]);
    if (fs) cudaStreamDestroy(fs);
    cudaFreeAsync(Q[0], st);
    if (Q[1]) cudaFreeAsync(Q[1], st);
    return s;
}

// End-to-end reconstruction of the slab k0..k0+nk-1 from host views, copying only detector
// rows v0..v0+n_rows-1 of each view (the full detector for ifdk_reconstruct_host; the slab's
// row band for ifdk_reconstruct_slab_host).
static ifdk_status reconstruct_host_impl(const ifdk_geometry* g, const float* raw_host,
                                         long n_views, int k0s, int nks, int v0, int n_rows,
                                         float* vol_host, cudaStream_t st)
{
    ifdk_status s = IFDK_OK;
    const size_t view_elems = (size_t)n_rows * g->Nu;          // staged elements per view
    const size_t host_view_elems = (size_t)g->Nv * g->Nu;      // elements per host view
    const size_t plane = (size_t)g->Ny * g->Nx;
    const size_t vol_elems = (size_t)nks * plane;
    const long batch = n_views < kViewBatch ? (n_views > 0 ? n_views : 1) : kViewBatch;
    // Two staging buffers: batch b+1 is copied and filtered (in place) on `cp` while batch b
    // is back-projected on `st`.
    cudaStream_t cp = nullptr;
    cudaEvent_t copied[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    float* buf[2] = {nullptr, nullptr};
    float* vol = nullptr;
    cudaError_t e = cudaStreamCreateWithFlags(&cp, cudaStreamNonBlocking);
    if (e != cudaSuccess) return cuda_fail(e, "cudaStreamCreate");
    for (int q = 0; q < 2; ++q) {
        cudaEventCreateWithFlags(&copied[q], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&consumed[q], cudaEventDisableTiming);
    }
    cudaEvent_t slab_done = nullptr;
    cudaEventCreateWithFlags(&slab_done, cudaEventDisableTiming);
    ifdk_geometry* gm = const_cast<ifdk_geometry*>(g);
    e = scratch_alloc(gm, (void**)&vol, sizeof(float) * vol_elems, st);
    if (e == cudaSuccess) e = scratch_alloc(gm, (void**)&buf[0], sizeof(float) * view_elems * batch, st);
    if (e == cudaSuccess) e = scratch_alloc(gm, (void**)&buf[1], sizeof(float) * view_elems * batch, st);
    if (e != cudaSuccess) s = fail(IFDK_ERR_OUT_OF_MEMORY, "cudaMallocAsync(reconstruct_host)");
    if (s == IFDK_OK) {
        cudaEvent_t ready;
        cudaEventCreateWithFlags(&ready, cudaEventDisableTiming);
        cudaEventRecord(ready, st);  // allocations visible to the copy stream
        cudaStreamWaitEvent(cp, ready, 0);
        cudaEventDestroy(ready);
        if (n_views == 0) s = launch_backproject(g, buf[0], 0, 0, v0, n_rows, vol, k0s, nks, 0, st);
        // Batches of `batch` views, the first full batch split in two halves (views 0..127,
        // 128..255, one per staging buffer) so that the one H2D nothing overlaps is half a
        // batch; the last batch stays full, so its back-projection still covers the volume's
        // D2H (a half-size last batch measured e2e 9.18 s vs 9.10 s on config 4).  Every
        // boundary is a multiple of 128 views, the BP's summation batch: the result is
        // bitwise that of one launch.
        std::vector<std::pair<long, long>> bat;  // (first view, views)
        for (long b0 = 0; b0 < n_views;) {
            long nb = (b0 < kViewBatch && batch == kViewBatch) ? kViewBatch / 2 : batch;
            if (nb > n_views - b0) nb = n_views - b0;
            bat.emplace_back(b0, nb);
            b0 += nb;
        }
        const long nbatches = (long)bat.size();
        auto enqueue_copy = [&](long b) {
            const int q = (int)(b & 1);
            const long b0 = bat[b].first;
            const long nb = bat[b].second;
            if (b >= 2) cudaStreamWaitEvent(cp, consumed[q], 0);
            // rows v0..v0+n_rows-1 of views b0..b0+nb-1: one 2-D copy (a contiguous run per view)
            const cudaError_t ce =
                cudaMemcpy2DAsync(buf[q], sizeof(float) * view_elems,
                                  raw_host + b0 * host_view_elems + (size_t)v0 * g->Nu,
                                  sizeof(float) * host_view_elems, sizeof(float) * view_elems, nb,
                                  cudaMemcpyHostToDevice, cp);
            if (ce != cudaSuccess && s == IFDK_OK) s = cuda_fail(ce, "cudaMemcpy2DAsync(views H2D)");
            // filtered in place on the copy stream: overlaps the back-projection of batch b - 1
            const ifdk_status fst = launch_filter(const_cast<ifdk_geometry*>(g), buf[q], buf[q], nb,
                                                  v0, n_rows, cp);
            if (fst != IFDK_OK && s == IFDK_OK) s = fst;
            cudaEventRecord(copied[q], cp);
        };
        if (nbatches > 0) enqueue_copy(0);
        if (nbatches > 1) enqueue_copy(1);
        for (long b = 0; b < nbatches && s == IFDK_OK; ++b) {
            const int q = (int)(b & 1);
            const long b0 = bat[b].first;
            const long nb = bat[b].second;
            cudaStreamWaitEvent(st, copied[q], 0);  // copied and filtered
            if (b + 1 < nbatches) {
                s = launch_backproject(g, buf[q], b0, nb, v0, n_rows, vol, k0s, nks,
                                       b0 > 0 ? 1 : 0, st);
            } else {
                // Last batch: back-project slab by slab and stream each finished slab to the
                // host on `cp` while the next slab computes (slab starts on multiples of 64
                // slices, so the result is bitwise that of one launch).
                // 256-slice slabs, the last 256 slices in 64-slice ones: the final D2H, which
                // nothing overlaps, is then a quarter of a slab.
                std::vector<std::pair<int, int>> slabs;
                const int kend = k0s + nks;
                if (nks > 512) {
                    int k0 = k0s;
                    for (; k0 + 512 <= kend; k0 += 256) slabs.emplace_back(k0, 256);
                    for (; k0 < kend; k0 += 64) slabs.emplace_back(k0, std::min(64, kend - k0));
                } else {
                    slabs.emplace_back(k0s, nks);
                }
                for (size_t si = 0; si < slabs.size() && s == IFDK_OK; ++si) {
                    const int k0 = slabs[si].first, nk = slabs[si].second;
                    float* vs = vol + (size_t)(k0 - k0s) * plane;
                    s = launch_backproject(g, buf[q], b0, nb, v0, n_rows, vs, k0, nk,
                                           b0 > 0 ? 1 : 0, st);
                    cudaEventRecord(slab_done, st);
                    cudaStreamWaitEvent(cp, slab_done, 0);
                    e = cudaMemcpyAsync(vol_host + (size_t)(k0 - k0s) * plane, vs,
                                        sizeof(float) * (size_t)nk * plane,
                                        cudaMemcpyDeviceToHost, cp);
                    if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync(volume D2H)");
                }
            }
            cudaEventRecord(consumed[q], st);
            if (b + 2 < nbatches) enqueue_copy(b + 2);
        }
        if (s == IFDK_OK && nbatches == 0) {
            e = cudaMemcpyAsync(vol_host, vol, sizeof(float) * vol_elems, cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync(volume D2H)");
        }
        // the copy stream must finish before the scratch is released on `st`
        cudaEventRecord(slab_done, cp);
        cudaStreamWaitEvent(st, slab_done, 0);
    }
    if (buf[0]) cudaFreeAsync(buf[0], st);
    if (buf[1]) cudaFreeAsync(buf[1], st);
    if (vol) cudaFreeAsync(vol, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess && s == IFDK_OK) s = cuda_fail(e, "reconstruct_host");
    cudaStreamSynchronize(cp);
    for (int q = 0; q < 2; ++q) {
        cudaEventDestroy(copied[q]);
        cudaEventDestroy(consumed[q]);
    }
    cudaEventDestroy(slab_done);
    cudaStreamDestroy(cp);
    return s;
}

extern "C" ifdk_status ifdk_reconstruct_host(const ifdk_geometry* g, const float* raw_host,
                                             long n_views, float* vol_host, void* stream)
{
    t_launches = 0;
    if (!g || !raw_host || !vol_host) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_views < 0) return fail(IFDK_ERR_SHAPE, "n_views < 0");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    return reconstruct_host_impl(g, raw_host, n_views, 0, g->Nz, 0, g->Nv, vol_host,
                                 (cudaStream_t)stream);
}

extern "C" ifdk_status ifdk_reconstruct_slab_host(const ifdk_geometry* g, const float* raw_host,
                                                  long n_views, int k0, int nk, float* vol_host,
                                                  void* stream)
{
    t_launches = 0;
    if (!g || !raw_host || !vol_host) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (n_views < 0) return fail(IFDK_ERR_SHAPE, "n_views < 0");
    if (k0 < 0 || nk < 1 || (long)k0 + nk > g->Nz)
        return fail(IFDK_ERR_SHAPE, "slab k0..k0+nk-1 outside [0, Nz)");
    ifdk_status s = need_device();
    if (s != IFDK_OK) return s;
    // the union of the rows the slab's taps can touch over all views
    int lo = g->Nv, hi = -1;
    for (long t = 0; t < n_views; ++t) {
        int a, b;
        band_rows(g, k0, nk, t, &a, &b);
        if (a <= b) {
            lo = std::min(lo, a);
            hi = std::max(hi, b);
        }
    }
    if (hi < lo) {  // no view reaches the slab: it is zero
        lo = 0;
        hi = 0;
    }
    return reconstruct_host_impl(g, raw_host, n_views, k0, nk, lo, hi - lo + 1, vol_host,
                                 (cudaStream_t)stream);
}

extern "C" void ifdk_geometry_destroy(ifdk_geometry* g)
{
    if (!g) return;
    for (auto& d : g->dev) {
        if (d.Hs) cudaFree(d.Hs);
        if (d.tw) cudaFree(d.tw);
        if (d.pool) cudaMemPoolDestroy(d.pool);  // deferred until outstanding frees complete
    }
    delete g;
}

extern "C" int ifdk_last_launch_count(void) { return t_launches; }

extern "C" const char* ifdk_last_error(void) { return t_last_error.c_str(); }

extern "C" ifdk_status ifdk_set_bp_variant(int walk, int raster)
{
    if (walk < 0 || raster < 0) return fail(IFDK_ERR_INVALID_ARGUMENT, "walk and raster must be >= 0");
    set_bp_variant(walk, raster);
    return IFDK_OK;
}
