// ifdk_internal.h -- internal declarations shared by the libifdk translation units.
#pragma once
#include <cuda_runtime.h>

#include <mutex>
#include <string>
#include <vector>

#include "../../include/ifdk.h"

struct ifdk_geometry {
    // Table tbl:cbct-param
    int Nu, Nv, Nx, Ny, Nz;
    double Du, Dv, Dx, Dy, Dz, D, d, theta;
    // derived
    double cu, cv, cx, cy, cz;  // (N-1)/2 centres
    double C;                   // FDK constant theta d D / (2 Du), reading c-A7
    double zmin, zmax;          // bounds of z over the volume and all views
    double rxy;                 // circumscribed radius of the volume in the rotation plane
    // ramp filter spectrum (lazy): L = FFT length, Hs[f] = C/L * DFT(h1 circular)[f]
    int log2L = 0;
    std::vector<float> Hs;      // L/2 + 1 values
    std::vector<float> tw;      // 2L floats: (cos, -sin)(2 pi t / L)
    // per-device copies of the filter tables
    struct Dev {
        float* Hs = nullptr;
        float2* tw = nullptr;
        // stream-ordered pool for ifdk_reconstruct* scratch; keeps its memory between calls
        // (release threshold = max) and is destroyed with the geometry
        cudaMemPool_t pool = nullptr;
    } dev[32];
    std::mutex mu;
};

namespace ifdk {

// error plumbing (api.cu)
ifdk_status fail(ifdk_status st, const std::string& msg);
ifdk_status cuda_fail(cudaError_t e, const char* what);
void count_launch(int n = 1);

// Scratch from the geometry's per-device pool (api.cu); freed with cudaFreeAsync.
cudaError_t scratch_alloc(ifdk_geometry* g, void** ptr, size_t bytes, cudaStream_t st);

// geometry.cpp
void projection_matrix(const ifdk_geometry* g, long s, double P[12]);
void band_rows(const ifdk_geometry* g, int k0, int nk, long s, int* lo, int* hi);
void ensure_filter_tables_host(ifdk_geometry* g);

// Conservative bound on the detector patch (columns, rows) that a tile of
// ti x tj voxel columns and kc slices can touch, over all views and positions.
void patch_bound(const ifdk_geometry* g, int ti, int tj, int kc, double* w, double* h);

// filter.cu (n_dest > 0: write each row to the destination bands instead of `out`)
constexpr int kMaxFilterDest = 16;

// Device words incremented (system-scope atomics) once a launch's stores are complete
// (peer.cu): the signals of the fused exchange.
struct PeerFlags {
    int n = 0;
    unsigned int* flag[kMaxFilterDest] = {};
    unsigned int* ticket = nullptr;  // device word, 0 between launches ("last CTA" counter)
};

ifdk_status launch_filter(ifdk_geometry* g, const float* raw, float* out, long n_views, int v0,
                          int n_rows, cudaStream_t st, int n_dest = 0,
                          const ifdk_band_dest* dests = nullptr, const PeerFlags* flags = nullptr);

// peer.cu: flags[i] += 1 after all earlier work on the stream
ifdk_status launch_signal(const PeerFlags& f, cudaStream_t st);

// Force-load (lazy module loading) every kernel that can run while a wait kernel spins.
void preload_filter_kernels();
void preload_bp_kernels();

// backproject.cu
// Fused reduce of the projection split (ifdk_backproject_reduce): the flush of each 128-view
// partial sum adds into the destination slab that holds its slice -- red.global.add (mode 0;
// local or NVLink-peer memory) or multimem.red (mode 1; multicast mappings).  base[d] holds
// slices k0[d] .. k0[d + 1] - 1 (the last to the end of the launch's slab), chunk-aligned.
constexpr int kMaxRedDest = 16;
struct RedDest {
    int mode = 0;
    int n = 0;
    int k0[kMaxRedDest] = {};
    float* base[kMaxRedDest] = {};
};
ifdk_status launch_backproject(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                               int v0, int n_rows, float* vol, int k0, int nk, int accumulate,
                               cudaStream_t st, const RedDest* red = nullptr);
// tuning hook behind ifdk_set_bp_variant (0 = automatic)
void set_bp_variant(int walk, int raster);

// forward.cu: the matched forward projector (transpose of launch_backproject) and the
// element-wise SART / SIRT steps
ifdk_status launch_forward_project(const ifdk_geometry* g, const float* vol, int k0, int nk,
                                   long s0, long n_views, float* proj, int v0, int n_rows,
                                   int accumulate, cudaStream_t st);
ifdk_status launch_sart_ratio(const float* b, const float* ax, const float* R, float* out, long n,
                              cudaStream_t st);
ifdk_status launch_sart_update(float* x, const float* c, const float* C, float lam, long n,
                               int nonneg, cudaStream_t st);
ifdk_status launch_mlem_ratio(const float* b, const float* ax, float* out, long n,
                              cudaStream_t st);
ifdk_status launch_mlem_update(float* x, const float* c, const float* C, long n, cudaStream_t st);
ifdk_status launch_fill(float* x, float value, long n, cudaStream_t st);

// baseline.cu (measured baselines, not the production path)
ifdk_status launch_backproject_alg2(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                                    float* vol, int k0, int nk, int accumulate, int hw,
                                    cudaStream_t st);
ifdk_status launch_backproject_alg4(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                                    float* vol, int accumulate, int hw, cudaStream_t st);

}  // namespace ifdk
