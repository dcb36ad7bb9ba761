// baseline.cu -- the paper's straightforward kernel on B200, kept as a measured baseline
// (SURVEY 8(f) row 3): Alg. alg:bp per voxel, literally, in fp32 -- [x, y, z] =
// P_s [i, j, k, 1], f = 1/z, (u, v) = (x f, y f), acc += f^2 interp2(Q_s, u, v) -- with the
// bilinear sample taken either by the texture unit (cudaFilterModeLinear: the weights are
// 1.8 fixed point, 8 fractional bits) or in software from global memory (Alg. alg:subpixel,
// P:431-447, fp32 weights).  One thread per voxel, i fastest (coalesced volume stores), all
// views of the launch accumulated in a register.  These are what the paper's GPU path
// (texture-based RTK kernel) looks like recompiled for sm_100a; the
// production kernel (backproject.cu) is measured against them, and their error against the
// fp64 oracle shows why it computes coordinates in fp64 per column and weights in fp32
// (DESIGN.md "Numerics").  bp_alg4_kernel is the paper's own proposed Alg. alg:bp-v1 on the
// same footing, to re-measure its claimed speed-up over Alg. alg:bp on B200.
#include <cstdint>
#include <vector>

#include "ifdk_internal.h"

namespace ifdk {
namespace {

constexpr int kMaxViews = 256;

struct P12Table {
    float P[kMaxViews][12];  // fp32 P_s, row-major 3x4 (the paper's single precision)
};

struct BaseParams {
    const float* Q;  // [n_views][Nv][Nu] (software path)
    float* vol;      // slab [nk][Ny][Nx]
    int n_views, Nu, Nv, Nx, Ny, k0, nk, accumulate;
    cudaTextureObject_t tex;  // layered texture of the n_views projections (hardware path)
};

__device__ __forceinline__ float tap(const float* Qv, int Nu, int Nv, int a, int b)
{
    return (a >= 0 && a < Nu && b >= 0 && b < Nv) ? __ldg(Qv + (long)b * Nu + a) : 0.f;  // c-A9
}

template <bool HW>
__global__ void __launch_bounds__(256) bp_alg2_kernel(const __grid_constant__ BaseParams p,
                                                      const __grid_constant__ P12Table pt)
{
    const long nvox = (long)p.nk * p.Ny * p.Nx;
    const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= nvox) return;
    const int i = (int)(idx % p.Nx);
    const int j = (int)((idx / p.Nx) % p.Ny);
    const int k = p.k0 + (int)(idx / ((long)p.Nx * p.Ny));
    const float fi = (float)i, fj = (float)j, fk = (float)k;
    float acc = 0.f;
    for (int t = 0; t < p.n_views; ++t) {
        const float* P = pt.P[t];  // constant bank, uniform address
        const float x = fmaf(P[0], fi, fmaf(P[1], fj, fmaf(P[2], fk, P[3])));
        const float y = fmaf(P[4], fi, fmaf(P[5], fj, fmaf(P[6], fk, P[7])));
        const float z = fmaf(P[8], fi, fmaf(P[9], fj, fmaf(P[10], fk, P[11])));
        const float f = 1.f / z;
        const float u = x * f, v = y * f;
        float val;
        if (HW) {
            // texel centres sit at +0.5; border address mode returns 0 per tap (c-A9)
            val = tex2DLayered<float>(p.tex, u + 0.5f, v + 0.5f, t);
        } else {
            const float* Qv = p.Q + (long)t * p.Nv * p.Nu;
            const float fu = floorf(u), fv = floorf(v);
            const int nu = (int)fu, nv = (int)fv;
            const float du = u - fu, dv = v - fv;
            const float t1 = fmaf(du, tap(Qv, p.Nu, p.Nv, nu + 1, nv) - tap(Qv, p.Nu, p.Nv, nu, nv),
                                  tap(Qv, p.Nu, p.Nv, nu, nv));
            const float t2 = fmaf(du, tap(Qv, p.Nu, p.Nv, nu + 1, nv + 1) -
                                          tap(Qv, p.Nu, p.Nv, nu, nv + 1),
                                  tap(Qv, p.Nu, p.Nv, nu, nv + 1));
            val = fmaf(dv, t2 - t1, t1);
        }
        acc = fmaf(f * f, val, acc);  // W_dis = f^2, Alg. alg:bp line 8-10
    }
    float* o = p.vol + idx;
    *o = p.accumulate ? *o + acc : acc;
}

// The paper's proposed Alg. alg:bp-v1 as printed, in fp32, on the same footing as
// bp_alg2_kernel (row-major Q, i-major volume; the transposes of lines 3 and 22 are layout
// choices orthogonal to the operation count): per (column, view) the two inner products x, z
// (line 7), f, u and W_dis (lines 8-10) once; per k < N_z/2 the one inner product y (line 12),
// v = y f, and the mirrored sample at v~ = N_v - 1 - v for slice N_z - 1 - k (lines 15-17,
// Theorem 1).  A thread owns one column and kAlg4K of its k pairs, accumulating all views of
// the launch in registers.  Whole volume only (the mirror pairs k with N_z - 1 - k).
constexpr int kAlg4K = 16;

__device__ __forceinline__ float sample_sw(const float* Qv, int Nu, int Nv, float u, float v)
{
    const float fu = floorf(u), fv = floorf(v);
    const int nu = (int)fu, nv = (int)fv;
    const float du = u - fu, dv = v - fv;
    const float t1 = fmaf(du, tap(Qv, Nu, Nv, nu + 1, nv) - tap(Qv, Nu, Nv, nu, nv),
                          tap(Qv, Nu, Nv, nu, nv));
    const float t2 = fmaf(du, tap(Qv, Nu, Nv, nu + 1, nv + 1) - tap(Qv, Nu, Nv, nu, nv + 1),
                          tap(Qv, Nu, Nv, nu, nv + 1));
    return fmaf(dv, t2 - t1, t1);
}

template <bool HW>
__global__ void __launch_bounds__(256) bp_alg4_kernel(const __grid_constant__ BaseParams p,
                                                      const __grid_constant__ P12Table pt)
{
    const int nkh = (p.nk + 1) / 2;  // k in [0, ceil(N_z / 2)): line 11
    const long ncol = (long)p.Ny * p.Nx;
    const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
    const long kblk = idx / ncol;
    if (kblk * kAlg4K >= nkh) return;
    const long col = idx - kblk * ncol;
    const int i = (int)(col % p.Nx), j = (int)(col / p.Nx);
    const int kbase = (int)kblk * kAlg4K;
    const float fi = (float)i, fj = (float)j;
    float acc[kAlg4K], accm[kAlg4K];
#pragma unroll
    for (int q = 0; q < kAlg4K; ++q) acc[q] = accm[q] = 0.f;
    for (int t = 0; t < p.n_views; ++t) {
        const float* P = pt.P[t];
        const float x = fmaf(P[0], fi, fmaf(P[1], fj, P[3]));   // line 7, t = [i, j, 0, 1]
        const float z = fmaf(P[8], fi, fmaf(P[9], fj, P[11]));
        const float f = 1.f / z;                                 // line 8
        const float u = x * f;                                   // line 9
        const float W = f * f;                                   // line 10
        const float yb = fmaf(P[4], fi, fmaf(P[5], fj, P[7]));
        const float* Qv = HW ? nullptr : p.Q + (long)t * p.Nv * p.Nu;
#pragma unroll
        for (int q = 0; q < kAlg4K; ++q) {
            const int k = kbase + q;
            const float y = fmaf(P[6], (float)k, yb);            // line 12: one inner product
            const float v = y * f;                               // line 13
            const float vm = (float)(p.Nv - 1) - v;              // line 16
            float a, b;
            if (HW) {
                a = tex2DLayered<float>(p.tex, u + 0.5f, v + 0.5f, t);
                b = tex2DLayered<float>(p.tex, u + 0.5f, vm + 0.5f, t);
            } else {
                a = sample_sw(Qv, p.Nu, p.Nv, u, v);
                b = sample_sw(Qv, p.Nu, p.Nv, u, vm);
            }
            acc[q] = fmaf(W, a, acc[q]);                          // line 14
            accm[q] = fmaf(W, b, accm[q]);                        // line 17
        }
    }
#pragma unroll
    for (int q = 0; q < kAlg4K; ++q) {
        const int k = kbase + q, km = p.nk - 1 - k;
        if (k >= nkh) break;
        float* o = p.vol + ((long)k * p.Ny + j) * p.Nx + i;
        *o = p.accumulate ? *o + acc[q] : acc[q];
        if (km != k) {  // odd N_z: the middle slice is its own mirror
            float* om = p.vol + ((long)km * p.Ny + j) * p.Nx + i;
            *om = p.accumulate ? *om + accm[q] : accm[q];
        }
    }
}

}  // namespace

static ifdk_status launch_baseline(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                                   float* vol, int k0, int nk, int accumulate, int hw, bool alg4,
                                   cudaStream_t st)
{
    const size_t view_elems = (size_t)g->Nv * g->Nu;
    for (long t0 = 0; t0 < n_views; t0 += kMaxViews) {
        const int n = (int)((n_views - t0) < kMaxViews ? (n_views - t0) : kMaxViews);
        P12Table pt;
        for (int t = 0; t < n; ++t) {
            double P[12];
            projection_matrix(g, s0 + t0 + t, P);
            for (int q = 0; q < 12; ++q) pt.P[t][q] = (float)P[q];
        }
        BaseParams p{};
        p.Q = Q + t0 * view_elems;
        p.vol = vol;
        p.n_views = n;
        p.Nu = g->Nu; p.Nv = g->Nv; p.Nx = g->Nx; p.Ny = g->Ny;
        p.k0 = k0; p.nk = nk;
        p.accumulate = (accumulate || t0 > 0) ? 1 : 0;
        cudaArray_t arr = nullptr;
        cudaError_t e = cudaSuccess;
        if (hw) {
            // Layered 2-D texture: Nu x Nv texels, one layer per view.
            cudaChannelFormatDesc ch = cudaCreateChannelDesc<float>();
            e = cudaMalloc3DArray(&arr, &ch, make_cudaExtent(g->Nu, g->Nv, n), cudaArrayLayered);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc3DArray(texture baseline)");
            cudaMemcpy3DParms cp{};
            cp.srcPtr = make_cudaPitchedPtr((void*)p.Q, sizeof(float) * g->Nu, g->Nu, g->Nv);
            cp.dstArray = arr;
            cp.extent = make_cudaExtent(g->Nu, g->Nv, n);
            cp.kind = cudaMemcpyDeviceToDevice;
            if ((e = cudaMemcpy3DAsync(&cp, st)) != cudaSuccess) {
                cudaFreeArray(arr);
                return cuda_fail(e, "cudaMemcpy3DAsync(texture baseline)");
            }
            cudaResourceDesc rd{};
            rd.resType = cudaResourceTypeArray;
            rd.res.array.array = arr;
            cudaTextureDesc td{};
            td.addressMode[0] = td.addressMode[1] = td.addressMode[2] = cudaAddressModeBorder;
            td.filterMode = cudaFilterModeLinear;
            td.readMode = cudaReadModeElementType;
            td.normalizedCoords = 0;
            if ((e = cudaCreateTextureObject(&p.tex, &rd, &td, nullptr)) != cudaSuccess) {
                cudaFreeArray(arr);
                return cuda_fail(e, "cudaCreateTextureObject(texture baseline)");
            }
        }
        const long nvox = (long)nk * g->Ny * g->Nx;
        const long nthr = alg4 ? (long)((nk + 1) / 2 + kAlg4K - 1) / kAlg4K * g->Ny * g->Nx : nvox;
        const unsigned grid = (unsigned)((nthr + 255) / 256);
        if (alg4 && hw)
            bp_alg4_kernel<true><<<grid, 256, 0, st>>>(p, pt);
        else if (alg4)
            bp_alg4_kernel<false><<<grid, 256, 0, st>>>(p, pt);
        else if (hw)
            bp_alg2_kernel<true><<<grid, 256, 0, st>>>(p, pt);
        else
            bp_alg2_kernel<false><<<grid, 256, 0, st>>>(p, pt);
        e = cudaGetLastError();
        if (hw) {
            // the texture and its array must outlive the kernel
            cudaStreamSynchronize(st);
            cudaDestroyTextureObject(p.tex);
            cudaFreeArray(arr);
        }
        if (e != cudaSuccess) return cuda_fail(e, "baseline bp kernel launch");
        count_launch();
    }
    return IFDK_OK;
}

ifdk_status launch_backproject_alg2(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                                    float* vol, int k0, int nk, int accumulate, int hw,
                                    cudaStream_t st)
{
    return launch_baseline(g, Q, s0, n_views, vol, k0, nk, accumulate, hw, false, st);
}

ifdk_status launch_backproject_alg4(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                                    float* vol, int accumulate, int hw, cudaStream_t st)
{
    return launch_baseline(g, Q, s0, n_views, vol, 0, g->Nz, accumulate, hw, true, st);
}

}  // namespace ifdk
