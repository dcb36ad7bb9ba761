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
// (DESIGN.md "Numerics").
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

}  // namespace

ifdk_status launch_backproject_alg2(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                                    float* vol, int k0, int nk, int accumulate, int hw,
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
        const unsigned grid = (unsigned)((nvox + 255) / 256);
        if (hw)
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
        if (e != cudaSuccess) return cuda_fail(e, "bp_alg2_kernel launch");
        count_launch();
    }
    return IFDK_OK;
}

}  // namespace ifdk
