// kwalk.cuh -- the k-walk arithmetic shared by the back-projector (backproject.cu) and its
// transpose, the matched forward projector (forward.cu): per-launch tables of P_s and the
// per-(column, view) invariants of the appendix (Theorems 2-3).
#pragma once
#include <cstdint>

#include "ifdk_internal.h"

namespace ifdk {

// Views per launch: their projection matrices ride in the kernel's parameter space
// (20 KB of the 32 KB parameter limit).  A multiple of the summation batch vb = 128.
constexpr int kMaxViewsPerLaunch = 256;

// The used entries of P_s (P[0][2] = P[2][2] = 0, Theorems 2-3):
// P00 P01 P03 | P10 P11 P12 P13 | P20 P21 P23
struct PTable {
    double P[kMaxViewsPerLaunch][10];
};

// Host: the used entries of P_s for views s0 .. s0+n_views-1 (n_views <= kMaxViewsPerLaunch).
inline void fill_ptable(const ifdk_geometry* g, long s0, long n_views, PTable& pt)
{
    for (long t = 0; t < n_views; ++t) {
        double P[12];
        projection_matrix(g, s0 + t, P);
        double* o = pt.P[t];
        o[0] = P[0]; o[1] = P[1]; o[2] = P[3];
        o[3] = P[4]; o[4] = P[5]; o[5] = P[6]; o[6] = P[7];
        o[7] = P[8]; o[8] = P[9]; o[9] = P[11];
    }
    for (long t = n_views; t < kMaxViewsPerLaunch; ++t)
        for (int q = 0; q < 10; ++q) pt.P[t][q] = 0.0;
}

// Per-(column, view) invariants in fp64 (Theorems 2-3): u and 1/z are k-invariant; v at the
// chunk base kb; dv = dv/dk.  Shared by the threads and by the patch-bound computation so
// that corner columns reproduce the threads' values bit for bit.
struct ColInv {
    double u, v, f, dv, z;
};

__device__ __forceinline__ ColInv column_invariants(const double* P, double i, double j, double kb)
{
    ColInv c;
    const double x = fma(P[0], i, fma(P[1], j, P[2]));
    const double y = fma(P[3], i, fma(P[4], j, fma(P[5], kb, P[6])));
    const double z = fma(P[7], i, fma(P[8], j, P[9]));
    c.z = z;
    c.f = __drcp_rn(z);
    c.u = x * c.f;
    c.v = y * c.f;
    c.dv = P[5] * c.f;
    return c;
}

// Thread-side split of the invariants: integer detector column/row + fp32 fractions.
struct ThreadInv {
    int nu, nv;
    float du, fv0, dv, dvm1, W;
    // dv = dvi + dvf split in fp64 (the single-slice walk, any dv: v(kk) = fv0 + kk dvf in fp32
    // plus kk dvi whole rows, so its fp32 part stays below KC + 1 instead of KC dv)
    int dvi;
    float dvf;
};

__device__ __forceinline__ ThreadInv split(const ColInv& c)
{
    ThreadInv t;
    const double fu = floor(c.u), fv = floor(c.v);
    t.nu = (int)fu;
    t.nv = (int)fv;
    t.du = (float)(c.u - fu);
    t.fv0 = (float)(c.v - fv);
    t.dv = (float)c.dv;
    t.dvm1 = t.dv - 1.f;
    const double fdv = floor(c.dv);
    t.dvi = (int)fdv;
    t.dvf = (float)(c.dv - fdv);
    t.W = (float)(c.f * c.f);  // W_dis = f^2, Alg. alg:bp line 8
    return t;
}

// floor() of a non-negative fp32 v < 2^23 through the round-down magic add: the returned
// bits are 0x4B000000 + floor(v); *fr = v - floor(v) exactly.
__device__ __forceinline__ uint32_t floor_bits(float v, float* fr)
{
    const float t = __fadd_rd(v, 8388608.0f);
    *fr = v - (t - 8388608.0f);
    return __float_as_uint(t);
}

}  // namespace ifdk
