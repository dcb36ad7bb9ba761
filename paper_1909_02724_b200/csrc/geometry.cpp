// geometry.cpp -- host geometry core of libifdk (fp64).
//
// P_s is the top three rows of M1 . Mrot . M0 (appendix).
// Expanding the printed product once by hand gives, with X = Dx (i - cx),
// Y = Dy (j - cy), c = cos(beta), s = sin(beta):
//     z = d + s X - c Y                                    (Eq. equ:z)
//     x = (D/Du) (c X + s Y) + cu z
//     y = (D/Dv) Dz (k - cz) + cv z
// so row 2 and row 0 have no k term (Theorems 2-3).  The rows are
// assembled from these closed forms; P[0][2] = P[2][2] = 0 exactly.
#include <cmath>
#include <cstring>

#include "ifdk_internal.h"

namespace ifdk {

void projection_matrix(const ifdk_geometry* g, long s, double P[12])
{
    const double beta = (double)s * g->theta;  // beta = i theta
    const double c = std::cos(beta), sn = std::sin(beta);
    // row 2: z
    P[8] = sn * g->Dx;
    P[9] = -c * g->Dy;
    P[10] = 0.0;
    P[11] = g->d - sn * g->Dx * g->cx + c * g->Dy * g->cy;
    // row 0: x = (D/Du)(c X + s Y) + cu z
    const double mu = g->D / g->Du;
    P[0] = mu * c * g->Dx + g->cu * P[8];
    P[1] = mu * sn * g->Dy + g->cu * P[9];
    P[2] = 0.0;
    P[3] = mu * (-c * g->Dx * g->cx - sn * g->Dy * g->cy) + g->cu * P[11];
    // row 1: y = (D/Dv) Dz (k - cz) + cv z
    const double mv = g->D / g->Dv;
    P[4] = g->cv * P[8];
    P[5] = g->cv * P[9];
    P[6] = mv * g->Dz;
    P[7] = -mv * g->Dz * g->cz + g->cv * P[11];
}

void band_rows(const ifdk_geometry* g, int k0, int nk, long s, int* lo, int* hi)
{
    const double beta = (double)s * g->theta;
    const double c = std::cos(beta), sn = std::sin(beta);
    double zlo = 1e300, zhi = -1e300;
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            const double X = g->Dx * ((a ? g->Nx - 1 : 0) - g->cx);
            const double Y = g->Dy * ((b ? g->Ny - 1 : 0) - g->cy);
            const double z = g->d + sn * X - c * Y;
            zlo = std::fmin(zlo, z);
            zhi = std::fmax(zhi, z);
        }
    const double K = g->D * g->Dz / g->Dv;
    double vmin = 1e300, vmax = -1e300;
    const int ks[2] = {k0, k0 + nk - 1};
    const double zs[2] = {zlo, zhi};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b) {
            const double v = g->cv + K * (ks[a] - g->cz) / zs[b];
            vmin = std::fmin(vmin, v);
            vmax = std::fmax(vmax, v);
        }
    long l = (long)std::floor(vmin) - 1, h = (long)std::floor(vmax) + 2;
    if (l < 0) l = 0;
    if (h > g->Nv - 1) h = g->Nv - 1;
    *lo = (int)l;
    *hi = (int)h;
}

void patch_bound(const ifdk_geometry* g, int ti, int tj, int kc, double* w, double* h)
{
    // For two points of one tile, |u1-u2| <= (D/Du) [L / zmin + rxy L / zmin^2] with L the
    // tile diagonal in the rotation plane (u - cu = (D/Du) a / z, |a| <= rxy, |da|,|dz| <= L).
    const double Lx = (ti - 1) * g->Dx, Ly = (tj - 1) * g->Dy;
    const double L = std::sqrt(Lx * Lx + Ly * Ly);
    const double zmin = g->zmin;
    *w = g->D / g->Du * (L / zmin + g->rxy * L / (zmin * zmin));
    // v - cv = K (k - cz) / z: over kc slices and the tile's z spread.
    const double K = g->D * g->Dz / g->Dv;
    const double kmax = std::fmax(g->cz, (g->Nz - 1) - g->cz);
    *h = K * ((kc - 1) / zmin + kmax * L / (zmin * zmin));
}

// Ramp filter spectrum for an FFT of length L >= 2 Nu - 1 (reading c-A6: full-length linear
// convolution with the unit-spacing Ram-Lak kernel h1).  h1 is even, so its DFT is real:
//   H[f] = h1[0] + 2 sum_{l=1}^{Nu-1} h1[l] cos(2 pi f l / L).
// The FDK constant C (reading c-A7) and the 1/L of the inverse transform are folded in.
void ensure_filter_tables_host(ifdk_geometry* g)
{
    if (g->log2L) return;
    // Nu <= 2048: the register radix-16 kernel of fixed length 4096 (any L >= 2 Nu - 1 gives
    // the same linear convolution); larger rows: the generic Stockham kernel, minimal L.
    int log2L = 12;
    if (g->Nu > 2048)
        while ((1 << log2L) < 2 * g->Nu - 1) ++log2L;
    const int L = 1 << log2L;
    const double pi = 3.14159265358979323846;
    std::vector<double> h(g->Nu, 0.0);
    h[0] = 0.25;
    for (int l = 1; l < g->Nu; l += 2) h[l] = -1.0 / (pi * pi * (double)l * (double)l);
    g->Hs.assign(L / 2 + 1, 0.f);
    for (int f = 0; f <= L / 2; ++f) {
        double acc = h[0];
        for (int l = 1; l < g->Nu; l += 2) {
            // cos(2 pi f l / L) with the argument reduced exactly in integers
            const long r = ((long)f * l) % L;
            acc += 2.0 * h[l] * std::cos(2.0 * pi * (double)r / L);
        }
        // C / L and the D of F_cos = D / sqrt(D^2 + u^2 + v^2) (the kernels weight by the
        // reciprocal square root alone; the filter is linear)
        g->Hs[f] = (float)(acc * g->C * g->D / L);
    }
    g->tw.assign(2 * (size_t)L, 0.f);
    for (int t = 0; t < L; ++t) {
        g->tw[2 * t] = (float)std::cos(2.0 * pi * t / L);
        g->tw[2 * t + 1] = (float)(-std::sin(2.0 * pi * t / L));
    }
    g->log2L = log2L;
}

}  // namespace ifdk

using namespace ifdk;

extern "C" ifdk_status ifdk_geometry_create(int Nu, int Nv, int Nx, int Ny, int Nz, double Du,
                                            double Dv, double Dx, double Dy, double Dz, double D,
                                            double d, double theta, ifdk_geometry** out)
{
    if (!out) return fail(IFDK_ERR_INVALID_ARGUMENT, "out is NULL");
    *out = nullptr;
    if (Nu < 1 || Nv < 1 || Nx < 1 || Ny < 1 || Nz < 1)
        return fail(IFDK_ERR_INVALID_ARGUMENT, "every dimension must be >= 1");
    if (Nu > (1 << 16) || Nv > (1 << 20) || Nx > (1 << 16) || Ny > (1 << 16) || Nz > (1 << 20))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "dimension too large");
    const double pit[5] = {Du, Dv, Dx, Dy, Dz};
    for (double p : pit)
        if (!(p > 0.0) || !std::isfinite(p))
            return fail(IFDK_ERR_INVALID_ARGUMENT, "every pitch must be finite and > 0");
    if (!(d > 0.0) || !(D > d) || !std::isfinite(D))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "need 0 < d < D (finite)");
    if (!std::isfinite(theta) || !(theta > 0.0))
        return fail(IFDK_ERR_INVALID_ARGUMENT, "theta must be finite and > 0");
    auto* g = new ifdk_geometry();
    g->Nu = Nu; g->Nv = Nv; g->Nx = Nx; g->Ny = Ny; g->Nz = Nz;
    g->Du = Du; g->Dv = Dv; g->Dx = Dx; g->Dy = Dy; g->Dz = Dz;
    g->D = D; g->d = d; g->theta = theta;
    g->cu = (Nu - 1) / 2.0; g->cv = (Nv - 1) / 2.0;
    g->cx = (Nx - 1) / 2.0; g->cy = (Ny - 1) / 2.0; g->cz = (Nz - 1) / 2.0;
    g->C = theta * d * D / (2.0 * Du);
    const double hx = g->cx * Dx, hy = g->cy * Dy;
    g->rxy = std::sqrt(hx * hx + hy * hy);
    if (!(g->rxy < d)) {
        delete g;
        return fail(IFDK_ERR_DEGENERATE_GEOMETRY,
                    "volume not inside the source circle: some voxel could reach z <= 0");
    }
    g->zmin = d - g->rxy;
    g->zmax = d + g->rxy;
    *out = g;
    return IFDK_OK;
}

extern "C" ifdk_status ifdk_projection_matrix(const ifdk_geometry* g, long s, double P[12])
{
    if (!g || !P) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    projection_matrix(g, s, P);
    return IFDK_OK;
}

extern "C" ifdk_status ifdk_band_rows(const ifdk_geometry* g, int k0, int nk, long s, int* v_lo,
                                      int* v_hi)
{
    if (!g || !v_lo || !v_hi) return fail(IFDK_ERR_INVALID_ARGUMENT, "NULL argument");
    if (k0 < 0 || nk < 1 || (long)k0 + nk > g->Nz)
        return fail(IFDK_ERR_SHAPE, "slab outside [0, Nz)");
    band_rows(g, k0, nk, s, v_lo, v_hi);
    return IFDK_OK;
}
