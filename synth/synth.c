/*
 * synth.c -- seeded synthetic inputs shared by the oracle and the CUDA path.
 *
 * This module holds NO arithmetic of the FDK method (no filter, no projection
 * matrix, no interpolation, no back-projection).  It only generates inputs:
 *   - raw projections E: analytic line integrals of an ellipsoid phantom
 *     (the paper's "standard Shepp-Logan phantom ... forward-projection",
 *     P:953) through detector pixel centres, computed in fp64, stored fp32;
 *   - the phantom's point density (for truth volumes);
 *   - an optional counter-based Gaussian noise field (seeded).
 * The scanner is described physically (source, detector centre, detector
 * axes) -- reading c-A15 in DESIGN.md -- not through projection matrices.
 *
 * Ellipsoid record (10 doubles): cx, cy, cz, a, b, c, cos(phi), sin(phi), rho, pad.
 * World frame: voxel (i,j,k) centre = (Dx(i-cx), -Dy(j-cy), -Dz(k-cz)).
 */
#include <math.h>
#include <stdint.h>

typedef struct {
    int Nu, Nv;
    double Du, Dv, D, d, theta;
} synth_scanner;

/* Ray from the source through pixel (m, n) of view s; returns source S and
 * direction R (= pixel - S, not normalised). */
static void ray(const synth_scanner *sc, long s, double m, double n, double S[3], double R[3])
{
    const double beta = (double)s * sc->theta;
    const double cb = cos(beta), sb = sin(beta);
    S[0] = -sc->d * sb;
    S[1] = -sc->d * cb;
    S[2] = 0.0;
    const double L = sc->D - sc->d;
    const double uo = (m - (sc->Nu - 1) / 2.0) * sc->Du;
    const double vo = (n - (sc->Nv - 1) / 2.0) * sc->Dv;
    const double px = L * sb + uo * cb;
    const double py = L * cb - uo * sb;
    const double pz = -vo;
    R[0] = px - S[0];
    R[1] = py - S[1];
    R[2] = pz - S[2];
}

/* Length of the chord of line S + t R inside ellipsoid e, times |R| (i.e. in mm). */
static double chord(const double *e, const double S[3], const double R[3])
{
    const double c = e[6], s = e[7];
    /* translate, rotate by -phi about z, scale by semi-axes */
    const double ax = S[0] - e[0], ay = S[1] - e[1], az = S[2] - e[2];
    const double A0 = (c * ax + s * ay) / e[3];
    const double A1 = (-s * ax + c * ay) / e[4];
    const double A2 = az / e[5];
    const double B0 = (c * R[0] + s * R[1]) / e[3];
    const double B1 = (-s * R[0] + c * R[1]) / e[4];
    const double B2 = R[2] / e[5];
    const double qa = B0 * B0 + B1 * B1 + B2 * B2;
    const double qb = A0 * B0 + A1 * B1 + A2 * B2; /* half of the linear coefficient */
    const double qc = A0 * A0 + A1 * A1 + A2 * A2 - 1.0;
    const double disc = qb * qb - qa * qc;
    if (disc <= 0.0) return 0.0;
    const double rn = sqrt(R[0] * R[0] + R[1] * R[1] + R[2] * R[2]);
    return 2.0 * sqrt(disc) / qa * rn;
}

/* E for views s0..s0+n_views-1, detector rows v0..v0+n_rows-1: [n_views][n_rows][Nu] fp32. */
void synth_project(const synth_scanner *sc, const double *ell, int n_ell, long s0, long n_views,
                   int v0, int n_rows, float *E)
{
    const long total = n_views * (long)n_rows;
#pragma omp parallel for schedule(dynamic, 16)
    for (long r = 0; r < total; ++r) {
        const long s = s0 + r / n_rows;
        const int n = v0 + (int)(r % n_rows);
        for (int m = 0; m < sc->Nu; ++m) {
            double S[3], R[3];
            ray(sc, s, m, n, S, R);
            double acc = 0.0;
            for (int q = 0; q < n_ell; ++q) acc += ell[10 * q + 8] * chord(ell + 10 * q, S, R);
            E[r * sc->Nu + m] = (float)acc;
        }
    }
}

/* Phantom density at world points xyz[3*n]. */
void synth_density(const double *ell, int n_ell, long n_pts, const double *xyz, double *out)
{
#pragma omp parallel for schedule(static)
    for (long p = 0; p < n_pts; ++p) {
        double acc = 0.0;
        for (int q = 0; q < n_ell; ++q) {
            const double *e = ell + 10 * q;
            const double ax = xyz[3 * p] - e[0], ay = xyz[3 * p + 1] - e[1], az = xyz[3 * p + 2] - e[2];
            const double x = (e[6] * ax + e[7] * ay) / e[3];
            const double y = (-e[7] * ax + e[6] * ay) / e[4];
            const double z = az / e[5];
            if (x * x + y * y + z * z <= 1.0) acc += e[8];
        }
        out[p] = acc;
    }
}

/* splitmix64 finaliser: the counter-based generator both sides implement. */
static uint64_t mix64(uint64_t x)
{
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

/* E[idx] += sigma * N(0,1), N from Box-Muller on two counter draws of (seed, base+idx). */
void synth_add_noise(float *E, long n, long base, uint64_t seed, double sigma)
{
#pragma omp parallel for schedule(static)
    for (long t = 0; t < n; ++t) {
        const uint64_t c = (uint64_t)(base + t);
        const uint64_t h1 = mix64(seed ^ mix64(2 * c));
        const uint64_t h2 = mix64(seed ^ mix64(2 * c + 1));
        const double u1 = ((double)(h1 >> 11) + 0.5) * (1.0 / 9007199254740992.0);
        const double u2 = (double)(h2 >> 11) * (1.0 / 9007199254740992.0);
        const double g = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        E[t] = (float)((double)E[t] + sigma * g);
    }
}
