/*
 * oracle.c -- plain, slow, double-precision CPU FDK for iFDK (arXiv 1909.02724).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1909_02724_b200/) never links, imports or calls it,
 * and it shares no code, headers, tables or constants with that path.
 *
 * Citation convention: "P:n" is /root/reference/PAPER.md line n (the LaTeX
 * source; the appendix comes first).  Every function follows the paper's
 * definition literally and in the paper's order; there is no blocking,
 * fusion, reordering or incremental evaluation.  All arithmetic is fp64;
 * the only fp32 quantity is the raw projection E, which is the input.
 *
 * Readings of silent / garbled passages are listed in DESIGN.md ("Readings");
 * the ids used below (c-A1 ... c-A16) refer to that list.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

/* Table tbl:cbct-param.  Np is not a field: beta_s = s*theta
 * for the global view index s (reading c-A4). */
typedef struct {
    int Nu, Nv, Nx, Ny, Nz;
    double Du, Dv, Dx, Dy, Dz;
    double D, d, theta;
} oracle_geom;

#define ORACLE_OK 0
#define ORACLE_ERR_BAND 3 /* a tap inside the detector lies outside the supplied row band */

static void mat4_mul(const double A[16], const double B[16], double C[16])
{
    for (int r = 0; r < 4; ++r)
        for (int c = 0; c < 4; ++c) {
            double s = 0.0;
            for (int t = 0; t < 4; ++t) s += A[4 * r + t] * B[4 * t + c];
            C[4 * r + c] = s;
        }
}

/* P_s = (M1 . Mrot . M0)[0:3] -- appendix, P:15-82 (repeated P:524-589).
 * The matrices are typed exactly as printed; P is the top three rows
 * (reading c-A1: 3x4).  Row-major, P[4*r + c]. */
void oracle_projection_matrix(const oracle_geom *g, long s, double P[12])
{
    const double beta = (double)s * g->theta; /* beta = i*theta */
    const double cb = cos(beta), sb = sin(beta);
    const double S0[16] = {g->Dx, 0, 0, 0, 0, g->Dy, 0, 0, 0, 0, g->Dz, 0, 0, 0, 0, 1};
    const double C0[16] = {1, 0, 0, -(g->Nx - 1) / 2.0,
                           0, -1, 0, (g->Ny - 1) / 2.0,
                           0, 0, -1, (g->Nz - 1) / 2.0,
                           0, 0, 0, 1};
    const double SW[16] = {1, 0, 0, 0, 0, 0, -1, 0, 0, 1, 0, g->d, 0, 0, 0, 1};
    const double RO[16] = {cb, -sb, 0, 0, sb, cb, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
    const double SC[16] = {1.0 / g->Du, 0, 0, 0, 0, 1.0 / g->Dv, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1};
    const double PR[16] = {g->D, 0, (g->Nu - 1) * g->Du / 2.0, 0,
                           0, g->D, (g->Nv - 1) * g->Dv / 2.0, 0,
                           0, 0, 1, 0,
                           0, 0, 0, 1};
    double M0[16], Mrot[16], M1[16], T[16], Phat[16];
    mat4_mul(S0, C0, M0);   /* M0   = Scale . Center  */
    mat4_mul(SW, RO, Mrot); /* Mrot = Swap  . Rot(beta)  */
    mat4_mul(SC, PR, M1);   /* M1   = Pitch^-1 . Persp  */
    mat4_mul(Mrot, M0, T);
    mat4_mul(M1, T, Phat); /* P^ = M1 . Mrot . M0     */
    memcpy(P, Phat, 12 * sizeof(double)); /* P = P^[0:3]  */
}

/* F_cos, the 2-D cosine table (Alg. alg:filter line 2).
 * Reading c-A5: D / sqrt(D^2 + u^2 + v^2) with u, v the physical offsets of
 * detector pixel (m, v) from the detector centre. */
double oracle_cos_weight(const oracle_geom *g, int m, int v)
{
    const double uh = (m - (g->Nu - 1) / 2.0) * g->Du;
    const double vh = (v - (g->Nv - 1) / 2.0) * g->Dv;
    return g->D / sqrt(g->D * g->D + uh * uh + vh * vh);
}

/* F_ramp, reading c-A6: the unit-spacing Ram-Lak kernel
 * h1[0] = 1/4, h1[n odd] = -1/(pi^2 n^2), h1[n even != 0] = 0. */
double oracle_ramp_h1(long n)
{
    if (n == 0) return 0.25;
    if (n % 2 == 0) return 0.0;
    const double pi = 3.14159265358979323846;
    return -1.0 / (pi * pi * (double)n * (double)n);
}

/* Reading c-A7: the FDK constant folded into Q,  C = theta * d * D / (2 Du). */
double oracle_fdk_scale(const oracle_geom *g)
{
    return g->theta * g->d * g->D / (2.0 * g->Du);
}

/* Alg. alg:filter on detector rows v0 .. v0+n_rows-1 of n_views
 * projections.  E and Q are [n_views][n_rows][Nu]; E is fp32 (the input),
 * Q is fp64.  Line 2: E~ = E . F_cos (point-wise).  Line 4: each row of E~
 * convolved with F_ramp -- a full-length linear convolution written out as
 * the direct sum (reading c-A6), output aligned with input index n. */
void oracle_filter(const oracle_geom *g, const float *E, long n_views, int v0, int n_rows,
                   double *Q)
{
    const int Nu = g->Nu;
    const double C = oracle_fdk_scale(g);
    const long n_total = n_views * (long)n_rows;
#pragma omp parallel
    {
        double *Et = (double *)malloc(sizeof(double) * (size_t)Nu);
#pragma omp for schedule(dynamic, 4)
        for (long r = 0; r < n_total; ++r) {
            const int v = v0 + (int)(r % n_rows);
            const float *e = E + r * Nu;
            for (int m = 0; m < Nu; ++m) Et[m] = (double)e[m] * oracle_cos_weight(g, m, v);
            double *q = Q + r * Nu;
            for (int n = 0; n < Nu; ++n) {
                double s = 0.0;
                for (int m = 0; m < Nu; ++m) s += Et[m] * oracle_ramp_h1((long)n - m);
                q[n] = C * s;
            }
        }
        free(Et);
    }
}

/* One tap T(a, b) = X(a, b) of Alg. alg:subpixel, where X(n_u, n_v)
 * is Q[n_v][n_u] (reading c-A10) and taps off the detector read 0 (reading
 * c-A9).  Q holds only detector rows v0 .. v0+n_rows-1: a tap on the detector
 * but outside that band sets *missing. */
static double tap(const oracle_geom *g, const double *Q, int v0, int n_rows, long a, long b,
                  int *missing)
{
    if (a < 0 || a >= g->Nu || b < 0 || b >= g->Nv) return 0.0;
    if (b < v0 || b >= (long)v0 + n_rows) {
        *missing = 1;
        return 0.0;
    }
    return Q[(b - v0) * (long)g->Nu + a];
}

/* Alg. alg:subpixel, bilinear interpolation with sub-pixel
 * precision; int() is read as floor (reading c-A8). */
double oracle_interp2(const oracle_geom *g, const double *Q, int v0, int n_rows, double u,
                      double v, int *missing)
{
    const double fu = floor(u), fv = floor(v);
    const long nu = (long)fu, nv = (long)fv;
    const double du = u - fu, dv = v - fv;
    const double t1 = tap(g, Q, v0, n_rows, nu, nv, missing) * (1.0 - du) +
                      tap(g, Q, v0, n_rows, nu + 1, nv, missing) * du;
    const double t2 = tap(g, Q, v0, n_rows, nu, nv + 1, missing) * (1.0 - du) +
                      tap(g, Q, v0, n_rows, nu + 1, nv + 1, missing) * du;
    return t1 * (1.0 - dv) + t2 * dv;
}

/* Alg. alg:bp, the plain back-projection, for a list of voxels.
 * Q: filtered views s0 .. s0+n_views-1, each holding detector rows
 * v0 .. v0+n_rows-1, [n_views][n_rows][Nu] fp64.  ijk: n_vox triples (i,j,k).
 * out[n] = sum over s (in order) of f^2 * interp2(Q_s, x f, y f),
 * [x,y,z] = P_s . [i,j,k,1], f = 1/z  (lines 6-10).
 * Returns ORACLE_ERR_BAND if any in-detector tap falls outside the band. */
int oracle_backproject(const oracle_geom *g, const double *Q, long s0, long n_views, int v0,
                       int n_rows, long n_vox, const int *ijk, double *out)
{
    double *P = (double *)malloc(sizeof(double) * 12 * (size_t)(n_views > 0 ? n_views : 1));
    for (long t = 0; t < n_views; ++t) oracle_projection_matrix(g, s0 + t, P + 12 * t);
    int missing_any = 0;
#pragma omp parallel for schedule(dynamic, 64) reduction(| : missing_any)
    for (long n = 0; n < n_vox; ++n) {
        const double i = ijk[3 * n], j = ijk[3 * n + 1], k = ijk[3 * n + 2];
        double I = 0.0;
        int missing = 0;
        for (long t = 0; t < n_views; ++t) {
            const double *Ps = P + 12 * t;
            const double x = Ps[0] * i + Ps[1] * j + Ps[2] * k + Ps[3];
            const double y = Ps[4] * i + Ps[5] * j + Ps[6] * k + Ps[7];
            const double z = Ps[8] * i + Ps[9] * j + Ps[10] * k + Ps[11];
            const double f = 1.0 / z;
            const double W = f * f; /* distance weight, line 8 */
            const double u = x * f, v = y * f;
            I += W * oracle_interp2(g, Q + t * (long)n_rows * g->Nu, v0, n_rows, u, v, &missing);
        }
        out[n] = I;
        missing_any |= missing;
    }
    free(P);
    return missing_any ? ORACLE_ERR_BAND : ORACLE_OK;
}

/* Whole-volume form of Alg. alg:bp: out is [Nz][Ny][Nx] (i fastest) for the
 * k range k0 .. k0+nk-1.  Same arithmetic as oracle_backproject. */
int oracle_backproject_volume(const oracle_geom *g, const double *Q, long s0, long n_views,
                              int v0, int n_rows, int k0, int nk, double *out)
{
    const long n_vox = (long)nk * g->Ny * g->Nx;
    int *ijk = (int *)malloc(sizeof(int) * 3 * (size_t)(n_vox > 0 ? n_vox : 1));
    long n = 0;
    for (int k = k0; k < k0 + nk; ++k)
        for (int j = 0; j < g->Ny; ++j)
            for (int i = 0; i < g->Nx; ++i, ++n) {
                ijk[3 * n] = i;
                ijk[3 * n + 1] = j;
                ijk[3 * n + 2] = k;
            }
    int st = oracle_backproject(g, Q, s0, n_views, v0, n_rows, n_vox, ijk, out);
    free(ijk);
    return st;
}

/* The matched forward projector (reading c-I1): the transpose of Alg. alg:bp +
 * alg:subpixel.  Back-projection is V = sum_s sum_taps W w_tap Q_s[tap] (lines
 * 6-10 with interp2 written as its four weighted taps), so its transpose adds
 * W * w_tap * vol(i,j,k) into every tap of every voxel's projection:
 *   out[t][b - v0][a] = sum_{i,j,k} f^2 w_(a,b)(x f, y f) vol[k - k0][j][i],
 * with w_(a,b) the bilinear weight of tap (a, b) in Alg. alg:subpixel (t1, t2
 * and the final lerp multiplied out), taps off the detector dropped (c-A9).
 * vol: [nk][Ny][Nx] slab k0..k0+nk-1 (fp64); out: [n_views][n_rows][Nu] fp64,
 * rows v0 .. v0+n_rows-1, overwritten.  Views in parallel, voxels in order.
 * Returns ORACLE_ERR_BAND if a tap on the detector falls outside the band. */
int oracle_forward_project(const oracle_geom *g, const double *vol, int k0, int nk, long s0,
                           long n_views, int v0, int n_rows, double *out)
{
    int missing_any = 0;
#pragma omp parallel for schedule(dynamic, 1) reduction(| : missing_any)
    for (long t = 0; t < n_views; ++t) {
        double P[12];
        oracle_projection_matrix(g, s0 + t, P);
        double *o = out + t * (long)n_rows * g->Nu;
        for (long e = 0; e < (long)n_rows * g->Nu; ++e) o[e] = 0.0;
        for (int k = k0; k < k0 + nk; ++k)
            for (int j = 0; j < g->Ny; ++j)
                for (int i = 0; i < g->Nx; ++i) {
                    const double val = vol[((long)(k - k0) * g->Ny + j) * g->Nx + i];
                    const double x = P[0] * i + P[1] * j + P[2] * k + P[3];
                    const double y = P[4] * i + P[5] * j + P[6] * k + P[7];
                    const double z = P[8] * i + P[9] * j + P[10] * k + P[11];
                    const double f = 1.0 / z;
                    const double W = f * f; /* line 8 */
                    const double u = x * f, v = y * f;
                    const double fu = floor(u), fv = floor(v); /* c-A8 */
                    const long nu = (long)fu, nv = (long)fv;
                    const double du = u - fu, dv = v - fv;
                    /* interp2 = T(nu,nv)(1-du)(1-dv) + T(nu+1,nv) du(1-dv)
                     *         + T(nu,nv+1)(1-du) dv + T(nu+1,nv+1) du dv */
                    const long ta[4] = {nu, nu + 1, nu, nu + 1};
                    const long tb[4] = {nv, nv, nv + 1, nv + 1};
                    const double w[4] = {(1.0 - du) * (1.0 - dv), du * (1.0 - dv),
                                         (1.0 - du) * dv, du * dv};
                    for (int q = 0; q < 4; ++q) {
                        const long a = ta[q], b = tb[q];
                        if (a < 0 || a >= g->Nu || b < 0 || b >= g->Nv) continue; /* c-A9 */
                        if (b < v0 || b >= (long)v0 + n_rows) {
                            if (w[q] * val != 0.0) missing_any = 1;
                            continue;
                        }
                        o[(b - v0) * (long)g->Nu + a] += W * w[q] * val;
                    }
                }
    }
    return missing_any ? ORACLE_ERR_BAND : ORACLE_OK;
}

int oracle_num_threads(void)
{
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
