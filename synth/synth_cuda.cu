// synth_cuda.cu -- GPU twin of synth.c's synth_project (input generation only;
// no FDK arithmetic).  Same physical scanner description, same fp64 formulas,
// so that config-4/5 inputs can be made in HBM in well under a second.
#include <cuda_runtime.h>
#include <math.h>

struct synth_scanner {
    int Nu, Nv;
    double Du, Dv, D, d, theta;
};

__global__ void synth_project_kernel(synth_scanner sc, const double* __restrict__ ell, int n_ell,
                                     long s0, long n_views, int v0, int n_rows,
                                     float* __restrict__ E)
{
    const long total = n_views * (long)n_rows * sc.Nu;
    for (long p = blockIdx.x * (long)blockDim.x + threadIdx.x; p < total;
         p += (long)gridDim.x * blockDim.x) {
        const int m = (int)(p % sc.Nu);
        const long r = p / sc.Nu;
        const long s = s0 + r / n_rows;
        const int n = v0 + (int)(r % n_rows);
        const double beta = (double)s * sc.theta;
        double sb, cb;
        sincos(beta, &sb, &cb);
        const double S0 = -sc.d * sb, S1 = -sc.d * cb, S2 = 0.0;
        const double L = sc.D - sc.d;
        const double uo = (m - (sc.Nu - 1) / 2.0) * sc.Du;
        const double vo = (n - (sc.Nv - 1) / 2.0) * sc.Dv;
        const double R0 = (L * sb + uo * cb) - S0;
        const double R1 = (L * cb - uo * sb) - S1;
        const double R2 = -vo - S2;
        const double rn = sqrt(R0 * R0 + R1 * R1 + R2 * R2);
        double acc = 0.0;
        for (int q = 0; q < n_ell; ++q) {
            const double* e = ell + 10 * q;
            const double c = e[6], s_ = e[7];
            const double ax = S0 - e[0], ay = S1 - e[1], az = S2 - e[2];
            const double A0 = (c * ax + s_ * ay) / e[3];
            const double A1 = (-s_ * ax + c * ay) / e[4];
            const double A2 = az / e[5];
            const double B0 = (c * R0 + s_ * R1) / e[3];
            const double B1 = (-s_ * R0 + c * R1) / e[4];
            const double B2 = R2 / e[5];
            const double qa = B0 * B0 + B1 * B1 + B2 * B2;
            const double qb = A0 * B0 + A1 * B1 + A2 * B2;
            const double qc = A0 * A0 + A1 * A1 + A2 * A2 - 1.0;
            const double disc = qb * qb - qa * qc;
            if (disc > 0.0) acc += e[8] * (2.0 * sqrt(disc) / qa * rn);
        }
        E[p] = (float)acc;
    }
}

extern "C" int synth_project_cuda(const synth_scanner* sc, const double* ell_host, int n_ell,
                                  long s0, long n_views, int v0, int n_rows, void* E_dev,
                                  void* stream)
{
    cudaStream_t st = (cudaStream_t)stream;
    double* ell_dev = nullptr;
    if (cudaMallocAsync(&ell_dev, sizeof(double) * 10 * n_ell, st) != cudaSuccess) return 1;
    cudaMemcpyAsync(ell_dev, ell_host, sizeof(double) * 10 * n_ell, cudaMemcpyHostToDevice, st);
    synth_project_kernel<<<148 * 16, 256, 0, st>>>(*sc, ell_dev, n_ell, s0, n_views, v0, n_rows,
                                                   (float*)E_dev);
    cudaFreeAsync(ell_dev, st);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
