// filter.cu -- FILT-sm100: fused cosine weight + ramp filter (Alg. alg:filter).
//
// Each detector row of Nu samples is cosine weighted (reading c-A5), zero padded to
// L = 2^k >= 2 Nu - 1 and convolved with the full-length Ram-Lak kernel through the
// convolution theorem: Q = IFFT(FFT(E~) . H), keeping samples 0..Nu-1, which
// equals the linear convolution exactly (reading c-A6).  H is real and even, so two rows
// ride in one complex transform (row A in the real part, row B in the imaginary part):
// FFT(a + i b) . H = FFT(a) H + i FFT(b) H, and both filtered rows are real.
// The inverse uses conj(FFT(conj(Y))); the FDK constant C and 1/L live in H.
//
// One CTA of 256 threads owns a pair of rows at a time (persistent grid); the transform is
// a shared-memory Stockham autosort FFT (one radix-2 pass when log2 L is odd, then radix-4
// passes), ping-ponging between two L-element complex buffers.  The roofline is HBM:
// 8 algorithmic bytes per detector pixel (read E, write Q).
#include <cmath>

#include "ifdk_internal.h"

namespace ifdk {
namespace {

constexpr int kThreads = 256;

struct FilterParams {
    const float* raw;
    float* out;
    long n_rows_total;  // n_views * n_rows
    int n_rows;         // rows per view
    int v0;             // first detector row of each view
    int Nu;
    float D2, D, Du, Dv, cu, cv;
};

__device__ __forceinline__ float2 cmul(float2 a, float2 b)
{
    return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}

// One Stockham pass of radix R (2 or 4) over length L: in -> out, span p.
template <int R>
__device__ __forceinline__ void stockham_pass(const float2* __restrict__ in, float2* __restrict__ out,
                                              const float2* __restrict__ tw, int L, int p)
{
    const int T = L / R;
    const int twstep = L / (R * p);
    for (int i = threadIdx.x; i < T; i += kThreads) {
        const int k = i & (p - 1);
        if (R == 2) {
            const float2 u0 = in[i];
            const float2 u1 = cmul(in[i + T], __ldg(&tw[k * twstep]));
            const int b = ((i - k) << 1) + k;
            out[b] = make_float2(u0.x + u1.x, u0.y + u1.y);
            out[b + p] = make_float2(u0.x - u1.x, u0.y - u1.y);
        } else {
            const float2 u0 = in[i];
            const float2 u1 = cmul(in[i + T], __ldg(&tw[k * twstep]));
            const float2 u2 = cmul(in[i + 2 * T], __ldg(&tw[2 * k * twstep]));
            const float2 u3 = cmul(in[i + 3 * T], __ldg(&tw[3 * k * twstep]));
            const float2 a0 = make_float2(u0.x + u2.x, u0.y + u2.y);
            const float2 a1 = make_float2(u0.x - u2.x, u0.y - u2.y);
            const float2 a2 = make_float2(u1.x + u3.x, u1.y + u3.y);
            const float2 a3 = make_float2(u1.y - u3.y, u3.x - u1.x);  // -i (u1 - u3)
            const int b = ((i - k) << 2) + k;
            out[b] = make_float2(a0.x + a2.x, a0.y + a2.y);
            out[b + p] = make_float2(a1.x + a3.x, a1.y + a3.y);
            out[b + 2 * p] = make_float2(a0.x - a2.x, a0.y - a2.y);
            out[b + 3 * p] = make_float2(a1.x - a3.x, a1.y - a3.y);
        }
    }
}

// Full forward FFT of buf[0] (natural order in and out); returns the buffer index holding
// the result.
__device__ __forceinline__ int fft_forward(float2* buf0, float2* buf1, const float2* tw, int log2L)
{
    const int L = 1 << log2L;
    float2* src = buf0;
    float2* dst = buf1;
    int cur = 0, p = 1;
    if (log2L & 1) {
        stockham_pass<2>(src, dst, tw, L, p);
        __syncthreads();
        float2* t = src; src = dst; dst = t;
        cur ^= 1;
        p <<= 1;
    }
    while (p < L) {
        stockham_pass<4>(src, dst, tw, L, p);
        __syncthreads();
        float2* t = src; src = dst; dst = t;
        cur ^= 1;
        p <<= 2;
    }
    return cur;
}

__global__ void __launch_bounds__(kThreads) filter_fft_kernel(const FilterParams p,
                                                              const float2* __restrict__ tw,
                                                              const float* __restrict__ Hs,
                                                              int log2L)
{
    extern __shared__ float2 smem[];
    const int L = 1 << log2L;
    float2* buf0 = smem;
    float2* buf1 = smem + L;
    const long n_pairs = (p.n_rows_total + 1) / 2;
    for (long pr = blockIdx.x; pr < n_pairs; pr += gridDim.x) {
        const long rA = 2 * pr, rB = 2 * pr + 1;
        const bool hasB = rB < p.n_rows_total;
        const float vA = (float)(p.v0 + (int)(rA % p.n_rows)) - p.cv;
        const float vB = (float)(p.v0 + (int)(rB % p.n_rows)) - p.cv;
        const float vhA = vA * p.Dv, vhB = vB * p.Dv;
        const float* eA = p.raw + rA * p.Nu;
        const float* eB = p.raw + rB * p.Nu;
        // Alg. alg:filter line 2: E~ = E . F_cos, packed as (row A, row B), zero padded.
        for (int m = threadIdx.x; m < L; m += kThreads) {
            float2 x = make_float2(0.f, 0.f);
            if (m < p.Nu) {
                const float uh = ((float)m - p.cu) * p.Du;
                const float uh2 = uh * uh;
                const float wA = p.D / sqrtf(p.D2 + uh2 + vhA * vhA);
                x.x = __ldg(eA + m) * wA;
                if (hasB) {
                    const float wB = p.D / sqrtf(p.D2 + uh2 + vhB * vhB);
                    x.y = __ldg(eB + m) * wB;
                }
            }
            buf0[m] = x;
        }
        __syncthreads();
        int cur = fft_forward(buf0, buf1, tw, log2L);
        float2* X = cur ? buf1 : buf0;
        // Y = X . H (H real, even), then conj for the inverse-by-forward trick.
        for (int f = threadIdx.x; f < L; f += kThreads) {
            const float h = __ldg(&Hs[f <= L / 2 ? f : L - f]);
            const float2 v = X[f];
            X[f] = make_float2(v.x * h, -v.y * h);
        }
        __syncthreads();
        float2* other = cur ? buf0 : buf1;
        cur = fft_forward(X, other, tw, log2L);
        float2* Z = (cur ? other : X);
        // Q = conj(Z): real part -> row A, -imag part -> row B (first Nu samples).
        float* qA = p.out + rA * p.Nu;
        float* qB = p.out + rB * p.Nu;
        for (int n = threadIdx.x; n < p.Nu; n += kThreads) {
            const float2 z = Z[n];
            qA[n] = z.x;
            if (hasB) qB[n] = -z.y;
        }
        __syncthreads();
    }
}

}  // namespace

ifdk_status launch_filter(ifdk_geometry* g, const float* raw, float* out, long n_views, int v0,
                          int n_rows, cudaStream_t st)
{
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev >= 32) return fail(IFDK_ERR_CUDA, "device index >= 32 unsupported");
    {
        std::lock_guard<std::mutex> lk(g->mu);
        ensure_filter_tables_host(g);
        auto& D = g->dev[dev];
        if (!D.Hs) {
            const int L = 1 << g->log2L;
            if ((e = cudaMalloc(&D.Hs, sizeof(float) * (L / 2 + 1))) != cudaSuccess)
                return cuda_fail(e, "cudaMalloc(filter spectrum)");
            if ((e = cudaMalloc(&D.tw, sizeof(float2) * L)) != cudaSuccess)
                return cuda_fail(e, "cudaMalloc(twiddles)");
            cudaMemcpy(D.Hs, g->Hs.data(), sizeof(float) * (L / 2 + 1), cudaMemcpyHostToDevice);
            e = cudaMemcpy(D.tw, g->tw.data(), sizeof(float2) * L, cudaMemcpyHostToDevice);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(filter tables)");
        }
    }
    const long total = n_views * (long)n_rows;
    if (total == 0) return IFDK_OK;
    const int L = 1 << g->log2L;
    const size_t smem = 2 * sizeof(float2) * (size_t)L;
    e = cudaFuncSetAttribute(filter_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(filter)");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, filter_fft_kernel, kThreads, smem);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (per_sm < 1) return fail(IFDK_ERR_SHAPE, "Nu too large for the shared-memory FFT");
    const long pairs = (total + 1) / 2;
    long grid = (long)sms * per_sm;
    if (grid > pairs) grid = pairs;
    FilterParams p;
    p.raw = raw;
    p.out = out;
    p.n_rows_total = total;
    p.n_rows = n_rows;
    p.v0 = v0;
    p.Nu = g->Nu;
    p.D = (float)g->D;
    p.D2 = (float)(g->D * g->D);
    p.Du = (float)g->Du;
    p.Dv = (float)g->Dv;
    p.cu = (float)g->cu;
    p.cv = (float)g->cv;
    filter_fft_kernel<<<(unsigned)grid, kThreads, smem, st>>>(p, g->dev[dev].tw, g->dev[dev].Hs,
                                                              g->log2L);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "filter_fft_kernel launch");
    count_launch();
    return IFDK_OK;
}

}  // namespace ifdk
