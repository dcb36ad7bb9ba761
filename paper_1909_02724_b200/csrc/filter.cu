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
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "ifdk_internal.h"
#include "mbar.cuh"

namespace ifdk {
namespace {

constexpr int kThreads = 256;

struct FilterParams {
    const float* raw;
    float* out;         // [n_views][n_rows][Nu] (n_dest == 0)
    long n_rows_total;  // n_views * n_rows
    int n_rows;         // rows per view
    int v0;             // first detector row of each view
    int Nu;
    float D2, D, Du, Dv, cu, cv;
    // Band scatter (n_dest > 0): row v of view t goes to every destination d with
    // lo[d] <= v <= hi[d], at base[d] + (t (hi[d]-lo[d]+1) + v - lo[d]) Nu -- local or
    // peer-mapped (NVLink) memory, so the exchange of the k-slab split rides the filter.
    int n_dest;
    float* base[kMaxFilterDest];
    int lo[kMaxFilterDest], hi[kMaxFilterDest];
    // Completion signal of the fused exchange (flags.n > 0; peer.cu): after its stores every
    // thread fences at system scope, and the CTA that takes the last ticket increments the
    // flags -- the destinations' consumers wait on them.
    PeerFlags flags;
};

// The "last block" pattern at system scope (CUDA C++ Programming Guide, Memory Fence
// Functions): every row this launch stored is visible to the peers before any flag moves.
__device__ __forceinline__ void signal_done(const FilterParams& p)
{
    if (p.flags.n == 0) return;
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned ticket = atomicAdd(p.flags.ticket, 1u);
        if (ticket == gridDim.x - 1) {
            __threadfence_system();
            for (int f = 0; f < p.flags.n; ++f) atomicAdd_system(p.flags.flag[f], 1u);
            atomicExch(p.flags.ticket, 0u);  // ready for the next launch on the stream
        }
    }
}

// Output row r (= t n_rows + (v - v0)) of destination d, or nullptr if v is outside its band.
__device__ __forceinline__ float* dest_row(const FilterParams& p, long r, int d)
{
    const long t = r / p.n_rows;
    const int v = p.v0 + (int)(r - t * p.n_rows);
    if (v < p.lo[d] || v > p.hi[d]) return nullptr;
    return p.base[d] + (t * (p.hi[d] - p.lo[d] + 1) + (v - p.lo[d])) * (long)p.Nu;
}

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
                const float wA = 1.0f / sqrtf(p.D2 + uh2 + vhA * vhA);  // D is in H
                x.x = __ldg(eA + m) * wA;
                if (hasB) {
                    const float wB = 1.0f / sqrtf(p.D2 + uh2 + vhB * vhB);
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
        const int nd = p.n_dest > 0 ? p.n_dest : 1;
        for (int d = 0; d < nd; ++d) {
            float* qA = p.n_dest > 0 ? dest_row(p, rA, d) : p.out + rA * p.Nu;
            float* qB = !hasB ? nullptr : p.n_dest > 0 ? dest_row(p, rB, d) : p.out + rB * p.Nu;
            for (int n = threadIdx.x; n < p.Nu; n += kThreads) {
                const float2 z = Z[n];
                if (qA) qA[n] = z.x;
                if (qB) qB[n] = -z.y;
            }
        }
        __syncthreads();
    }
    signal_done(p);
}


// ----------------------------------------------------------------------------------------
// Length-4096 FFT filter (Nu <= 2048): 256 threads, 16 complex values per thread, three
// radix-16 Stockham passes (span 1, 16, 256) with the 16-point DFT in registers (4 x 4) and
// two shared-memory exchanges per transform.  Pass 1 reads the rows straight from HBM (the
// upper half of the padded signal is zero), the last forward pass leaves thread i holding
// X[i + 256 m], which is exactly the input the inverse's first pass needs, so the filter
// multiply and the conj of the inverse happen in registers; the inverse's last pass leaves
// Z[i + 256 m] and the first Nu samples go straight back to HBM.
namespace f4k {

constexpr int L = 4096, T = 256;


// Complex values ride in one 64-bit register pair (re, im) and every butterfly is a Blackwell
// packed fp32x2 instruction: a complex add is one FADD2, a multiplication by -i is free (the
// consumer's operand takes the halves swapped and one negated, .LO_HI / .N modifiers), a
// complex multiply is FMUL2 + FFMA2 with broadcast operands -- half the FP32 instructions of
// the scalar butterflies.
using cx = unsigned long long;

__device__ __forceinline__ cx mk(float re, float im)
{
    cx r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(re), "f"(im));
    return r;
}
__device__ __forceinline__ float re_(cx v)
{
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return a;
}
__device__ __forceinline__ float im_(cx v)
{
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
    return b;
}
__device__ __forceinline__ cx cadd(cx a, cx b)
{
    cx r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cx csub(cx a, cx b)
{
    cx r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cx cmul2(cx a, cx b)  // element-wise
{
    cx r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ cx cfma2(cx a, cx b, cx c)  // element-wise a b + c
{
    cx r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ cx negi(cx v) { return mk(im_(v), -re_(v)); }  // -i v

// a b = b.re (a.re, a.im) + b.im (-a.im, a.re): the swapped, half-negated operand i a sits in
// the first source slot, where ptxas folds it into a .LO_HI.NP operand modifier, and b's halves
// are register broadcasts -- one FMUL2 + one FFMA2, no moves (the form with i b in the second
// slot cost a MOV and an FADD per product).
__device__ __forceinline__ cx ia(cx v) { return mk(-im_(v), re_(v)); }  // i v
__device__ __forceinline__ cx cmulf(cx a, cx b)
{
    const float br = re_(b), bi = im_(b);
    return cfma2(ia(a), mk(bi, bi), cmul2(a, mk(br, br)));
}
__device__ __forceinline__ float rsqrt_ftz(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// a (c + i s) for compile-time c, s: FMUL2 / FFMA2 with broadcast immediates
__device__ __forceinline__ cx cmulk(cx a, float c, float s)
{
    return cfma2(ia(a), mk(s, s), cmul2(a, mk(c, c)));
}

__device__ __forceinline__ void dft4(cx& a, cx& b, cx& c, cx& d)
{
    const cx t0 = cadd(a, c), t1 = csub(a, c);
    const cx t2 = cadd(b, d);
    const cx t3 = negi(csub(b, d));  // -i (b - d)
    a = cadd(t0, t2);
    c = csub(t0, t2);
    b = cadd(t1, t3);
    d = csub(t1, t3);
}

// dft4 of (a, b, 0, 0): the zero-padded upper half of a row costs no additions
__device__ __forceinline__ void dft4_half(cx& a, cx& b, cx& c, cx& d)
{
    const cx t3 = negi(b);  // -i b
    c = csub(a, b);
    d = csub(a, t3);
    const cx a0 = a;
    a = cadd(a0, b);
    b = cadd(a0, t3);
}

// 16-point forward DFT in place: n = 4 n1 + n2, k = k1 + 4 k2 (two radix-4 stages).
// HALF: u[8..15] are zero (the first pass of a zero-padded row).
template <bool HALF = false>
__device__ __forceinline__ void dft16(cx (&u)[16])
{
    constexpr float C1 = 0.92387953251128674f, S1 = 0.38268343236508977f,
                    C2 = 0.70710678118654752f;
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
        if (HALF)
            dft4_half(u[n2], u[4 + n2], u[8 + n2], u[12 + n2]);
        else
            dft4(u[n2], u[4 + n2], u[8 + n2], u[12 + n2]);
    }
    // A[n2][k1] (at u[4 k1 + n2]) *= W16^(n2 k1)
    u[5] = cmulk(u[5], C1, -S1);    // W^1
    u[6] = cmulk(u[6], C2, -C2);    // W^2
    u[7] = cmulk(u[7], S1, -C1);    // W^3
    u[9] = cmulk(u[9], C2, -C2);    // W^2
    u[10] = negi(u[10]);            // W^4 = -i
    u[11] = cmulk(u[11], -C2, -C2); // W^6
    u[13] = cmulk(u[13], S1, -C1);  // W^3
    u[14] = cmulk(u[14], -C2, -C2); // W^6
    u[15] = cmulk(u[15], -C1, S1);  // W^9
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) dft4(u[4 * k1], u[4 * k1 + 1], u[4 * k1 + 2], u[4 * k1 + 3]);
    // X[k1 + 4 k2] sits at u[4 k1 + k2]: transpose by renaming
    cx v[16];
#pragma unroll
    for (int m = 0; m < 16; ++m) v[m] = u[4 * (m & 3) + (m >> 2)];
#pragma unroll
    for (int m = 0; m < 16; ++m) u[m] = v[m];
}

// Per-thread twiddles in tensor memory.  Thread i's span-16 pass multiplies u[j] by w^(16 j k)
// (k = i mod 16) and its span-256 pass by w^(j i), j = 1..15, w = e^(-2 pi i / 4096): the same
// 2 x 15 complex values for every row group the (persistent) thread transforms.  They are read
// once per launch from the host's table of w^e (fp64, rounded once) and kept in the CTA's
// tensor memory -- 128 columns; warp w owns lanes 32 (w mod 4) .. +31 and columns 64 (w / 4)
// .. +63: columns 0..29 hold the span-16 set, 32..61 the span-256 set -- so a twiddled pass
// costs one tcgen05.ld of 32 registers (issued before the exchange's shared loads, awaited
// after them) and 15 complex multiplies.  (Round 2's first form read four power tables per
// pass and composed the other eleven powers: 22 % of the kernel's instructions, r2x capture.)
__device__ __forceinline__ void tm_ld16(uint32_t taddr, cx* w)  // w[0..7] = columns 0..15
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
          "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int m = 0; m < 8; ++m) w[m] = mk(__uint_as_float(r[2 * m]), __uint_as_float(r[2 * m + 1]));
}
// Two 16-column loads rather than one of 32: a 32-register destination block made ptxas move
// the live transform values out of its way (about 30 moves per row group, r2z6 capture).
__device__ __forceinline__ void tm_ld32(uint32_t taddr, cx (&w)[16])
{
    tm_ld16(taddr, w);
    tm_ld16(taddr + 16, w + 8);
}

__device__ __forceinline__ void tm_st32(uint32_t taddr, const cx (&w)[16])
{
    float r[32];
#pragma unroll
    for (int m = 0; m < 16; ++m) {
        r[2 * m] = re_(w[m]);
        r[2 * m + 1] = im_(w[m]);
    }
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31, %32};" ::"r"(taddr),
        "f"(r[0]), "f"(r[1]), "f"(r[2]), "f"(r[3]), "f"(r[4]), "f"(r[5]), "f"(r[6]), "f"(r[7]),
        "f"(r[8]), "f"(r[9]), "f"(r[10]), "f"(r[11]), "f"(r[12]), "f"(r[13]), "f"(r[14]),
        "f"(r[15]), "f"(r[16]), "f"(r[17]), "f"(r[18]), "f"(r[19]), "f"(r[20]), "f"(r[21]),
        "f"(r[22]), "f"(r[23]), "f"(r[24]), "f"(r[25]), "f"(r[26]), "f"(r[27]), "f"(r[28]),
        "f"(r[29]), "f"(r[30]), "f"(r[31]));
}

__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ void apply_twiddles(cx (&u)[16], const cx (&w)[16])
{
#pragma unroll
    for (int j = 1; j < 16; ++j) u[j] = cmulf(u[j], w[j - 1]);
}

// The length-4096 transform as 16 x 256 (n = n1 + 256 n2, k = k1 + 16 k2; thread i, half-warp
// h = i / 16, lane l = i mod 16):
//   X[k1 + 16 k2] = sum_n1 w256^(n1 k2) w^(n1 k1) [sum_n2 w16^(n2 k1) x[n1 + 256 n2]].
// S1: thread i = n1 takes the 16-point DFT over n2 of x[i + 256 n2] (its own registers) and the
// twiddles w^(i k1).  One CTA exchange (the buffer A: 16 rows k1 of 272 slots) hands row k1 to
// half-warp h = k1, lane l taking n1 = l + 16 b.  S3: the 256-point DFT of each row inside its
// half-warp, itself 16 x 16 -- a DFT over b, the twiddles w256^(l c) = w^(16 l c), a warp-local
// exchange through the half-warp's own row of A (slot 17 c + l, padded) and a DFT over l --
// leaves lane l = c holding X[h + 16 l + 256 d], d = 0..15.  The inverse is the same algorithm
// run backwards (the transpose of a DFT is itself, every stage is a block of symmetric DFT16s or
// a diagonal of twiddles), so it uses the same two twiddle sets and starts from exactly that
// spectral distribution and ends with thread i holding z[i + 256 n2] -- the input layout -- with
// the conj trick IDFT(Y) = conj(DFT(conj Y)).  Per transform: one CTA barrier and one warp
// barrier (Round 2's Stockham form needed two CTA exchanges and two buffers); the row of A a
// half-warp uses for its warp exchange is the row only it reads, so one 34 KB buffer serves
// both exchanges of both transforms, and three CTAs fit on an SM.  Bank conflicts: none (the
// CTA exchange moves consecutive slots per half-warp, the warp exchange has stride 17).
constexpr int kRow = 272;        // slots per row of A (256 + the 16 x 17 warp exchange)
constexpr int kXBuf = 16 * kRow;  // complex slots of A

// S1 + twiddles + the write of the CTA exchange.  HALF: x[i + 256 j] = 0 for j >= 8.
template <bool HALF>
__device__ __forceinline__ void fwd_s1(cx (&u)[16], cx* A, uint32_t tw, int i)
{
    dft16<HALF>(u);
    cx w[16];
    tm_ld32(tw + 32, w);  // w^(j i)
    tm_wait_ld();
    apply_twiddles(u, w);
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) A[k1 * kRow + i] = u[k1];
}

// After the CTA barrier: S3 on row h.  Returns X[h + 16 l + 256 d] in u[d].
__device__ __forceinline__ void fwd_s3(cx (&u)[16], cx* A, uint32_t tw, int i)
{
    const int h = i >> 4, l = i & 15;
    cx* const row = A + h * kRow;
#pragma unroll
    for (int b = 0; b < 16; ++b) u[b] = row[l + 16 * b];
    dft16(u);  // over b -> c
    {
        cx w[16];
        tm_ld32(tw, w);  // w^(16 l j)
        tm_wait_ld();
        apply_twiddles(u, w);
    }
    __syncwarp();  // the half-warp's reads of its row are done
#pragma unroll
    for (int c = 0; c < 16; ++c) row[17 * c + l] = u[c];
    __syncwarp();
#pragma unroll
    for (int ll = 0; ll < 16; ++ll) u[ll] = row[17 * l + ll];
    dft16(u);  // over l -> d
}

// The inverse's S3 backwards from the spectral distribution, then the write of its CTA
// exchange (row h, n1 = l + 16 b).
__device__ __forceinline__ void inv_s3(cx (&u)[16], cx* A, uint32_t tw, int i)
{
    const int h = i >> 4, l = i & 15;
    cx* const row = A + h * kRow;
    dft16(u);  // over d -> l'
    {
        cx w[16];
        tm_ld32(tw, w);  // w^(16 l j)
        tm_wait_ld();
        apply_twiddles(u, w);
    }
    __syncwarp();  // the forward's warp-exchange reads of this row are done
#pragma unroll
    for (int ll = 0; ll < 16; ++ll) row[17 * l + ll] = u[ll];
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 16; ++c) u[c] = row[17 * c + l];
    dft16(u);  // over c -> b
    __syncwarp();  // the warp-exchange reads of this row are done
#pragma unroll
    for (int b = 0; b < 16; ++b) row[l + 16 * b] = u[b];
}

// After the CTA barrier: thread i = n1 gathers its 16 k1 values, twiddles, DFT over k1.
// Returns z[i + 256 n2] in u[n2] (before the final conj).
__device__ __forceinline__ void inv_s1(cx (&u)[16], const cx* A, uint32_t tw, int i)
{
    cx w[16];
    tm_ld32(tw + 32, w);  // w^(j i)
#pragma unroll
    for (int k1 = 0; k1 < 16; ++k1) u[k1] = A[k1 * kRow + i];
    tm_wait_ld();
    apply_twiddles(u, w);
    dft16(u);
}

}  // namespace f4k

// ASYNC (rows 16-byte aligned, Nu % 4 == 0): the next group's rows are fetched into a shared
// staging buffer by 1-D bulk copies (the TMA engine; one instruction per row, completion on an
// mbarrier) while the current group is transformed, hiding HBM latency.  The staging slots are
// zeroed once per launch: a copy writes the first N_u floats of a slot, so the padding after
// them stays zero and the rows are read without masks.
constexpr int kF4kStage = 2048;  // floats per staged row (Nu <= 2048)
constexpr size_t kF4kSmem = sizeof(float2) * f4k::kXBuf + sizeof(float) * 4096 +
                            sizeof(float) * 2 * kF4kStage + 16;

// Destination row of view t, detector row v in band d, or nullptr if v is outside the band.
__device__ __forceinline__ float* dest_row_tv(const FilterParams& p, long t, int v, int d)
{
    if (v < p.lo[d] || v > p.hi[d]) return nullptr;
    return p.base[d] + (t * (p.hi[d] - p.lo[d] + 1) + (v - p.lo[d])) * (long)p.Nu;
}

// R row pairs per transform (multi-row packing): with N_u <= 2048 / R every row's linear
// convolution needs only a 2 N_u - 1 window of the length-4096 circular one, so R rows share
// the real part (and R the imaginary part) in slots of S = 4096 / R samples: the ramp's
// support (|n - m| <= N_u - 1) never reaches from one slot into another (S - N_u >= N_u - 1),
// and each slot's first N_u outputs are exactly that row's linear convolution.  Configs 2 / 3
// (N_u = 512 / 1024) run 4 / 2 row pairs per transform.
template <bool ASYNC, int R>
__global__ void __launch_bounds__(256, 3) filter_f4k_kernel(const FilterParams p,
                                                            const float2* __restrict__ tw_g,
                                                            const float* __restrict__ Hs_g)
{
    using namespace f4k;
    constexpr int SJ = 16 / R;          // values j of a thread per slot (slot = S / 256 j's)
    constexpr int ROWS = 2 * R;         // rows per transform
    constexpr int SLOT_F = 4096 / ROWS; // staged floats per row (>= N_u)
    extern __shared__ __align__(16) unsigned char fsm[];
    cx* const A = reinterpret_cast<cx*>(fsm);                  // the exchange buffer
    float* const Hp = reinterpret_cast<float*>(A + kXBuf);      // H in spectral order
    float* const stage = Hp + 4096;                             // ROWS rows of SLOT_F
    uint64_t* const sbar = reinterpret_cast<uint64_t*>(stage + 2 * kF4kStage);  // staging barrier
    uint32_t* const tslot = reinterpret_cast<uint32_t*>(sbar + 1);             // TMEM address
    const int i = threadIdx.x, warp = i >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                         smem_u32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    // Hp[256 d + i'] = H[f], f = h' + 16 l' + 256 d (h' = i' / 16, l' = i' mod 16): the
    // frequency thread i' holds in u[d] after the forward transform (H real and even:
    // H[f] = H[L - f] past L / 2), read without bank conflicts.
    for (int e = i; e < L; e += T) {
        const int ii = e & 255, f = (ii >> 4) + 16 * (ii & 15) + (e & ~255);
        Hp[e] = Hs_g[f <= L / 2 ? f : L - f];
    }
    if (ASYNC)
        for (int e = i; e < 2 * kF4kStage; e += T) stage[e] = 0.f;
    const long n_groups = (p.n_rows_total + ROWS - 1) / ROWS;
    if (ASYNC && i == 0) {
        mbar_init(sbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmw = *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    {
        const cx* twc = reinterpret_cast<const cx*>(tw_g);  // w^e, e = 0 .. 4095
        cx w[16];
        w[15] = 0ull;
#pragma unroll
        for (int j = 1; j < 16; ++j) w[j - 1] = twc[(16 * j * (i & 15)) & 4095];
        tm_st32(tmw, w);
#pragma unroll
        for (int j = 1; j < 16; ++j) w[j - 1] = twc[(j * i) & 4095];
        tm_st32(tmw + 32, w);
        tm_wait_st();
    }
    auto prefetch = [&](long gi) {  // one thread: the group's rows by 1-D bulk copies
        if (!ASYNC || i != 0 || gi >= n_groups) return;
        const long r0 = ROWS * gi;
        const int nrow = (int)min((long)ROWS, p.n_rows_total - r0);
        // a partial last group: the missing rows' slots are zeroed (they share the transforms)
        for (int r = nrow; r < ROWS; ++r)
            for (int n = 0; n < SLOT_F; ++n) stage[r * SLOT_F + n] = 0.f;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // after the generic accesses
        mbar_expect_tx(sbar, (uint32_t)(nrow * p.Nu * 4));
        for (int r = 0; r < nrow; ++r)
            bulk_load(stage + r * SLOT_F, p.raw + (r0 + r) * p.Nu, (uint32_t)(p.Nu * 4), sbar);
    };
    prefetch(blockIdx.x);
    // (view, detector row) of the group's first row, stepped without a division per group
    const int nr = p.n_rows;
    const long stepR = (long)ROWS * gridDim.x;
    const long sq = stepR / nr;
    const int sr = (int)(stepR - sq * nr);
    long t0 = (long)ROWS * blockIdx.x / nr;
    int vr0 = (int)((long)ROWS * blockIdx.x - t0 * nr);
    uint32_t sphase = 0;
    const float uh0 = ((float)i - p.cu) * p.Du;  // uh of sample n = i + 256 jj: uh0 + 256 jj Du
    for (long gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
        const long r0 = ROWS * gi;
        // D^2 + vh^2 of rows A = r0 + 2 s (real part) and B = r0 + 2 s + 1 (imaginary part)
        float dA[R], dB[R];
#pragma unroll
        for (int sl = 0; sl < R; ++sl) {
            int vA = vr0 + 2 * sl, vB = vA + 1;
            while (vA >= nr) vA -= nr;
            while (vB >= nr) vB -= nr;
            const float vhA = ((float)(p.v0 + vA) - p.cv) * p.Dv;
            const float vhB = ((float)(p.v0 + vB) - p.cv) * p.Dv;
            dA[sl] = p.D2 + vhA * vhA;
            dB[sl] = p.D2 + vhB * vhB;
        }
        if (ASYNC) {
            mbar_wait(sbar, sphase);
            sphase ^= 1u;
        }
        cx u[16];
        // Alg. alg:filter line 2: E~ = E . F_cos (reading c-A5), rows packed per slot, padded.
        // F_cos = D / sqrt(D^2 + uh^2 + vh^2); D is folded into the filter spectrum H (the
        // filter is linear), the rows' pair (A, B) shares one FFMA2 and one FMUL2, and the
        // reciprocal square root is the hardware approximation (<= 2 ulp; the argument is
        // >= D^2, never denormal) -- far below the filter tolerance.
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            const int sl = j / SJ, jj = j % SJ;
            if (jj >= SJ / 2) {  // n >= S / 2 >= N_u: the zero padding of the slot
                u[j] = 0ull;
                continue;
            }
            const int n = i + jj * T;
            float ea = 0.f, eb = 0.f;
            if (ASYNC) {
                ea = stage[(2 * sl) * SLOT_F + n];
                eb = stage[(2 * sl + 1) * SLOT_F + n];
            } else {
                const long rA = r0 + 2 * sl, rB = rA + 1;
                if (n < p.Nu && rA < p.n_rows_total) {
                    ea = __ldg(p.raw + rA * p.Nu + n);
                    if (rB < p.n_rows_total) eb = __ldg(p.raw + rB * p.Nu + n);
                }
            }
            const float uh = fmaf((float)(jj * T), p.Du, uh0);
            const cx q = cfma2(mk(uh, uh), mk(uh, uh), mk(dA[sl], dB[sl]));
            u[j] = cmul2(mk(ea, eb), mk(rsqrt_ftz(re_(q)), rsqrt_ftz(im_(q))));
        }
        fwd_s1<R == 1>(u, A, tmw, i);
        __syncthreads();  // exchange written, staging read out: fetch the next group meanwhile
        prefetch(gi + gridDim.x);
        fwd_s3(u, A, tmw, i);
        // Y = X . H (real, even; C/L folded in), and the inverse by the forward transform:
        // DFT(i conj(Y)) = i conj(L z) = (im L z, re L z) -- multiplying conj(Y) by i swaps the
        // halves (free, a .LO_HI operand), and the transform then returns row B's samples in
        // the real halves and row A's in the imaginary ones, with no negation left anywhere.
#pragma unroll
        for (int d = 0; d < 16; ++d) {
            const float h = Hp[256 * d + i];
            u[d] = cmul2(mk(im_(u[d]), re_(u[d])), mk(h, h));
        }
        inv_s3(u, A, tmw, i);
        __syncthreads();
        inv_s1(u, A, tmw, i);
        // Q: imaginary halves -> row A, real halves -> row B of each slot, samples 0..Nu-1 (to every
        // destination band that holds the row when scattering).
        if (p.n_dest == 0 && p.Nu == SLOT_F && r0 + ROWS <= p.n_rows_total) {
            // whole group of full-width rows (configs 2-4): row stride SLOT_F, no masks
            float* const q0 = p.out + r0 * SLOT_F + i;
#pragma unroll
            for (int sl = 0; sl < R; ++sl)
#pragma unroll
                for (int jj = 0; jj < SJ / 2; ++jj) {
                    q0[(2 * sl) * SLOT_F + jj * T] = im_(u[sl * SJ + jj]);
                    q0[(2 * sl + 1) * SLOT_F + jj * T] = re_(u[sl * SJ + jj]);
                }
        } else if (p.n_dest == 0) {
#pragma unroll
            for (int sl = 0; sl < R; ++sl) {
                const long rA = r0 + 2 * sl;
                if (rA >= p.n_rows_total) break;
                const bool hasB = rA + 1 < p.n_rows_total;
                float* const qA = p.out + rA * p.Nu;
                float* const qB = qA + p.Nu;
#pragma unroll
                for (int jj = 0; jj < SJ / 2; ++jj) {
                    const int n = i + jj * T;
                    if (n < p.Nu) {
                        qA[n] = im_(u[sl * SJ + jj]);
                        if (hasB) qB[n] = re_(u[sl * SJ + jj]);
                    }
                }
            }
        } else {
            for (int d = 0; d < p.n_dest; ++d) {
#pragma unroll
                for (int sl = 0; sl < R; ++sl) {
                    const long rA = r0 + 2 * sl, rB = rA + 1;
                    if (rA >= p.n_rows_total) break;
                    int vA = vr0 + 2 * sl, vB = vA + 1;
                    long tA = t0, tB = t0;
                    while (vA >= nr) { vA -= nr; ++tA; }
                    while (vB >= nr) { vB -= nr; ++tB; }
                    float* qA = dest_row_tv(p, tA, p.v0 + vA, d);
                    float* qB = rB < p.n_rows_total ? dest_row_tv(p, tB, p.v0 + vB, d) : nullptr;
#pragma unroll
                    for (int jj = 0; jj < SJ / 2; ++jj) {
                        const int n = i + jj * T;
                        if (n < p.Nu) {
                            if (qA) qA[n] = im_(u[sl * SJ + jj]);
                            if (qB) qB[n] = re_(u[sl * SJ + jj]);
                        }
                    }
                }
            }
        }
        t0 += sq;
        vr0 += sr;
        if (vr0 >= nr) {
            vr0 -= nr;
            ++t0;
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tslot)
                     : "memory");
    signal_done(p);
}

}  // namespace

void preload_filter_kernels()  // see preload_bp_kernels (backproject.cu)
{
    cudaFuncAttributes a;
    const void* ks[] = {
        reinterpret_cast<const void*>(filter_fft_kernel),
        reinterpret_cast<const void*>(filter_f4k_kernel<true, 1>),
        reinterpret_cast<const void*>(filter_f4k_kernel<false, 1>),
        reinterpret_cast<const void*>(filter_f4k_kernel<true, 2>),
        reinterpret_cast<const void*>(filter_f4k_kernel<false, 2>),
        reinterpret_cast<const void*>(filter_f4k_kernel<true, 4>),
        reinterpret_cast<const void*>(filter_f4k_kernel<false, 4>),
        reinterpret_cast<const void*>(filter_f4k_kernel<true, 8>),
        reinterpret_cast<const void*>(filter_f4k_kernel<false, 8>)};
    for (const void* k : ks)
        if (cudaFuncGetAttributes(&a, k) != cudaSuccess) cudaGetLastError();
}

ifdk_status launch_filter(ifdk_geometry* g, const float* raw, float* out, long n_views, int v0,
                          int n_rows, cudaStream_t st, int n_dest, const ifdk_band_dest* dests,
                          const PeerFlags* flags)
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
    if (total == 0) return flags ? launch_signal(*flags, st) : IFDK_OK;
    const int L = 1 << g->log2L;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
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
    p.n_dest = n_dest;
    for (int d = 0; d < kMaxFilterDest; ++d) {
        p.base[d] = d < n_dest ? dests[d].base : nullptr;
        p.lo[d] = d < n_dest ? dests[d].v_lo : 0;
        p.hi[d] = d < n_dest ? dests[d].v_hi : -1;
    }
    if (flags) p.flags = *flags;
    const long pairs = (total + 1) / 2;
    if (L == 4096) {
        // row pairs per transform: the largest R <= 8 whose slot 4096 / R holds a full-length
        // linear convolution of an N_u-sample row (4096 / R >= 2 N_u - 1)
        int R = 1;
        while (R < 8 && 4096 / (2 * R) >= 2 * g->Nu - 1) R *= 2;
        const long groups = (total + 2 * R - 1) / (2 * R);
        // In-place filtering is safe with the prefetch: a group's rows are fetched before any
        // CTA writes them (each group belongs to one CTA) and never read again.  (A scatter
        // destination must not alias the raw views.)
        const bool async = (g->Nu % 4) == 0 && (reinterpret_cast<uintptr_t>(raw) % 16) == 0;
        auto pick = [&](auto ka, auto ks) { return async ? ka : ks; };
        void (*k)(const FilterParams, const float2*, const float*) =
            R == 8   ? pick(filter_f4k_kernel<true, 8>, filter_f4k_kernel<false, 8>)
            : R == 4 ? pick(filter_f4k_kernel<true, 4>, filter_f4k_kernel<false, 4>)
            : R == 2 ? pick(filter_f4k_kernel<true, 2>, filter_f4k_kernel<false, 2>)
                     : pick(filter_f4k_kernel<true, 1>, filter_f4k_kernel<false, 1>);
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4kSmem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(filter)");
        // persistent grid: the CTAs that fit on an SM by registers and shared memory (3 for the
        // 68 KB, <= 80-register kernel; 128 tensor-memory columns each, at most 4 per SM).
        // (cudaOccupancyMaxActiveBlocksPerMultiprocessor answered 1 for this kernel.)
        e = cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(filter carveout)");
        cudaFuncAttributes fa;
        if ((e = cudaFuncGetAttributes(&fa, k)) != cudaSuccess)
            return cuda_fail(e, "cudaFuncGetAttributes(filter)");
        int sm_smem = 0, reserved = 0;
        cudaDeviceGetAttribute(&sm_smem, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev);
        cudaDeviceGetAttribute(&reserved, cudaDevAttrReservedSharedMemoryPerBlock, dev);
        const int regs = (fa.numRegs + 7) / 8 * 8;
        int per_sm = 4;
        per_sm = std::min(per_sm, 65536 / (regs * 256));
        per_sm = std::min(per_sm, sm_smem / (int)(kF4kSmem + reserved));
        long grid = (long)sms * (per_sm > 0 ? per_sm : 1);
        if (grid > groups) grid = groups;
        k<<<(unsigned)grid, 256, kF4kSmem, st>>>(p, g->dev[dev].tw, g->dev[dev].Hs);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "filter_f4k_kernel launch");
        count_launch();
        return IFDK_OK;
    }
    const size_t smem = 2 * sizeof(float2) * (size_t)L;
    e = cudaFuncSetAttribute(filter_fft_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(filter)");
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, filter_fft_kernel, kThreads, smem);
    if (per_sm < 1) return fail(IFDK_ERR_SHAPE, "Nu too large for the shared-memory FFT");
    long grid = (long)sms * per_sm;
    if (grid > pairs) grid = pairs;
    filter_fft_kernel<<<(unsigned)grid, kThreads, smem, st>>>(p, g->dev[dev].tw, g->dev[dev].Hs,
                                                              g->log2L);
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "filter_fft_kernel launch");
    count_launch();
    return IFDK_OK;
}

}  // namespace ifdk
