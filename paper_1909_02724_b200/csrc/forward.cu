// forward.cu -- the matched forward projector: the exact transpose of BP-sm100 (Alg. alg:bp
// P:402-430 with Alg. alg:subpixel P:431-447), for iterative reconstruction (SART / SIRT,
// P:266).
//
// Back-projection is V(i,j,k) = sum_s W_s(i,j) sum_taps w_tap(u, v) Q_s[tap], i.e. V = M^T Q
// with M_s[(v,u),(i,j,k)] = W_s(i,j) w_tap.  Its transpose splats each voxel into the four
// bilinear taps of its projection:  F_s[tap] = sum_{i,j,k} W_s(i,j) w_tap(u,v) x(i,j,k)
// (reading c-I1 in DESIGN.md), taps off the detector dropped (the zero border, c-A9).
//
// Mapping (the BP kernel's, run backwards): a CTA of 256 threads owns a 16 x 16 column tile
// and a KC-slice chunk; each thread keeps its column's KC voxel values in registers for the
// whole launch, computes z, u, W and the base of v in fp64 per view (Theorems 2-3, the same
// kwalk.cuh code as BP), walks k in fp32 and adds W x w_tap into a shared-memory patch of the
// detector with shared-memory atomics.  After each view the CTA adds the non-zero part of its
// patch to the projection in global memory (red.global.add.f32).  The patch is double
// buffered: the flush of view t and the zeroing for view t+2 overlap the splat of view t+1.
// Summation order is that of the atomics, so the result is not bitwise reproducible (fp32
// rounding differences only).
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include "ifdk_internal.h"
#include "kwalk.cuh"

namespace ifdk {
namespace {

constexpr int kTI = 16, kTJ = 16, kThreads = 256, kKC = 32;

struct FPParams {
    const float* vol;  // slab [nk][Ny][Nx]
    float* proj;       // band [n_views][n_rows][Nu]
    int n_views;
    int Nu, Nv, Nx, Ny;
    int v0, n_rows;
    int k0, nk;
    int kb0;           // global k of chunk 0 (multiple of kKC)
    int tiles_i, raster;
    int box_w, box_h;  // patch capacity (columns, rows)
    float qfactor;     // bound on a patch pixel's sum per unit |x|: 256 (1/dv_min + 1) / zmin^2
};

__device__ __forceinline__ uint32_t smem_u32_fp(const void* q)
{
    return static_cast<uint32_t>(__cvta_generic_to_shared(q));
}

// shared-memory integer add, predicated in the instruction (no branch around it)
__device__ __forceinline__ void red_add_if(uint32_t addr, int v, uint32_t pred)
{
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.u32 p, %2, 0;\n @p red.shared.add.s32 [%0], %1;\n}" ::"r"(addr),
        "r"(v), "r"(pred)
        : "memory");
}

struct __align__(16) Box {
    int u_org, v_org, w, h;
    // the tile corner's invariants (fp64, split) and P_s in fp32: each thread adds its offset
    // from the corner in fp32 (backproject.cu quad_inv, reading c-N2)
    int uci, vci;
    float ucf, vcf;
    float uc, vc, zc, p0;
    float p1, p3, p4, p5;
    float p7, p8, pad0, pad1;
};

__device__ __forceinline__ float rcp_approx_fp(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// Per-(column, view) invariants from the corner values: u = u_c + (dx - u_c dz) / z (fp32
// offsets dx, dz of the column from the corner, < 16 voxels), the same for v(kb).
__device__ __forceinline__ ThreadInv corner_inv(const Box& m, float fdi, float fdj)
{
    ThreadInv t;
    const float dx = fmaf(m.p0, fdi, m.p1 * fdj);
    const float dy = fmaf(m.p3, fdi, m.p4 * fdj);
    const float dz = fmaf(m.p7, fdi, m.p8 * fdj);
    const float f = rcp_approx_fp(m.zc + dz);
    const float su = fmaf(fmaf(-m.uc, dz, dx), f, m.ucf);
    const float sv = fmaf(fmaf(-m.vc, dz, dy), f, m.vcf);
    const float tu = __fadd_rd(su, 12582912.0f), tv = __fadd_rd(sv, 12582912.0f);
    t.nu = m.uci + (int)(__float_as_uint(tu) - 0x4B400000u);
    t.nv = m.vci + (int)(__float_as_uint(tv) - 0x4B400000u);
    t.du = su - (tu - 12582912.0f);
    t.fv0 = sv - (tv - 12582912.0f);
    t.dv = m.p5 * f;
    t.dvm1 = t.dv - 1.f;
    t.W = f * f;
    t.dvi = 0;  // unused by the projector's walks
    t.dvf = t.dv;
    return t;
}
constexpr int kBoxRing = 16;

template <bool SMALL_DV>
__global__ void __launch_bounds__(kThreads, 2)
    fp_kernel(const __grid_constant__ FPParams p, const __grid_constant__ PTable pt)
{
    extern __shared__ __align__(16) float fsm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile_i = (int)blockIdx.z * p.raster + (int)(blockIdx.x % (unsigned)p.raster);
    const int tile_j = (int)(blockIdx.x / (unsigned)p.raster);
    if (tile_i >= p.tiles_i) return;
    // A warp's 32 columns are spread over the tile (stride 2 in i, 4 in j), not packed 8 x 4:
    // neighbouring columns project onto the same detector pixel whenever the ray runs between
    // them, and same-pixel lanes serialise a shared atomic; spread lanes collide only when the
    // ray is within a narrow angle of their separation.
    const int i = tile_i * kTI + (lane & 7) * 2 + (warp & 1);
    const int j = tile_j * kTJ + (lane >> 3) * 4 + (warp >> 1);
    const bool active = i < p.Nx && j < p.Ny;
    const float fdi = (float)(min(i, p.Nx - 1) - tile_i * kTI);
    const float fdj = (float)(min(j, p.Ny - 1) - tile_j * kTJ);
    const double di = (double)min(i, p.Nx - 1), dj = (double)min(j, p.Ny - 1);
    const int kb = p.kb0 + (int)blockIdx.y * kKC;
    const int kv0 = max(p.k0 - kb, 0), kv1 = min(p.k0 + p.nk - kb, kKC);
    const bool full = kv0 == 0 && kv1 == kKC;
    const int cap = p.box_w * p.box_h;
    Box* const box = reinterpret_cast<Box*>(fsm);  // ring of kBoxRing slots (t & 15)
    float* const wmax = fsm + kBoxRing * sizeof(Box) / sizeof(float);  // 8 per-warp maxima
    int* const patch0 = reinterpret_cast<int*>(wmax + 8);       // two buffers of cap ints

    // this column's voxels (0 outside the slab / volume): x(i, j, kb + kk)
    float x[kKC];
    float xmax = 0.f;
#pragma unroll
    for (int kk = 0; kk < kKC; ++kk) {
        const bool in = active && kk >= kv0 && kk < kv1;
        x[kk] = in ? __ldg(p.vol + ((long)(kb + kk - p.k0) * p.Ny + j) * p.Nx + i) : 0.f;
        xmax = fmaxf(xmax, fabsf(x[kk]));
    }
    // Fixed-point scale of the patch (shared-memory atomics are native only for 32-bit
    // integers; float adds would be CAS loops): 2^e with  max|x| * qfactor * 2^e < 2^30, so no
    // patch pixel can overflow, and every contribution keeps >= 19 bits below the largest one.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) xmax = fmaxf(xmax, __shfl_xor_sync(0xffffffffu, xmax, o));
    if (lane == 0) wmax[warp] = xmax;
    __syncthreads();
    xmax = wmax[0];
#pragma unroll
    for (int w = 1; w < kThreads / 32; ++w) xmax = fmaxf(xmax, wmax[w]);
    if (xmax == 0.f) return;  // an empty block of the volume adds nothing
    int ex;
    frexpf(xmax * p.qfactor, &ex);  // xmax qfactor < 2^ex
    const float scale = ldexpf(1.f, 30 - ex), inv_scale = ldexpf(1.f, ex - 30);
    // patch boxes of views t0 .. t0+7: lanes 4 v .. 4 v + 3 take view t0 + v at the tile's
    // corner columns (u, v are linear-fractional in the column position: extremes sit at
    // corners), so one warp computes eight views' boxes and corner invariants in one pass.
    auto make_box8 = [&](int t0) {
        const int t = t0 + (lane >> 2);
        const bool valid = t < p.n_views;
        const int c = lane & 3;
        const double ci = (c & 1) ? min(tile_i * kTI + kTI, p.Nx) - 1 : tile_i * kTI;
        const double cj = (c & 2) ? min(tile_j * kTJ + kTJ, p.Ny) - 1 : tile_j * kTJ;
        const double* Pc = pt.P[valid ? t : t0];
        const ColInv ci0 = column_invariants(Pc, ci, cj, (double)kb);
        double umin = ci0.u, umax = ci0.u;
        double vmin = ci0.v + kv0 * ci0.dv, vmax = ci0.v + (kv1 - 1) * ci0.dv;
        if (vmin > vmax) { const double q = vmin; vmin = vmax; vmax = q; }
#pragma unroll
        for (int o = 1; o < 4; o <<= 1) {
            umin = fmin(umin, __shfl_xor_sync(0xffffffffu, umin, o));
            umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
            vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
            vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
        }
        if (valid && c == 0) {  // the base corner (tile_i * 16, tile_j * 16)
            Box b;
            b.u_org = (int)floor(umin) - 1;
            b.v_org = (int)floor(vmin) - 1;
            b.w = (int)floor(umax) - b.u_org + 3;
            b.h = (int)floor(vmax) - b.v_org + 3;
            if (b.w > p.box_w || b.h > p.box_h) __trap();  // the host bound is conservative
            const double fu = floor(ci0.u), fv = floor(ci0.v);
            b.uci = (int)fu;
            b.vci = (int)fv;
            b.ucf = (float)(ci0.u - fu);
            b.vcf = (float)(ci0.v - fv);
            b.uc = (float)ci0.u;
            b.vc = (float)ci0.v;
            b.zc = (float)ci0.z;
            b.p0 = (float)Pc[0]; b.p1 = (float)Pc[1]; b.p3 = (float)Pc[3]; b.p4 = (float)Pc[4];
            b.p5 = (float)Pc[5]; b.p7 = (float)Pc[7]; b.p8 = (float)Pc[8];
            b.pad0 = b.pad1 = 0.f;
            box[t & (kBoxRing - 1)] = b;
        }
    };
    // add the patch of view t to the projection (non-zero, on-detector, in-band taps) and
    // zero what was read, so the buffer is clean for view t+2
    const int r0 = tid / p.box_w, c0 = tid - r0 * p.box_w;
    const int dr = kThreads / p.box_w, dc = kThreads - dr * p.box_w;
    auto flush = [&](int t) {
        const Box b = box[t & (kBoxRing - 1)];
        int* const pa = patch0 + (t & 1) * cap;
        float* const pv = p.proj + (long)t * p.n_rows * p.Nu;
        // (r, c) of element e = tid + kThreads q stepped incrementally (no division per element)
        int r = r0, c = c0;
        for (int e = tid; e < b.h * p.box_w; e += kThreads) {
            const int q = pa[e];
            pa[e] = 0;
            const int col = b.u_org + c, row = b.v_org + r;
            if (q != 0 && c < b.w && col >= 0 && col < p.Nu && row >= p.v0 &&
                row < p.v0 + p.n_rows)
                atomicAdd(pv + (long)(row - p.v0) * p.Nu + col, (float)q * inv_scale);
            c += dc;
            r += dr;
            if (c >= p.box_w) {
                c -= p.box_w;
                ++r;
            }
        }
    };

    for (int e = tid; e < 2 * cap; e += kThreads) patch0[e] = 0;
    if (warp == 0) make_box8(0);  // views 0 .. 7
    __syncthreads();
    // One barrier per view: splat view t into buffer t & 1 while view t-1's buffer is flushed
    // and the box of view t+1 is computed.
    for (int t = 0; t < p.n_views; ++t) {
        const Box b = box[t & (kBoxRing - 1)];
        int* const pa = patch0 + (t & 1) * cap;
        // dv < 1: fp32 offsets from the tile corner; many rows per slice: per-column fp64 with
        // dv split into whole rows + an fp32 fraction (an fp32 dv would carry ~1e-7 dv per slice)
        const ThreadInv ti = SMALL_DV ? corner_inv(b, fdi, fdj)
                                      : split(column_invariants(pt.P[t], di, dj, (double)kb));
        int* const base = pa + (ti.nv - b.v_org) * p.box_w + (ti.nu - b.u_org);
        const float ws1 = ti.du * scale, ws0 = (1.f - ti.du) * scale;  // columns nu, nu+1
        // Along k the column's contributions move down the detector rows (v affine in k, dv > 0):
        // accumulate the (1 - fr) and fr shares of rows cur, cur+1 in registers (A, B) and add
        // a row to the patch only when the walk leaves it -- two integer atomics per row
        // instead of four float atomics per slice.
        if (active) {
            float fr;
            int cur = (int)(floor_bits(fmaf((float)kv0, ti.dvf, ti.fv0), &fr) - 0x4B000000u) +
                      kv0 * ti.dvi;
            float A = 0.f, B = 0.f;
            auto add_row = [&](int r, float sv) {  // Alg. alg:subpixel lines 4-5, transposed
                int* q = base + r * p.box_w;
                atomicAdd(q, __float2int_rn(sv * ws0));
                atomicAdd(q + 1, __float2int_rn(sv * ws1));
            };
            if constexpr (SMALL_DV) {
                if (full) {
                    // dv < 1, whole chunk: each slice stays on row cur or moves to cur + 1.
                    // One branch around the two integer reds at a running row address, the
                    // A/B shift by selects, no slab masks (measured: 690 vs 655 GUPS; reds
                    // predicated inside the instruction were compiled to two branches, 560).
                    uint32_t rowp = smem_u32_fp(base + cur * p.box_w);
                    const uint32_t pitch = (uint32_t)p.box_w * 4u;
                    // W folded into the column weights; the walk keeps S = the x sum of the
                    // current row window and Bx = its fr-weighted part, so row cur holds
                    // S - Bx and row cur + 1 holds Bx (one FADD + one FFMA per slice).
                    const float wW0 = ws0 * ti.W, wW1 = ws1 * ti.W;
                    float S = 0.f, Bx = 0.f;
#pragma unroll
                    for (int kk = 0; kk < kKC; ++kk) {
                        const int n =
                            (int)(floor_bits(fmaf((float)kk, ti.dv, ti.fv0), &fr) - 0x4B000000u);
                        const uint32_t adv = n != cur ? 1u : 0u;
                        if (adv) {
                            const float a = S - Bx;
                            red_add_if(rowp, __float2int_rn(a * wW0), 1u);
                            red_add_if(rowp + 4, __float2int_rn(a * wW1), 1u);
                        }
                        S = adv ? Bx : S;
                        Bx = adv ? 0.f : Bx;
                        rowp += adv * pitch;
                        cur = n;
                        S += x[kk];                 // W_dis x (Alg. alg:bp line 8, transposed)
                        Bx = fmaf(x[kk], fr, Bx);   // rows n, n+1 (line 6)
                    }
                    A = (S - Bx) * ti.W;
                    B = Bx * ti.W;
                } else {
#pragma unroll
                    for (int kk = 0; kk < kKC; ++kk) {
                        const int n =
                            (int)(floor_bits(fmaf((float)kk, ti.dv, ti.fv0), &fr) - 0x4B000000u);
                        const bool adv = n != cur && kk >= kv0 && kk < kv1;
                        int* q = base + cur * p.box_w;
                        const int q0 = __float2int_rn(A * ws0), q1 = __float2int_rn(A * ws1);
                        if (adv) {
                            atomicAdd(q, q0);
                            atomicAdd(q + 1, q1);
                        }
                        A = adv ? B : A;
                        B = adv ? 0.f : B;
                        cur += adv ? 1 : 0;
                        const float val = ti.W * x[kk];
                        A = fmaf(val, 1.f - fr, A);
                        B = fmaf(val, fr, B);
                    }
                }
            } else {
#pragma unroll
                for (int kk = 0; kk < kKC; ++kk) {
                    if (x[kk] == 0.f) continue;  // outside the slab (and empty voxels)
                    const int n =
                        (int)(floor_bits(fmaf((float)kk, ti.dvf, ti.fv0), &fr) - 0x4B000000u) +
                        kk * ti.dvi;  // whole rows of dv added as integers (backproject.cu walk 1)
                    if (n != cur) {  // the walk left row cur (n > cur)
                        if (A != 0.f) add_row(cur, A);
                        if (n == cur + 1) {
                            A = B;
                        } else {
                            if (B != 0.f) add_row(cur + 1, B);
                            A = 0.f;
                        }
                        B = 0.f;
                        cur = n;
                    }
                    const float val = ti.W * x[kk];
                    A = fmaf(val, 1.f - fr, A);
                    B = fmaf(val, fr, B);
                }
            }
            add_row(cur, A);
            add_row(cur + 1, B);
        }
        if (t > 0) flush(t - 1);
        // views t+2 .. t+9 (slots of views t-1, t in use; t+1 already computed)
        if (((t + 2) & 7) == 0 && warp == (((t + 2) >> 3) & 7)) make_box8(t + 2);
        __syncthreads();
    }
    if (p.n_views > 0) flush(p.n_views - 1);
}

}  // namespace

ifdk_status launch_forward_project(const ifdk_geometry* g, const float* vol, int k0, int nk,
                                   long s0, long n_views, float* proj, int v0, int n_rows,
                                   int accumulate, cudaStream_t st)
{
    cudaError_t e;
    if (!accumulate && n_views > 0) {
        e = cudaMemsetAsync(proj, 0, sizeof(float) * (size_t)n_views * n_rows * g->Nu, st);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
    }
    if (n_views == 0 || nk == 0) return IFDK_OK;
    FPParams p{};
    p.vol = vol;
    p.Nu = g->Nu; p.Nv = g->Nv; p.Nx = g->Nx; p.Ny = g->Ny;
    p.v0 = v0; p.n_rows = n_rows;
    p.k0 = k0; p.nk = nk;
    p.kb0 = (k0 / kKC) * kKC;
    p.tiles_i = (g->Nx + kTI - 1) / kTI;
    const int tiles_j = (g->Ny + kTJ - 1) / kTJ;
    const int n_chunks = (k0 + nk - p.kb0 + kKC - 1) / kKC;
    p.raster = std::min(16, p.tiles_i);
    double wb, hb;
    patch_bound(g, kTI, kTJ, kKC, &wb, &hb);
    p.box_w = (int)std::ceil(wb) + 6;
    p.box_h = (int)std::ceil(hb) + 6;
    const size_t smem =
        sizeof(int) * 2 * (size_t)p.box_w * p.box_h + kBoxRing * sizeof(Box) + 8 * sizeof(float);
    const double dv_min = g->D * g->Dz / (g->Dv * g->zmax);
    p.qfactor = (float)(256.0 * (1.0 / dv_min + 1.0) / (g->zmin * g->zmin));
    if (smem > 200 * 1024) return fail(IFDK_ERR_INVALID_ARGUMENT, "forward projector patch too large");
    // dv/dk < 1 everywhere (all five configs): the branch-free walk
    const bool small_dv = g->D * g->Dz / (g->Dv * g->zmin) < 0.999;
    auto kern = small_dv ? fp_kernel<true> : fp_kernel<false>;
    e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(fp)");
    dim3 grid((unsigned)(p.raster * tiles_j), (unsigned)n_chunks,
              (unsigned)((p.tiles_i + p.raster - 1) / p.raster));
    PTable pt;
    for (long t = 0; t < n_views; t += kMaxViewsPerLaunch) {
        const long n = std::min<long>(kMaxViewsPerLaunch, n_views - t);
        fill_ptable(g, s0 + t, n, pt);
        p.n_views = (int)n;
        p.proj = proj + (size_t)t * n_rows * g->Nu;
        kern<<<grid, kThreads, smem, st>>>(p, pt);
        e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "fp_kernel launch");
        count_launch();
    }
    return IFDK_OK;
}

}  // namespace ifdk

// ---- element-wise steps of SART / SIRT (reading c-I2) ---------------------------------------
namespace ifdk {
namespace {

__global__ void sart_ratio_kernel(const float* __restrict__ b, const float* ax,
                                  const float* __restrict__ R, float* out, long n)
{
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n;
         e += (long)gridDim.x * blockDim.x) {
        const float r = R[e];
        out[e] = r > 0.f ? (b[e] - ax[e]) / r : 0.f;  // rays no voxel reaches: 0 (c-I3)
    }
}

__global__ void sart_update_kernel(float* x, const float* __restrict__ c,
                                   const float* __restrict__ C, float lam, long n, int nonneg)
{
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n;
         e += (long)gridDim.x * blockDim.x) {
        const float w = C[e];
        float v = x[e] + (w > 0.f ? lam * c[e] / w : 0.f);  // voxels no ray sees: kept (c-I3)
        if (nonneg) v = fmaxf(v, 0.f);
        x[e] = v;
    }
}

// MLEM / OS-EM (reading c-I4): ratio b / (M x) where M x > 0 (else 0), and the
// multiplicative update x <- x c / C where C = M^T 1 > 0 (else x unchanged).
__global__ void mlem_ratio_kernel(const float* __restrict__ b, const float* ax, float* out, long n)
{
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n;
         e += (long)gridDim.x * blockDim.x) {
        const float a = ax[e];
        out[e] = a > 0.f ? b[e] / a : 0.f;
    }
}

__global__ void mlem_update_kernel(float* x, const float* __restrict__ c,
                                   const float* __restrict__ C, long n)
{
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n;
         e += (long)gridDim.x * blockDim.x) {
        const float w = C[e];
        if (w > 0.f) x[e] = x[e] * c[e] / w;
    }
}

__global__ void fill_kernel(float* x, float value, long n)
{
    for (long e = blockIdx.x * (long)blockDim.x + threadIdx.x; e < n;
         e += (long)gridDim.x * blockDim.x)
        x[e] = value;
}

unsigned elementwise_grid(long n)
{
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long blocks = (n + 255) / 256;
    return (unsigned)std::max(1L, std::min(blocks, (long)sms * 8));
}

}  // namespace

ifdk_status launch_sart_ratio(const float* b, const float* ax, const float* R, float* out, long n,
                              cudaStream_t st)
{
    if (n == 0) return IFDK_OK;
    sart_ratio_kernel<<<elementwise_grid(n), 256, 0, st>>>(b, ax, R, out, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "sart_ratio_kernel launch");
    count_launch();
    return IFDK_OK;
}

ifdk_status launch_sart_update(float* x, const float* c, const float* C, float lam, long n,
                               int nonneg, cudaStream_t st)
{
    if (n == 0) return IFDK_OK;
    sart_update_kernel<<<elementwise_grid(n), 256, 0, st>>>(x, c, C, lam, n, nonneg);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "sart_update_kernel launch");
    count_launch();
    return IFDK_OK;
}

ifdk_status launch_mlem_ratio(const float* b, const float* ax, float* out, long n,
                              cudaStream_t st)
{
    if (n == 0) return IFDK_OK;
    mlem_ratio_kernel<<<elementwise_grid(n), 256, 0, st>>>(b, ax, out, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "mlem_ratio_kernel launch");
    count_launch();
    return IFDK_OK;
}

ifdk_status launch_mlem_update(float* x, const float* c, const float* C, long n, cudaStream_t st)
{
    if (n == 0) return IFDK_OK;
    mlem_update_kernel<<<elementwise_grid(n), 256, 0, st>>>(x, c, C, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "mlem_update_kernel launch");
    count_launch();
    return IFDK_OK;
}

ifdk_status launch_fill(float* x, float value, long n, cudaStream_t st)
{
    if (n == 0) return IFDK_OK;
    fill_kernel<<<elementwise_grid(n), 256, 0, st>>>(x, value, n);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "fill_kernel launch");
    count_launch();
    return IFDK_OK;
}

}  // namespace ifdk
