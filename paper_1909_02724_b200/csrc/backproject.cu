// backproject.cu -- BP-sm100: voxel-driven FDK back-projection (Alg. alg:bp P:402-430,
// Alg. alg:subpixel P:431-447) organised around the appendix invariant (Theorems 2-3,
// P:506-507): for fixed (i, j, beta) the depth z, the detector column u and the weight
// 1/z^2 are constant along k, and v is affine in k.
//
// Mapping (B200-first; not the paper's shflBP design):
//  * A CTA (256 threads = 8 warps of 8(i) x 4(j) columns) owns a 16 x 16 column tile and a
//    64-slice k-chunk aligned to global multiples of 64.  Each thread owns one voxel column;
//    per (column, view) it forms u, the base of v, dv/dk and 1/z^2 once, then per update only
//    v = fv0 + kappa dv in fp32, a floor, shared-memory tap loads and packed fp32x2 FMAs.
//  * The detector patch the tile x chunk projects onto (its extent is bounded from the
//    tile corners: u, v are linear-fractional, so extremes sit at corners) is staged per
//    view by TMA (cp.async.bulk.tensor, OOB zero fill = the per-tap zero border, reading
//    c-A9) into a ring of boxes (mbarrier completion); the walk reads both taps of a row
//    straight from the box (two LDS.32, row pitch 8 mod 32 words: conflict-free).
//  * Default (bp_quad2_kernel, walks 13 / 14): runs of four (QUAD, 0.5 <= dv/dk < 1) or five
//    (QUINT, dv/dk < 1/2) slices share one floor; the 64 partial sums of a thread live in
//    tensor memory (tcgen05.alloc / ld / st), two views per step, three CTAs per SM; the
//    per-(column, view) invariants are fp32 offsets from the tile corner's fp64 values; slab
//    ends inside a chunk are walked by the same kernel with a masked write-back.  Variants
//    (A/B and tests, ifdk_set_bp_variant): the TRIPLE family (bp_tmem2_kernel, bp_tmem_kernel,
//    bp_raw_kernel, pair-patch companions in bp_kernel for partial chunks; fp64 per-thread
//    invariants, bitwise equal to each other) and the PAIR family (walks 2, 4, 5).
//  * P_s lives in constant memory: each launch carries the fp64 rows of its <= 256 views in
//    a __grid_constant__ kernel parameter (param space = the constant bank), so no
//    per-launch device allocation or host-to-device copy is needed.  Longer view ranges are
//    split into launches at global multiples of 256 views, which are also flush points of
//    the two-level summation, so the split does not change a bit.
//  * Views are summed in order; every VB = 128 views (aligned to the global view index) the
//    partial sums are added to the volume, a two-level summation.
//  * The box is sized from a conservative geometric bound (patch_bound), so every view's
//    patch fits it; a violation is a bug and traps (it kills the CUDA context).  Geometries
//    whose box cannot be described to TMA or exceeds the opt-in shared memory (N_u % 4 != 0,
//    box taller than 256 rows or too large) take a walk with taps read from global memory.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "ifdk_internal.h"
#include "kwalk.cuh"
#include "mbar.cuh"

namespace ifdk {
namespace {

constexpr int kTI = 16, kTJ = 16, kThreads = 256;
constexpr int kRasterTiles = 16;  // tile columns per raster band (see bp_kernel)

struct BPParams {
    const float* Q;   // band [n_views][n_rows][Nu]
    float* vol;       // slab [nk][Ny][Nx]
    long n_views;
    long s0;
    int Nu, Nv, Nx, Ny;
    int v0, n_rows;
    int k0, nk;       // slab (global k)
    int kb0;          // global k of chunk 0 (multiple of KC)
    int tiles_i;
    int raster;       // tile columns per raster band (see bp_kernel)
    int box_w, box_h;
    int raw_bytes;    // bytes of one raw box (multiple of 128)
    int vb;           // view batch of the two-level summation
    uint32_t neg_magic;  // -0x4B000000 * P2 * 8 mod 2^32 (see accumulate_view_smem)
    int pair;            // rows of slack for a multi-slice walk (PAIR / TRIPLE): 1, else 0
    int walk;            // slices per floor: 1, 2 (PAIR) or 3 (TRIPLE)
    int accumulate;
    // fused reduce (RedDest): 0 = write / accumulate into vol; 1 = red.global.add, 2 =
    // multimem.red into dest[d] (slices dest_k0[d] ..); vol is unused then
    int red;
    int n_dest;
    int dest_k0[kMaxRedDest];
    float* dest[kMaxRedDest];
};

// Address of voxel (i, j, k) in the slab vol (the flush walks it slice by slice).
__device__ __forceinline__ float* vol_voxel(const BPParams& p, int k, int j, int i)
{
    return p.vol + ((long)(k - p.k0) * p.Ny + j) * p.Nx + i;
}

// One partial sum of voxel (i, j, k) into the volume: q (its address in vol) overwritten /
// added, or -- the fused reduce -- atomically added into the destination slab holding slice k
// (slabs need not align with the 64-slice chunks; the order of the adds from different
// launches / GPUs is not fixed, so fp32 rounding may differ).
__device__ __noinline__ void red_voxel(const BPParams& p, int k, int j, int i, float v)
{
    int d = 0;
    while (d + 1 < p.n_dest && k >= p.dest_k0[d + 1]) ++d;
    float* r = p.dest[d] + ((long)(k - p.dest_k0[d]) * p.Ny + j) * p.Nx + i;
    if (p.red == 1)
        asm volatile("red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(r), "f"(v) : "memory");
    else
        asm volatile("multimem.red.relaxed.sys.global.add.f32 [%0], %1;" ::"l"(r), "f"(v)
                     : "memory");
}

// RED: the kernel instantiation may run the fused reduce (checked at run time, the reduce path
// out of line).  The TMEM kernels (bp_quad2_kernel, bp_tmem2_kernel) have separate RED = false
// instantiations without it: the mere call site cost 1.2 % (2193 vs 2220 GUPS, config 4).
template <bool RED = true>
__device__ __forceinline__ void put_voxel(const BPParams& p, float* q, int k, int j, int i,
                                          float v, bool overwrite)
{
    if (!RED || p.red == 0)
        *q = overwrite ? v : *q + v;
    else
        red_voxel(p, k, j, i, v);
}

struct __align__(16) Meta {
    double P[10];        // P_s (bp_kernel reads it from here, 128-bit loads)
    int u_org, v_org;    // box origin (detector column, row)
    int w_need, h_need;  // columns / rows of the box the tile x chunk can touch
    // QUAD / QUINT walks (WALK 13): the tile corner's invariants in fp64, split (u_c = uci +
    // ucf, v_c(kb) = vci + vcf), the corner's u_c, v_c, z_c rounded to fp32 and the used entries
    // of P_s rounded to fp32 -- each thread adds its small offset from the corner in fp32.
    // Laid out in 16-byte quads so a thread reads them with three 128-bit loads.
    int uci, vci;
    float ucf, vcf;
    float uc, vc, zc, p0;
    float p1, p3, p4, p5;
    float p7, p8;
    int fast;            // the patch fits the box
    int pad;
};

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}

__device__ __forceinline__ float2 lds64(uint32_t addr)
{
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(addr));
    return v;
}

// Partial chunks (FULL = false) run the whole unrolled walk and mask only the accumulation,
// so the floors of masked slices -- below the first slice of a head chunk, past the last one
// of a tail chunk -- can point outside the box, which was sized for the slices in the slab
// only; clamping the floor address into the box keeps every shared load inside the
// allocation.  Unmasked slices' addresses are inside the box already, so their values do not
// change.  [lo, hi] = first and last floor address whose NR rows stay in the box.
template <bool FULL>
__device__ __forceinline__ uint32_t clamp_floor(uint32_t addr, uint32_t lo, uint32_t hi)
{
    if constexpr (FULL) return addr;
    else return min(max(addr, lo), hi);
}

// One view from the (a, delta) pair patch in shared memory.
//
// PAIR (needs dv < 1 px per slice, true for every config): two consecutive slices kk, kk+1
// touch at most three detector rows n, n+1, n+2 (v grows by dv < 1), so one floor, three
// LDS.64 and three horizontal lerps serve both updates: slice kk+1 uses rows (n, n+1) or
// (n+1, n+2) depending on whether fr + dv crosses 1 (one FSEL, no second floor).  12 B of shared memory per update
// instead of 16.  The partial-chunk path runs the same arithmetic and only masks the
// accumulation, so a slab split never changes a bit.
// `hook(q)` runs once per 8-slice group q (0 .. KC/8 - 1) in program order with the group's
// updates: the kernel uses it to transform row q of the next view's patch while this view's
// shared loads are in flight.
template <int KC, int P2, bool FULL, int WALK, typename Hook>
__device__ __forceinline__ void accumulate_view_smem(float (&acc)[KC], uint32_t pair_base,
                                                     uint32_t neg_magic, const ThreadInv& t,
                                                     int u_org, int v_org, int kv0, int kv1,
                                                     uint32_t lo_a, uint32_t hi_a, Hook&& hook)
{
    // byte address of pair (row nv + n, col nu) = pair_base + ((nv - v_org + n) P2 + nu - u_org) 8
    // neg_magic = -0x4B000000 * P2 * 8 (mod 2^32) arrives as a kernel parameter so that ptxas
    // cannot split it back out of the base: one IMAD per floor forms the tap address.
    const uint32_t a0 =
        pair_base + (uint32_t)(((t.nv - v_org) * P2 + (t.nu - u_org)) * 8) + neg_magic;
    constexpr uint32_t S = P2 * 8;
    float fv0 = t.fv0;
    if constexpr (WALK == 3) {
        // TRIPLE (needs 0.5 <= dv < 1, configs 1-4): slices kk, kk+1, kk+2 lie within rows
        // n .. n+3 (fr + 2 dv < 3), and slice kk+2 sits g2 = fr + 2 dv - 2 in [-1, 1) rows past
        // row n+2 (2 dv >= 1): four LDS.64 and one floor serve three updates, 10.7 B of shared
        // memory per update.
        // Triples cover slices 0 .. KC-5; the last four run as two PAIR steps, exactly as the
        // RAW triple walk (walk 6) does, so the two are bitwise equal (walk 3 serves walk 6's
        // partial chunks).
        constexpr int TRI_END = KC - 4;
        static_assert(TRI_END % 3 == 0, "whole triples before the pair tail");
#pragma unroll
        for (int kk = 0; kk + 3 <= TRI_END; kk += 3) {
            if (kk == 0 || (kk >> 3) != ((kk - 3) >> 3)) {  // first triple of an 8-slice group
                hook(kk >> 3);
                asm volatile("mov.b32 %0, %0;" : "+f"(fv0));
            }
            float fr0;
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dv, fv0), &fr0);
            const uint32_t addr = clamp_floor<FULL>(bits * S + a0, lo_a, hi_a);
            const float2 p0 = lds64(addr);
            const float2 p1 = lds64(addr + S);
            const float2 p2 = lds64(addr + 2 * S);
            const float2 p3 = lds64(addr + 3 * S);
            const float h0 = fmaf(t.du, p0.y, p0.x);  // Alg. alg:subpixel lines 4-5
            const float h1 = fmaf(t.du, p1.y, p1.x);
            const float h2 = fmaf(t.du, p2.y, p2.x);
            const float h3 = fmaf(t.du, p3.y, p3.x);
            const float d01 = h1 - h0, d12 = h2 - h1;
            if (FULL || (kk >= kv0 && kk < kv1))
                acc[kk] = fmaf(t.W, fmaf(fr0, d01, h0), acc[kk]);  // line 6; Alg. alg:bp line 10
            const float g1 = fr0 + t.dvm1;
            const float e1 = g1 >= 0.f ? d12 : d01;
            if (FULL || (kk + 1 >= kv0 && kk + 1 < kv1))
                acc[kk + 1] = fmaf(t.W, fmaf(g1, e1, h1), acc[kk + 1]);
            const float g2 = g1 + t.dvm1;  // fr + 2 dv - 2
            const float e2 = g2 >= 0.f ? h3 - h2 : d12;
            if (FULL || (kk + 2 >= kv0 && kk + 2 < kv1))
                acc[kk + 2] = fmaf(t.W, fmaf(g2, e2, h2), acc[kk + 2]);
        }
#pragma unroll
        for (int kk = TRI_END; kk < KC; kk += 2) {  // the PAIR tail (see WALK == 2)
            float fr0;
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dv, fv0), &fr0);
            const uint32_t addr = clamp_floor<FULL>(bits * S + a0, lo_a, hi_a);
            const float2 p0 = lds64(addr);
            const float2 p1 = lds64(addr + S);
            const float2 p2 = lds64(addr + 2 * S);
            const float h0 = fmaf(t.du, p0.y, p0.x);
            const float h1 = fmaf(t.du, p1.y, p1.x);
            const float h2 = fmaf(t.du, p2.y, p2.x);
            const float d01 = h1 - h0;
            if (FULL || (kk >= kv0 && kk < kv1))
                acc[kk] = fmaf(t.W, fmaf(fr0, d01, h0), acc[kk]);
            const float g = fr0 + t.dvm1;
            const float d = g >= 0.f ? h2 - h1 : d01;
            if (FULL || (kk + 1 >= kv0 && kk + 1 < kv1))
                acc[kk + 1] = fmaf(t.W, fmaf(g, d, h1), acc[kk + 1]);
        }
    } else if constexpr (WALK == 8) {
        // 3-ROW TRIPLE (needs dv < 1/2, config 5): slices kk, kk+1, kk+2 all lie within rows
        // n .. n+2 (fr + 2 dv < 2); slices kk+1 and kk+2 sit g1 = fr + dv - 1 and g2 = g1 + dv
        // rows past row n+1 (both in [-1, 1)).  Same grouping and pair tail as the RAW form
        // (walk 7), which it serves on partial chunks, bitwise.
        constexpr int TRI_END = KC - 4;
        static_assert(TRI_END % 3 == 0, "whole triples before the pair tail");
#pragma unroll
        for (int kk = 0; kk + 3 <= TRI_END; kk += 3) {
            if (kk == 0 || (kk >> 3) != ((kk - 3) >> 3)) {
                hook(kk >> 3);
                asm volatile("mov.b32 %0, %0;" : "+f"(fv0));
            }
            float fr0;
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dv, fv0), &fr0);
            const uint32_t addr = clamp_floor<FULL>(bits * S + a0, lo_a, hi_a);
            const float2 p0 = lds64(addr);
            const float2 p1 = lds64(addr + S);
            const float2 p2 = lds64(addr + 2 * S);
            const float h0 = fmaf(t.du, p0.y, p0.x);  // Alg. alg:subpixel lines 4-5
            const float h1 = fmaf(t.du, p1.y, p1.x);
            const float h2 = fmaf(t.du, p2.y, p2.x);
            const float d01 = h1 - h0, d12 = h2 - h1;
            if (FULL || (kk >= kv0 && kk < kv1))
                acc[kk] = fmaf(t.W, fmaf(fr0, d01, h0), acc[kk]);  // line 6; Alg. alg:bp line 10
            const float g1 = fr0 + t.dvm1;
            const float e1 = g1 >= 0.f ? d12 : d01;
            if (FULL || (kk + 1 >= kv0 && kk + 1 < kv1))
                acc[kk + 1] = fmaf(t.W, fmaf(g1, e1, h1), acc[kk + 1]);
            const float g2 = g1 + t.dv;
            const float e2 = g2 >= 0.f ? d12 : d01;
            if (FULL || (kk + 2 >= kv0 && kk + 2 < kv1))
                acc[kk + 2] = fmaf(t.W, fmaf(g2, e2, h1), acc[kk + 2]);
        }
#pragma unroll
        for (int kk = TRI_END; kk < KC; kk += 2) {  // the PAIR tail
            float fr0;
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dv, fv0), &fr0);
            const uint32_t addr = clamp_floor<FULL>(bits * S + a0, lo_a, hi_a);
            const float2 p0 = lds64(addr);
            const float2 p1 = lds64(addr + S);
            const float2 p2 = lds64(addr + 2 * S);
            const float h0 = fmaf(t.du, p0.y, p0.x);
            const float h1 = fmaf(t.du, p1.y, p1.x);
            const float h2 = fmaf(t.du, p2.y, p2.x);
            const float d01 = h1 - h0;
            if (FULL || (kk >= kv0 && kk < kv1))
                acc[kk] = fmaf(t.W, fmaf(fr0, d01, h0), acc[kk]);
            const float g = fr0 + t.dvm1;
            const float d = g >= 0.f ? h2 - h1 : d01;
            if (FULL || (kk + 1 >= kv0 && kk + 1 < kv1))
                acc[kk + 1] = fmaf(t.W, fmaf(g, d, h1), acc[kk + 1]);
        }
    } else if constexpr (WALK == 2) {
#pragma unroll
        for (int kk = 0; kk < KC; kk += 2) {
            // Every 8 slices, launder fv0 through a volatile asm so that the compiler cannot
            // hoist the address arithmetic of later slices above earlier shared loads.
            if ((kk & 7) == 0) {
                hook(kk >> 3);
                asm volatile("mov.b32 %0, %0;" : "+f"(fv0));
            }
            float fr0;
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dv, fv0), &fr0);
            const uint32_t addr = clamp_floor<FULL>(bits * S + a0, lo_a, hi_a);
            const float2 p0 = lds64(addr);
            const float2 p1 = lds64(addr + S);
            const float2 p2 = lds64(addr + 2 * S);
            const float h0 = fmaf(t.du, p0.y, p0.x);  // Alg. alg:subpixel lines 4-5
            const float h1 = fmaf(t.du, p1.y, p1.x);
            const float h2 = fmaf(t.du, p2.y, p2.x);
            const float d01 = h1 - h0;
            if (FULL || (kk >= kv0 && kk < kv1))
                acc[kk] = fmaf(t.W, fmaf(fr0, d01, h0), acc[kk]);  // line 6; Alg. alg:bp line 10
            // slice kk+1 sits g = fr0 + dv - 1 rows past row n+1 (g in [-1, 1)): interpolate
            // from h1 towards h2 (g >= 0) or back towards h0 (g < 0, h1 + g d01 = h0 + (1+g) d01).
            const float g = fr0 + t.dvm1;
            const float d = g >= 0.f ? h2 - h1 : d01;
            if (FULL || (kk + 1 >= kv0 && kk + 1 < kv1))
                acc[kk + 1] = fmaf(t.W, fmaf(g, d, h1), acc[kk + 1]);
        }
    } else {
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
            if ((kk & 7) == 0) {
                hook(kk >> 3);
                asm volatile("mov.b32 %0, %0;" : "+f"(fv0));
            }
            if (!FULL && (kk < kv0 || kk >= kv1)) continue;
            float fr;  // v = fv0 + kk dvf + kk dvi (whole rows): fp32 error ~ulp(KC), any dv
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dvf, fv0), &fr);
            const uint32_t addr =
                clamp_floor<FULL>((bits + (uint32_t)(kk * t.dvi)) * S + a0, lo_a, hi_a);
            const float2 p0 = lds64(addr);
            const float2 p1 = lds64(addr + S);
            const float h0 = fmaf(t.du, p0.y, p0.x);
            const float h1 = fmaf(t.du, p1.y, p1.x);
            acc[kk] = fmaf(t.W, fmaf(fr, h1 - h0, h0), acc[kk]);
        }
    }
}

// ---- PAIR walk on packed fp32x2 (Blackwell FFMA2 / FADD2): WALK == 4 ------------------
// The arithmetic of the WALK == 2 PAIR walk, element for element (same operations, same
// rounding), issued two slice pairs at a time: slice pair A = (kk, kk+1) in the low halves,
// B = (kk+2, kk+3) in the high halves.  v, the floor, the fractions, the row differences,
// the vertical lerps and the accumulation run as f32x2 instructions; only the address IMAD,
// the shared loads, the horizontal lerps (operands arrive as (a, delta) pairs of one row) and
// the row select stay scalar: 29 instructions per 4 updates instead of 38.  The accumulators
// are register pairs: acc2[kk/2] = (slice kk, slice kk+2), acc2[kk/2+1] = (kk+1, kk+3).
using f2x = unsigned long long;

__device__ __forceinline__ f2x pk2(float lo, float hi)
{
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float lo2(f2x r)
{
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return a;
}
__device__ __forceinline__ float hi2(f2x r)
{
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return b;
}
__device__ __forceinline__ f2x fma2(f2x a, f2x b, f2x c)
{
    f2x r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(a), "l"(b), "l"(c));
    return r;
}
__device__ __forceinline__ f2x add2(f2x a, f2x b)
{
    f2x r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2x add2_rd(f2x a, f2x b)
{
    f2x r;
    asm("add.rm.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ f2x sub2(f2x a, f2x b)
{
    f2x r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}

template <int KC, int P2, bool FULL, typename Hook>
__device__ __forceinline__ void accumulate_view_smem_x2(f2x (&acc)[KC / 2], uint32_t pair_base,
                                                        uint32_t neg_magic, const ThreadInv& t,
                                                        int u_org, int v_org, int kv0, int kv1,
                                                        uint32_t lo_a, uint32_t hi_a, Hook&& hook)
{
    static_assert(KC % 4 == 0, "x2 walk: whole slice quads");
    const uint32_t a0 =
        pair_base + (uint32_t)(((t.nv - v_org) * P2 + (t.nu - u_org)) * 8) + neg_magic;
    constexpr uint32_t S = P2 * 8;
    const f2x dv2 = pk2(t.dv, t.dv), dvm12 = pk2(t.dvm1, t.dvm1), W2 = pk2(t.W, t.W);
    const f2x magic2 = pk2(8388608.0f, 8388608.0f), nmagic2 = pk2(-8388608.0f, -8388608.0f);
    f2x fv02 = pk2(t.fv0, t.fv0);
    // (kk, kk+2) as floats, stepped by an exact FADD2 (kept opaque so that it is not
    // folded into two uniform-register moves per quad)
    f2x kpair = pk2(0.f, 2.f);
    const f2x four2 = pk2(4.f, 4.f);
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
        if ((kk & 7) == 0) {
            hook(kk >> 3);
            asm volatile("mov.b64 %0, %0;" : "+l"(fv02));
        }
        // v of slices kk (A) and kk+2 (B); floor by the round-down magic add (floor_bits)
        const f2x v = fma2(kpair, dv2, fv02);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(kpair) : "l"(four2));
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = clamp_floor<FULL>(__float_as_uint(lo2(tb)) * S + a0, lo_a, hi_a);
        const uint32_t adB = clamp_floor<FULL>(__float_as_uint(hi2(tb)) * S + a0, lo_a, hi_a);
        const float2 pA0 = lds64(adA), pA1 = lds64(adA + S), pA2 = lds64(adA + 2 * S);
        const float2 pB0 = lds64(adB), pB1 = lds64(adB + S), pB2 = lds64(adB + 2 * S);
        // Alg. alg:subpixel lines 4-5 (horizontal), rows n, n+1, n+2 of A and B
        const f2x h0 = pk2(fmaf(t.du, pA0.y, pA0.x), fmaf(t.du, pB0.y, pB0.x));
        const f2x h1 = pk2(fmaf(t.du, pA1.y, pA1.x), fmaf(t.du, pB1.y, pB1.x));
        const f2x h2 = pk2(fmaf(t.du, pA2.y, pA2.x), fmaf(t.du, pB2.y, pB2.x));
        const f2x d01 = sub2(h1, h0), d12 = sub2(h2, h1);
        const f2x g = add2(fr, dvm12);  // second slice of each pair: g rows past row n+1
        const float eA = lo2(g) >= 0.f ? lo2(d12) : lo2(d01);
        const float eB = hi2(g) >= 0.f ? hi2(d12) : hi2(d01);
        const f2x val0 = fma2(fr, d01, h0);           // slices kk, kk+2 (line 6)
        const f2x val1 = fma2(g, pk2(eA, eB), h1);    // slices kk+1, kk+3
        acc[kk / 2] = fma2(W2, val0, acc[kk / 2]);  // Alg. alg:bp line 10
        acc[kk / 2 + 1] = fma2(W2, val1, acc[kk / 2 + 1]);
    }
}

// Slice kk of the packed accumulators (see accumulate_view_smem_x2).
template <int KC>
__device__ __forceinline__ void flush_x2(f2x (&acc)[KC / 2], const BPParams& p, int i, int j,
                                         int kb, int kv0, int kv1, bool overwrite)
{
    float* q = vol_voxel(p, kb, j, i);
    long plane = (long)p.Ny * p.Nx;
    asm volatile("mov.b64 %0, %0;" : "+l"(plane));
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
        const f2x a = acc[(kk & ~3) / 2 + (kk & 1)];
        const float v = (kk & 2) ? hi2(a) : lo2(a);
        if (kk >= kv0 && kk < kv1) put_voxel(p, q, kb + kk, j, i, v, overwrite);
        q += plane;
    }
#pragma unroll
    for (int q2 = 0; q2 < KC / 2; ++q2) acc[q2] = 0ull;
}

__device__ __forceinline__ float tapg(const float* __restrict__ Qv, int Nu, int Nv, int v0,
                                      int n_rows, int row, int col)
{
    if (col < 0 || col >= Nu || row < 0 || row >= Nv) return 0.f;  // zero border, c-A9
    const int r = row - v0;
    if (r < 0 || r >= n_rows) return 0.f;  // host guarantees band coverage
    return __ldg(Qv + (long)r * Nu + col);
}

// Horizontal lerp of detector row `row` from global memory, as the pair patch would give it.
__device__ __forceinline__ float rowg(const float* Qv, const BPParams& p, const ThreadInv& t,
                                      int row)
{
    const float a = tapg(Qv, p.Nu, p.Nv, p.v0, p.n_rows, row, t.nu);
    const float b = tapg(Qv, p.Nu, p.Nv, p.v0, p.n_rows, row, t.nu + 1);
    return fmaf(t.du, b - a, a);
}

// One view from global memory (bitwise the same arithmetic as the shared-memory path).
template <int KC, bool PAIR>
__device__ __forceinline__ void accumulate_view_global(float (&acc)[KC], const float* Qv,
                                                       const BPParams& p, const ThreadInv& t,
                                                       int kv0, int kv1)
{
    float fv0 = t.fv0;
    if constexpr (PAIR) {
#pragma unroll
        for (int kk = 0; kk < KC; kk += 2) {
            if ((kk & 3) == 0) asm volatile("mov.b32 %0, %0;" : "+f"(fv0));
            float fr0;
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dv, fv0), &fr0);
            const int row = t.nv + (int)(bits - 0x4B000000u);
            const float h0 = rowg(Qv, p, t, row), h1 = rowg(Qv, p, t, row + 1),
                        h2 = rowg(Qv, p, t, row + 2);
            const float d01 = h1 - h0;
            if (kk >= kv0 && kk < kv1) acc[kk] = fmaf(t.W, fmaf(fr0, d01, h0), acc[kk]);
            const float g = fr0 + t.dvm1;
            const float d = g >= 0.f ? h2 - h1 : d01;
            if (kk + 1 >= kv0 && kk + 1 < kv1) acc[kk + 1] = fmaf(t.W, fmaf(g, d, h1), acc[kk + 1]);
        }
    } else {
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) {
            if ((kk & 3) == 0) asm volatile("mov.b32 %0, %0;" : "+f"(fv0));
            if (kk < kv0 || kk >= kv1) continue;
            float fr;
            const uint32_t bits = floor_bits(fmaf((float)kk, t.dvf, fv0), &fr);
            const int row = t.nv + (int)(bits - 0x4B000000u) + kk * t.dvi;
            const float h0 = rowg(Qv, p, t, row), h1 = rowg(Qv, p, t, row + 1);
            acc[kk] = fmaf(t.W, fmaf(fr, h1 - h0, h0), acc[kk]);
        }
    }
}

// Register accumulators of a thread's KC slices: scalar, or fp32x2 pairs for WALK == 4.
template <int KC, bool X2>
struct AccRegs {
    float a[KC];
};
template <int KC>
struct AccRegs<KC, true> {
    f2x a[KC / 2];
};

template <int KC>
__device__ __forceinline__ void flush(float (&acc)[KC], const BPParams& p, int i, int j, int kb,
                                      int kv0, int kv1, bool overwrite)
{
    float* q = vol_voxel(p, kb, j, i);
    long plane = (long)p.Ny * p.Nx;
    // Opaque to the optimiser: stops it from hoisting 64 addresses out of the view loop.
    asm volatile("mov.b64 %0, %0;" : "+l"(plane));
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
        if (kk >= kv0 && kk < kv1) put_voxel(p, q, kb + kk, j, i, acc[kk], overwrite);
        acc[kk] = 0.f;
        q += plane;
    }
}

// Patch box of view t for the tile, computed by one warp: lane l takes corner l%4 of the
// tile (u, v are linear-fractional in the column position, so the extremes over the tile sit
// at its corners) at both ends of the chunk; min/max over the 4 corners.  Every 8 views the
// 8 warps compute the boxes of the next 8 views together, so no warp straggles at the barrier.
constexpr int kMetaRing = 16;

template <int KC, int WALK>
__device__ void compute_meta1(Meta* ring, const BPParams& p, const double* Pc, int t, int i_corner,
                              int j_corner, int kb, int kv0, int kv1)
{
    const int lane = threadIdx.x & 31;
    double P[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) P[q] = Pc[q];  // constant bank, warp-uniform address
    Meta* m = &ring[t & (kMetaRing - 1)];
    if (lane < 10) m->P[lane] = Pc[lane];
    const double ci = i_corner, cj = j_corner;
    const ColInv c = column_invariants(P, ci, cj, (double)kb);
    double umin = c.u, umax = c.u;
    // slices whose rows are read: the PAIR walk reads from the even slice below kv0 to the odd
    // slice at or above kv1 - 1, and one row more (h_need below)
    int ka = kv0, kz = kv1 - 1;
    if constexpr (WALK == 2 || WALK == 4) {
        ka = kv0 & ~1;
        kz = (kv1 - 1) | 1;
    } else if constexpr (WALK == 3 || WALK == 8) {  // triples on multiples of 3; pair tail
        constexpr int TRI_END = KC - 4;
        ka = kv0 < TRI_END ? kv0 - kv0 % 3 : (kv0 & ~1);
        kz = (kv1 - 1) < TRI_END ? (kv1 - 1) / 3 * 3 + 2 : ((kv1 - 1) | 1);
        kz = min(kz, KC - 1);
    }
    const double va = c.v + ka * c.dv, vb = c.v + kz * c.dv;
    double vmin = fmin(va, vb), vmax = fmax(va, vb);
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {
        umin = fmin(umin, __shfl_xor_sync(0xffffffffu, umin, o));
        umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    if (lane == 0) {
        const double fu0 = floor(umin), fu1 = floor(umax), fv0 = floor(vmin), fv1 = floor(vmax);
        // TMA (tile mode, no swizzle) faults unless the innermost box coordinate is a
        // multiple of 16 bytes (measured: tools/tma_probe.cu), so the column origin is
        // rounded down to a multiple of 4 floats.
        const bool finite = fu0 > -1e9 && fu1 < 1e9 && fv0 > -1e9 && fv1 < 1e9;
        const int u_org = finite ? (((int)fu0 - 1) & ~3) : 0;
        const double w_need = fu1 + 3.0 - u_org, h_need = fv1 - fv0 + 4.0 + p.pair;
        const bool fits = finite && w_need <= p.box_w && h_need <= p.box_h;
        m->u_org = u_org;
        m->v_org = finite ? (int)fv0 - 1 : 0;
        m->fast = fits ? 1 : 0;
        m->w_need = fits ? (int)w_need : 0;
        m->h_need = fits ? (int)h_need : 0;
    }
}

// The metas of eight views in one warp (QUAD / QUINT kernel): lanes 4 v .. 4 v + 3 take view
// t0 + v at the tile's four corner columns (the same arithmetic as compute_meta1 over the whole
// chunk), so one warp does in one pass what eight warps did one view each.
template <int KC, int WALK>
__device__ void compute_meta8(Meta* ring, const BPParams& p, const PTable* pt, int t0, int n,
                              int tile_i, int tile_j, int kb)
{
    const int lane = threadIdx.x & 31;
    const int t = t0 + (lane >> 2);
    const bool valid = t < n;
    const double* Pc = pt->P[valid ? t : t0];
    double P[10];
#pragma unroll
    for (int q = 0; q < 10; ++q) P[q] = Pc[q];
    const int i_corner = (lane & 1) ? min(tile_i * 16 + 16, p.Nx) - 1 : tile_i * 16;
    const int j_corner = (lane & 2) ? min(tile_j * 16 + 16, p.Ny) - 1 : tile_j * 16;
    const ColInv c = column_invariants(P, (double)i_corner, (double)j_corner, (double)kb);
    double umin = c.u, umax = c.u;
    const double va = c.v, vb = c.v + (KC - 1) * c.dv;
    double vmin = fmin(va, vb), vmax = fmax(va, vb);
#pragma unroll
    for (int o = 1; o < 4; o <<= 1) {  // within the view's four lanes
        umin = fmin(umin, __shfl_xor_sync(0xffffffffu, umin, o));
        umax = fmax(umax, __shfl_xor_sync(0xffffffffu, umax, o));
        vmin = fmin(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
        vmax = fmax(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
    }
    if (valid && (lane & 3) == 0) {  // the tile's base corner (i_corner, j_corner)
        Meta* m = &ring[t & (kMetaRing - 1)];
        const double fu = floor(c.u), fv = floor(c.v);
        m->uci = (int)fu;
        m->vci = (int)fv;
        m->ucf = (float)(c.u - fu);
        m->vcf = (float)(c.v - fv);
        m->uc = (float)c.u;
        m->vc = (float)c.v;
        m->zc = (float)c.z;
        m->p0 = (float)P[0]; m->p1 = (float)P[1]; m->p3 = (float)P[3]; m->p4 = (float)P[4];
        m->p5 = (float)P[5]; m->p7 = (float)P[7]; m->p8 = (float)P[8];
        const double fu0 = floor(umin), fu1 = floor(umax), fv0 = floor(vmin), fv1 = floor(vmax);
        const bool finite = fu0 > -1e9 && fu1 < 1e9 && fv0 > -1e9 && fv1 < 1e9;
        const int u_org = finite ? (((int)fu0 - 1) & ~3) : 0;  // 16-byte TMA origin
        constexpr int MV = WALK == 15 ? 2 : 1;  // rows below: fp32 thread floors, HI runs
        const double w_need = fu1 + 3.0 - u_org, h_need = fv1 - fv0 + 4.0 + p.pair + MV;
        const bool fits = finite && w_need <= p.box_w && h_need <= p.box_h;
        m->u_org = u_org;
        m->v_org = finite ? (int)fv0 - 1 - MV : 0;
        m->fast = fits ? 1 : 0;
        m->w_need = fits ? (int)w_need : 0;
        m->h_need = fits ? (int)h_need : 0;
    }
}

template <int KC, int P2, bool TMA, int WALK>
__global__ void __launch_bounds__(kThreads, KC >= 64 ? 2 : 3)
    bp_kernel(const __grid_constant__ BPParams p, const __grid_constant__ CUtensorMap tmap,
              const __grid_constant__ PTable pt)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // L2-friendly raster: the grid is (raster x tiles_j, chunks, bands of `raster` tile
    // columns), so consecutive CTAs walk down one band and the ~300 resident CTAs cover a
    // block of raster x ~300/raster tiles whose detector patches (all views of the launch)
    // stay in L2; a row-major raster (raster = tiles_i) spans the whole i extent and
    // re-reads every view's rows from HBM once per wave.  CTAs past the volume edge of the
    // last band exit.
    const int tile_i = (int)blockIdx.z * p.raster + (int)(blockIdx.x % (unsigned)p.raster);
    const int tile_j = (int)(blockIdx.x / (unsigned)p.raster);
    if (tile_i >= p.tiles_i) return;
    const int i = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
    const int j = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
    const bool active = i < p.Nx && j < p.Ny;
    // Columns past the volume edge shadow the last valid column (branch-free update loop);
    // they never write.
    const double di = (double)min(i, p.Nx - 1), dj = (double)min(j, p.Ny - 1);
    // this lane's tile corner for the patch boxes: lane % 4 = corner (i_lo|i_hi, j_lo|j_hi)
    const int i_corner = (lane & 1) ? min(tile_i * kTI + kTI, p.Nx) - 1 : tile_i * kTI;
    const int j_corner = (lane & 2) ? min(tile_j * kTJ + kTJ, p.Ny) - 1 : tile_j * kTJ;
    const int kb = p.kb0 + (int)blockIdx.y * KC;
    const double dkb = (double)kb;
    const int kv0 = max(p.k0 - kb, 0), kv1 = min(p.k0 + p.nk - kb, KC);
    const bool full = kv0 == 0 && kv1 == KC;

    constexpr bool X2 = WALK == 4;
    AccRegs<KC, X2> acc;
    if constexpr (X2) {
#pragma unroll
        for (int q = 0; q < KC / 2; ++q) acc.a[q] = 0ull;
    } else {
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) acc.a[kk] = 0.f;
    }
    bool overwrite = !p.accumulate;
    const int n = (int)p.n_views;

    // raw box of view t: smem + (t & 1) raw_bytes; pair patch of view t: pair0 + (t & 1) box_h P2
    float2* const pair0 = reinterpret_cast<float2*>(smem + 2 * p.raw_bytes);
    Meta* const meta = reinterpret_cast<Meta*>(pair0 + 2 * p.box_h * P2);  // ring of kMetaRing
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(meta + kMetaRing);
    const uint32_t tx_bytes = (uint32_t)(p.box_w * p.box_h * 4);
    // The tensor map must be addressed in param space (__grid_constant__): take its address
    // here, in the kernel body, never through a by-reference lambda capture (which would copy
    // it to local memory, an illegal TMA operand).
    const CUtensorMap* const tmap_ptr = &tmap;
    const PTable* const ptab = &pt;  // same rule: the lambdas must not copy the 20 KB table

    auto issue = [=](int t) {  // one thread: TMA of view t's box into raw buffer t & 1
        const Meta& m = meta[t & (kMetaRing - 1)];
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[t & 1], tx_bytes);
        tma_load_3d(smem + (t & 1) * p.raw_bytes, tmap_ptr, &mbar[t & 1], m.u_org, m.v_org - p.v0,
                    t);
    };
    auto transform = [=](int t) {  // all threads: used part of the raw box -> (a, b - a) pairs
        const Meta& m = meta[t & (kMetaRing - 1)];
        const float* r = reinterpret_cast<const float*>(smem + (t & 1) * p.raw_bytes);
        float2* q = pair0 + (t & 1) * p.box_h * P2;
        const int wp = m.w_need - 1, hn = m.h_need;
        if (p.box_w <= 32) {
            // One detector row per warp and iteration, one column per lane; b = a of lane+1.
            const float* rp = r + warp * p.box_w + lane;
            float2* qp = q + warp * P2 + lane;
            const bool in_box = lane < p.box_w, wr = lane < wp;
            const int rstep = (kThreads / 32) * p.box_w;
            for (int rr = warp; rr < hn; rr += kThreads / 32) {
                const float a = in_box ? *rp : 0.f;
                const float b = __shfl_down_sync(0xffffffffu, a, 1);
                if (wr) *qp = make_float2(a, b - a);
                rp += rstep;
                qp += (kThreads / 32) * P2;
            }
        } else {
            for (int rr = warp; rr < hn; rr += kThreads / 32) {
                const float* rrow = r + rr * p.box_w;
                for (int c0 = 0; c0 < wp; c0 += 32) {
                    const int cc = c0 + lane;
                    const float a = cc < p.box_w ? rrow[cc] : 0.f;
                    float b = __shfl_down_sync(0xffffffffu, a, 1);
                    if (lane == 31 && cc + 1 < p.box_w) b = rrow[cc + 1];
                    if (cc < wp) q[rr * P2 + cc] = make_float2(a, b - a);
                }
            }
        }
    };
    auto metas = [=](int t0) {  // all warps: boxes of views t0 .. t0+7
        if (t0 + warp < n)
            compute_meta1<KC, WALK>(meta, p, ptab->P[t0 + warp], t0 + warp, i_corner, j_corner, kb, kv0,
                          kv1);
    };

    if (TMA) {
        if (tid == 0) {
            mbar_init(&mbar[0], 1);
            mbar_init(&mbar[1], 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        metas(0);
        __syncthreads();
        if (tid == 0) {
            if (n > 0) issue(0);
            if (n > 1) issue(1);
        }
        if (n > 0) {
            mbar_wait(&mbar[0], 0);
            if (!meta[0].fast) __trap();  // the host sizes the box from a conservative bound
            transform(0);
        }
        __syncthreads();
        if (tid == 0 && n > 2) issue(2);
    }

    // first view after which the partial sums are flushed: s0 + t + 1 = 0 (mod vb)
    int next_flush = (int)(p.vb - 1 - (p.s0 % p.vb + p.vb) % p.vb);
    for (int t = 0; t < n; ++t) {
        double Pr[10];
        int u_org = 0, v_org = 0;
        if (TMA) {
            const Meta& m = meta[t & (kMetaRing - 1)];
            const double2* P2v = reinterpret_cast<const double2*>(m.P);
#pragma unroll
            for (int q = 0; q < 5; ++q) {
                const double2 d = P2v[q];
                Pr[2 * q] = d.x;
                Pr[2 * q + 1] = d.y;
            }
            u_org = m.u_org;
            v_org = m.v_org;
        } else {
#pragma unroll
            for (int q = 0; q < 10; ++q) Pr[q] = ptab->P[t][q];
        }
        const ThreadInv ti = split(column_invariants(Pr, di, dj, dkb));
        if constexpr (TMA) {
            // Next view's raw box (TMA issued two iterations ago, normally landed): rewrite it
            // into pairs row by row inside this view's update loop (one row per warp per
            // 8-slice group), the rest after.
            const bool nxt = t + 1 < n;
            int hn = 0, wp = 0;
            const float* rbase = nullptr;
            float2* qbase = nullptr;
            if (nxt) {
                mbar_wait(&mbar[(t + 1) & 1], (uint32_t)(((t + 1) >> 1) & 1));
                const Meta& mn = meta[(t + 1) & (kMetaRing - 1)];
                if (!mn.fast) __trap();  // the host sizes the box from a conservative bound
                hn = mn.h_need;
                wp = mn.w_need - 1;
                rbase = reinterpret_cast<const float*>(smem + ((t + 1) & 1) * p.raw_bytes);
                qbase = pair0 + ((t + 1) & 1) * p.box_h * P2;
            }
            const bool narrow = p.box_w <= 32;
            const bool in_box = lane < p.box_w, wr = lane < wp;
            auto row = [&](int q) {  // transform row warp + 8 q of the next view (narrow boxes)
                const int rr = warp + (kThreads / 32) * q;
                if (narrow && rr < hn) {
                    const float a = in_box ? rbase[rr * p.box_w + lane] : 0.f;
                    const float b = __shfl_down_sync(0xffffffffu, a, 1);
                    if (wr) qbase[rr * P2 + lane] = make_float2(a, b - a);
                }
            };
            const uint32_t pb = smem_u32(pair0 + (t & 1) * p.box_h * P2);
            // floor addresses of masked slices are clamped to [pb, hb] (clamp_floor): every
            // valid floor lies in box rows 1 .. box_h - 3 - pair, and the walk reads at most
            // 2 + 2 pair rows from its floor
            const uint32_t hb = pb + (uint32_t)((p.box_h - 2 - p.pair) * P2 * 8 - 8);
            if constexpr (X2) {
                if (full)
                    accumulate_view_smem_x2<KC, P2, true>(acc.a, pb, p.neg_magic, ti, u_org,
                                                          v_org, kv0, kv1, pb, hb, row);
                else
                    accumulate_view_smem_x2<KC, P2, false>(acc.a, pb, p.neg_magic, ti, u_org,
                                                           v_org, kv0, kv1, pb, hb, row);
            } else {
                if (full)
                    accumulate_view_smem<KC, P2, true, WALK>(acc.a, pb, p.neg_magic, ti, u_org,
                                                             v_org, kv0, kv1, pb, hb, row);
                else
                    accumulate_view_smem<KC, P2, false, WALK>(acc.a, pb, p.neg_magic, ti, u_org,
                                                              v_org, kv0, kv1, pb, hb, row);
            }
            if (nxt) {
                if (narrow) {
                    for (int q = KC / 8; warp + (kThreads / 32) * q < hn; ++q) row(q);
                } else {
                    transform(t + 1);
                }
            }
        } else {
            if constexpr (!X2)
                accumulate_view_global<KC, (WALK >= 2)>(acc.a, p.Q + (long)t * p.n_rows * p.Nu, p, ti, kv0,
                                             kv1);
        }
        if (t == next_flush || t == n - 1) {
            if constexpr (X2) {
                if (active) flush_x2<KC>(acc.a, p, i, j, kb, kv0, kv1, overwrite);
            } else {
                if (active) flush<KC>(acc.a, p, i, j, kb, kv0, kv1, overwrite);
            }
            overwrite = false;
            next_flush += p.vb;
        }
        if (TMA) {
            if (((t + 3) & 7) == 0) metas(t + 3);
            __syncthreads();
            if (tid == 0 && t + 3 < n) issue(t + 3);
        }
    }
}

// ---- RAW staging: the k-walk reads the TMA box itself (no pair rewrite) ---------------------
// The PAIR walk on packed fp32x2 instructions (as accumulate_view_smem_x2) with the two taps of
// each detector row read by two LDS.32 from the raw TMA box (row pitch BW floats, BW = 8 mod 32:
// conflict-free for the 8 x 4 warp footprint) instead of one LDS.64 from a rewritten
// (a, b - a) patch: the same shared-memory wavefronts per update in the walk (a warp's LDS.32
// is one 128-byte wavefront, its LDS.64 two), and the rewrite -- 17 % of the kernel's shared
// traffic, one extra pass over every box -- disappears.  b - a is formed in registers (FADD2),
// so every value is bitwise that of the rewritten patch.
__device__ __forceinline__ float lds32(uint32_t addr)
{
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}

template <int KC, int BW>
__device__ __forceinline__ void accumulate_view_raw_x2(f2x (&acc)[KC / 2], uint32_t raw_base,
                                                       uint32_t neg_magic, const ThreadInv& t,
                                                       int u_org, int v_org)
{
    constexpr uint32_t S = BW * 4;
    const uint32_t a0 = raw_base + (uint32_t)(((t.nv - v_org) * BW + (t.nu - u_org)) * 4) + neg_magic;
    const f2x dv2 = pk2(t.dv, t.dv), dvm12 = pk2(t.dvm1, t.dvm1), W2 = pk2(t.W, t.W);
    const f2x du2 = pk2(t.du, t.du);
    const f2x magic2 = pk2(8388608.0f, 8388608.0f), nmagic2 = pk2(-8388608.0f, -8388608.0f);
    f2x fv02 = pk2(t.fv0, t.fv0);
    f2x kpair = pk2(0.f, 2.f);
    const f2x four2 = pk2(4.f, 4.f);
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
        if ((kk & 7) == 0) asm volatile("mov.b64 %0, %0;" : "+l"(fv02));
        const f2x v = fma2(kpair, dv2, fv02);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(kpair) : "l"(four2));
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
        const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
        f2x h[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const f2x a = pk2(lds32(adA + r * S), lds32(adB + r * S));
            const f2x b = pk2(lds32(adA + r * S + 4), lds32(adB + r * S + 4));
            h[r] = fma2(du2, sub2(b, a), a);  // Alg. alg:subpixel lines 4-5
        }
        const f2x d01 = sub2(h[1], h[0]), d12 = sub2(h[2], h[1]);
        const f2x g = add2(fr, dvm12);
        const float eA = lo2(g) >= 0.f ? lo2(d12) : lo2(d01);
        const float eB = hi2(g) >= 0.f ? hi2(d12) : hi2(d01);
        const f2x val0 = fma2(fr, d01, h[0]);
        const f2x val1 = fma2(g, pk2(eA, eB), h[1]);
        acc[kk / 2] = fma2(W2, val0, acc[kk / 2]);  // Alg. alg:bp line 10
        acc[kk / 2 + 1] = fma2(W2, val1, acc[kk / 2 + 1]);
        // Pin the accumulation of each 8-slice group before the next group's loads: without
        // it the compiler defers the FFMA2 chains to the end of the chunk and spills the
        // pending values.
        if ((kk & 7) == 4)
            asm volatile("" : "+l"(acc[kk / 2 - 2]), "+l"(acc[kk / 2 - 1]), "+l"(acc[kk / 2]),
                         "+l"(acc[kk / 2 + 1]));
    }
}

// TRIPLE form of the RAW walk (walk 6, opt-in; needs 0.5 <= dv < 1, configs 1-4): three
// slices per floor from four detector rows, two triples (kk..kk+2, kk+3..kk+5) packed in the
// fp32x2 halves: 16 LDS.32 per 6 updates (10.7 B/update of shared memory instead of 12).  The
// first 60 slices run as ten such groups, the last 4 as one PAIR quad.  Accumulator pairs:
// acc[3 q + r] = (slice 6 q + r, slice 6 q + 3 + r) for r < 3, acc[30 + r] = (60 + r, 62 + r).
template <int KC, int BW, bool ROWS3>
__device__ __forceinline__ void accumulate_view_raw_x2_triple(f2x (&acc)[KC / 2],
                                                              uint32_t raw_base,
                                                              uint32_t neg_magic,
                                                              const ThreadInv& t, int u_org,
                                                              int v_org)
{
    static_assert(KC == 64, "ten triple groups + one pair quad");
    constexpr uint32_t S = BW * 4;
    const uint32_t a0 = raw_base + (uint32_t)(((t.nv - v_org) * BW + (t.nu - u_org)) * 4) + neg_magic;
    const f2x dv2 = pk2(t.dv, t.dv), dvm12 = pk2(t.dvm1, t.dvm1), W2 = pk2(t.W, t.W);
    const f2x du2 = pk2(t.du, t.du);
    const f2x magic2 = pk2(8388608.0f, 8388608.0f), nmagic2 = pk2(-8388608.0f, -8388608.0f);
    f2x fv02 = pk2(t.fv0, t.fv0);
#pragma unroll
    for (int q = 0; q < 10; ++q) {
        const int kk = 6 * q;
        asm volatile("mov.b64 %0, %0;" : "+l"(fv02));
        const f2x v = fma2(pk2((float)kk, (float)(kk + 3)), dv2, fv02);
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
        const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
        constexpr int NR = ROWS3 ? 3 : 4;
        f2x h[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const f2x a = pk2(lds32(adA + r * S), lds32(adB + r * S));
            const f2x b = pk2(lds32(adA + r * S + 4), lds32(adB + r * S + 4));
            h[r] = fma2(du2, sub2(b, a), a);  // Alg. alg:subpixel lines 4-5
        }
        const f2x d01 = sub2(h[1], h[0]), d12 = sub2(h[2], h[1]);
        const f2x g1 = add2(fr, dvm12);   // second slice: g1 rows past row n+1, in [-1, 1)
        const f2x e1 = pk2(lo2(g1) >= 0.f ? lo2(d12) : lo2(d01), hi2(g1) >= 0.f ? hi2(d12) : hi2(d01));
        acc[3 * q] = fma2(W2, fma2(fr, d01, h[0]), acc[3 * q]);      // line 6; Alg. alg:bp line 10
        acc[3 * q + 1] = fma2(W2, fma2(g1, e1, h[1]), acc[3 * q + 1]);
        if constexpr (ROWS3) {
            // dv < 1/2: the third slice sits g2 = g1 + dv rows past row n+1, still in rows n..n+2
            const f2x g2 = add2(g1, dv2);
            const f2x e2 = pk2(lo2(g2) >= 0.f ? lo2(d12) : lo2(d01), hi2(g2) >= 0.f ? hi2(d12) : hi2(d01));
            acc[3 * q + 2] = fma2(W2, fma2(g2, e2, h[1]), acc[3 * q + 2]);
        } else {
            const f2x d23 = sub2(h[NR - 1], h[2]);
            const f2x g2 = add2(g1, dvm12);   // third slice: g2 rows past row n+2, in [-1, 1)
            const f2x e2 = pk2(lo2(g2) >= 0.f ? lo2(d23) : lo2(d12), hi2(g2) >= 0.f ? hi2(d23) : hi2(d12));
            acc[3 * q + 2] = fma2(W2, fma2(g2, e2, h[2]), acc[3 * q + 2]);
        }
        if (q & 1)
            asm volatile("" : "+l"(acc[3 * q - 3]), "+l"(acc[3 * q - 2]), "+l"(acc[3 * q - 1]),
                         "+l"(acc[3 * q]), "+l"(acc[3 * q + 1]), "+l"(acc[3 * q + 2]));
    }
    {  // slices 60..63: one PAIR quad (slice pairs (60, 61) and (62, 63))
        const f2x v = fma2(pk2(60.f, 62.f), dv2, fv02);
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
        const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
        f2x h[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const f2x a = pk2(lds32(adA + r * S), lds32(adB + r * S));
            const f2x b = pk2(lds32(adA + r * S + 4), lds32(adB + r * S + 4));
            h[r] = fma2(du2, sub2(b, a), a);
        }
        const f2x d01 = sub2(h[1], h[0]), d12 = sub2(h[2], h[1]);
        const f2x g = add2(fr, dvm12);
        const float eA = lo2(g) >= 0.f ? lo2(d12) : lo2(d01);
        const float eB = hi2(g) >= 0.f ? hi2(d12) : hi2(d01);
        acc[30] = fma2(W2, fma2(fr, d01, h[0]), acc[30]);
        acc[31] = fma2(W2, fma2(g, pk2(eA, eB), h[1]), acc[31]);
    }
}

template <int KC>
__device__ __forceinline__ void flush_x2_triple(f2x (&acc)[KC / 2], const BPParams& p, int i,
                                                int j, int kb, bool overwrite)
{
    float* q = vol_voxel(p, kb, j, i);
    long plane = (long)p.Ny * p.Nx;
    asm volatile("mov.b64 %0, %0;" : "+l"(plane));
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) {
        int pi, half;
        if (kk < 60) {
            pi = 3 * (kk / 6) + (kk % 6) % 3;
            half = (kk % 6) / 3;
        } else {
            pi = 30 + ((kk - 60) & 1);
            half = (kk - 60) >> 1;
        }
        const float v = half ? hi2(acc[pi]) : lo2(acc[pi]);
        put_voxel(p, q, kb + kk, j, i, v, overwrite);
        q += plane;
    }
#pragma unroll
    for (int q2 = 0; q2 < KC / 2; ++q2) acc[q2] = 0ull;
}

constexpr int kRawBuf = 4;  // TMA boxes in flight / in use per CTA

template <int KC, int BW, int TRI = 0>  // 0: PAIR walk, 1: 4-row TRIPLE, 2: 3-row TRIPLE
__global__ void __launch_bounds__(kThreads, 2)
    bp_raw_kernel(const __grid_constant__ BPParams p, const __grid_constant__ CUtensorMap tmap,
                  const __grid_constant__ PTable pt)
{
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile_i = (int)blockIdx.z * p.raster + (int)(blockIdx.x % (unsigned)p.raster);
    const int tile_j = (int)(blockIdx.x / (unsigned)p.raster);
    if (tile_i >= p.tiles_i) return;
    const int i = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
    const int j = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
    const int ic = min(i, p.Nx - 1), jc = min(j, p.Ny - 1);
    const int i_corner = (lane & 1) ? min(tile_i * kTI + kTI, p.Nx) - 1 : tile_i * kTI;
    const int j_corner = (lane & 2) ? min(tile_j * kTJ + kTJ, p.Ny) - 1 : tile_j * kTJ;
    const int kb = p.kb0 + (int)blockIdx.y * KC;
    if (kb < p.k0 || kb + KC > p.k0 + p.nk) __trap();  // whole chunks only (host)
    const int kv0 = 0, kv1 = KC;

    f2x acc[KC / 2];
#pragma unroll
    for (int q = 0; q < KC / 2; ++q) acc[q] = 0ull;
    const int n = (int)p.n_views;

    // shared memory: [raw box x kRawBuf | meta ring | mbarriers]; the box of view t is at
    // raw + (t % kRawBuf) raw_bytes.  Whole chunks only (the host sends partial ones to the
    // pair walk): every slice's rows lie inside the box.
    unsigned char* const raw = smem;
    Meta* const meta = reinterpret_cast<Meta*>(raw + kRawBuf * p.raw_bytes);
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(meta + kMetaRing);
    const uint32_t tx_bytes = (uint32_t)(BW * p.box_h * 4);
    const CUtensorMap* const tmap_ptr = &tmap;
    const PTable* const ptab = &pt;
    const uint32_t raw0 = smem_u32(raw);

    auto issue = [=](int t) {  // one thread: TMA of view t's box into raw buffer t % kRawBuf
        const Meta& m = meta[t & (kMetaRing - 1)];
        if (!m.fast) __trap();  // the host sizes the box from a conservative bound
        const int b = t % kRawBuf;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[b], tx_bytes);
        tma_load_3d(raw + b * p.raw_bytes, tmap_ptr, &mbar[b], m.u_org, m.v_org - p.v0, t);
    };
    auto metas = [=](int t0) {  // all warps: boxes of views t0 .. t0+7
        if (t0 + warp < n)
            compute_meta1<KC, 2>(meta, p, ptab->P[t0 + warp], t0 + warp, i_corner, j_corner, kb,
                                 kv0, kv1);
    };

    if (tid == 0) {
        for (int b = 0; b < kRawBuf; ++b) mbar_init(&mbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    metas(0);
    __syncthreads();
    if (tid == 0)
        for (int t = 0; t < kRawBuf && t < n; ++t) issue(t);

    // first view after which the partial sums are flushed: s0 + t + 1 = 0 (mod vb); later
    // flushes every vb views.  Derived from t (no loop-carried state next to the accumulators).
    const int first_flush = (int)(p.vb - 1 - (p.s0 % p.vb + p.vb) % p.vb);
    for (int t = 0; t < n; ++t) {
        const Meta& m = meta[t & (kMetaRing - 1)];
        const int u_org = m.u_org, v_org = m.v_org;
        // P_s straight from the constant bank (uniform per warp): no register copy of the 10
        // doubles next to the 64 accumulators
        // the column's coordinates are converted per view from laundered integers: hoisted out
        // of the loop as doubles they would be spilled next to the 64 accumulators
        int ic_ = ic, jc_ = jc, kb_ = kb;
        asm volatile("" : "+r"(ic_), "+r"(jc_), "+r"(kb_));
        const ThreadInv ti =
            split(column_invariants(ptab->P[t], (double)ic_, (double)jc_, (double)kb_));
        const int b = t % kRawBuf;
        mbar_wait(&mbar[b], (uint32_t)((t / kRawBuf) & 1));
        const uint32_t rb = raw0 + (uint32_t)(b * p.raw_bytes);
        if constexpr (TRI != 0)
            accumulate_view_raw_x2_triple<KC, BW, TRI == 2>(acc, rb, p.neg_magic, ti, u_org, v_org);
        else
            accumulate_view_raw_x2<KC, BW>(acc, rb, p.neg_magic, ti, u_org, v_org);
        if ((t >= first_flush && (t - first_flush) % p.vb == 0) || t == n - 1) {
            // recomputed here rather than kept live across the view loop
            const int fi = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
            const int fj = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
            const bool ow = !p.accumulate && t <= first_flush;
            if (fi < p.Nx && fj < p.Ny) {
                if constexpr (TRI != 0)
                    flush_x2_triple<KC>(acc, p, fi, fj, kb, ow);
                else
                    flush_x2<KC>(acc, p, fi, fj, kb, 0, KC, ow);
            }
        }
        // boxes of views t+kRawBuf+1 .. +8 (the ring slots of views <= t+kRawBuf are in use)
        if (((t + kRawBuf + 1) & 7) == 0) metas(t + kRawBuf + 1);
        __syncthreads();  // buffer b read out by every warp
        if (tid == 0 && t + kRawBuf < n) issue(t + kRawBuf);
    }
}

// ----------------------------------------------------------------------------------------
// TMEM-accumulator form of the TRIPLE RAW walks (walks 9 / 10 = 6 / 7 with the accumulators in
// tensor memory).  The register-resident walk holds 64 fp32 accumulators per thread (127
// registers, 2 CTAs = 16 warps per SM) and its measured limit is latency: 64.5 % issue, the
// top stall "wait" (fixed-latency dependencies; profiles/r2/ncu_bp_kernel_full_r2b.txt).  Here
// each thread's 64 partial sums live in TMEM (warp w owns lanes 32 (w % 4) .. +31 and 64
// columns at 64 (w / 4) of its CTA's 128-column allocation) and a view is walked in three
// sub-walks of 24 / 24 / 16 slices: tcgen05.ld the sub-walk's accumulators, the same FFMA2
// arithmetic in registers, tcgen05.st them back.  Freed registers buy a third CTA per SM
// (24 warps, 80 registers).  TMEM traffic is 8 B per update (4 B read, 4 B written) against a
// 64 B/clk per SM read port (B300_MICROARCH.md: TMEM), i.e. <= 55 % of it at 2,500 GUPS.  The
// order of every floating-point operation is the register walk's, so the result is bitwise
// that of walks 6 / 7 (and their partial-chunk companions 3 / 8).
__device__ __forceinline__ void tm_ld16(uint32_t taddr, f2x (&a)[8])
{
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int m = 0; m < 8; ++m) a[m] = pk2(__uint_as_float(r[2 * m]), __uint_as_float(r[2 * m + 1]));
}
__device__ __forceinline__ void tm_ld8(uint32_t taddr, f2x (&a)[4])
{
    uint32_t r[8];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7])
        : "r"(taddr));
#pragma unroll
    for (int m = 0; m < 4; ++m) a[m] = pk2(__uint_as_float(r[2 * m]), __uint_as_float(r[2 * m + 1]));
}
__device__ __forceinline__ void tm_st16(uint32_t taddr, const f2x (&a)[8])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16};" ::"r"(taddr),
        "f"(lo2(a[0])), "f"(hi2(a[0])), "f"(lo2(a[1])), "f"(hi2(a[1])), "f"(lo2(a[2])),
        "f"(hi2(a[2])), "f"(lo2(a[3])), "f"(hi2(a[3])), "f"(lo2(a[4])), "f"(hi2(a[4])),
        "f"(lo2(a[5])), "f"(hi2(a[5])), "f"(lo2(a[6])), "f"(hi2(a[6])), "f"(lo2(a[7])),
        "f"(hi2(a[7])));
}
__device__ __forceinline__ void tm_st8(uint32_t taddr, const f2x (&a)[4])
{
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
        "f"(lo2(a[0])), "f"(hi2(a[0])), "f"(lo2(a[1])), "f"(hi2(a[1])), "f"(lo2(a[2])),
        "f"(hi2(a[2])), "f"(lo2(a[3])), "f"(hi2(a[3])));
}
__device__ __forceinline__ void tm_ld4(uint32_t taddr, f2x (&a)[2])
{
    uint32_t r[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(taddr));
    a[0] = pk2(__uint_as_float(r[0]), __uint_as_float(r[1]));
    a[1] = pk2(__uint_as_float(r[2]), __uint_as_float(r[3]));
}
__device__ __forceinline__ void tm_st4(uint32_t taddr, const f2x (&a)[2])
{
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr),
                 "f"(lo2(a[0])), "f"(hi2(a[0])), "f"(lo2(a[1])), "f"(hi2(a[1])));
}
__device__ __forceinline__ void tm_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tm_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// (c >= 0 ? a : b) per fp32x2 half (PTX slct: one FSEL per half instead of two predicated moves)
__device__ __forceinline__ float slct(float a, float b, float c)
{
    float d;
    asm("slct.f32.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ f2x sel2(f2x a, f2x b, f2x c)
{
    return pk2(slct(lo2(a), lo2(b), lo2(c)), slct(hi2(a), hi2(b), hi2(c)));
}

// Triple groups q = Q0 .. Q0+NQ-1 of accumulate_view_raw_x2_triple (and its closing PAIR quad
// when QUAD) on the accumulator pairs acc[3 (q - Q0) + r] (the quad: acc[3 NQ], acc[3 NQ + 1]).
// Same operations in the same order, so bitwise the same sums.
template <int BW, bool ROWS3, int Q0, int NQ, bool QUAD>
__device__ __forceinline__ void triple_groups(f2x (&acc)[3 * NQ + (QUAD ? 2 : 0)], uint32_t a0,
                                              const ThreadInv& t)
{
    constexpr uint32_t S = BW * 4;
    const f2x dv2 = pk2(t.dv, t.dv), dvm12 = pk2(t.dvm1, t.dvm1), W2 = pk2(t.W, t.W);
    const f2x du2 = pk2(t.du, t.du);
    const f2x magic2 = pk2(8388608.0f, 8388608.0f), nmagic2 = pk2(-8388608.0f, -8388608.0f);
    const f2x fv02 = pk2(t.fv0, t.fv0);
    // (kk, kk + 3) in a register stepped by FADD2 (exact small integers): one instruction per
    // group instead of two uniform moves of the constants
    f2x kvec = pk2((float)(6 * Q0), (float)(6 * Q0 + 3));
    asm volatile("mov.b64 %0, %0;" : "+l"(kvec));
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {
        const f2x v = fma2(kvec, dv2, fv02);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(kvec) : "l"(pk2(6.f, 6.f)));
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
        const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
        constexpr int NR = ROWS3 ? 3 : 4;
        f2x h[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const f2x a = pk2(lds32(adA + r * S), lds32(adB + r * S));
            const f2x b = pk2(lds32(adA + r * S + 4), lds32(adB + r * S + 4));
            h[r] = fma2(du2, sub2(b, a), a);  // Alg. alg:subpixel lines 4-5
        }
        const f2x d01 = sub2(h[1], h[0]), d12 = sub2(h[2], h[1]);
        const f2x g1 = add2(fr, dvm12);
        const f2x e1 = sel2(d12, d01, g1);
        acc[3 * qq] = fma2(W2, fma2(fr, d01, h[0]), acc[3 * qq]);  // line 6; Alg. alg:bp line 10
        acc[3 * qq + 1] = fma2(W2, fma2(g1, e1, h[1]), acc[3 * qq + 1]);
        if constexpr (ROWS3) {
            const f2x g2 = add2(g1, dv2);
            acc[3 * qq + 2] = fma2(W2, fma2(g2, sel2(d12, d01, g2), h[1]), acc[3 * qq + 2]);
        } else {
            const f2x d23 = sub2(h[NR - 1], h[2]);
            const f2x g2 = add2(g1, dvm12);
            acc[3 * qq + 2] = fma2(W2, fma2(g2, sel2(d23, d12, g2), h[2]), acc[3 * qq + 2]);
        }
    }
    if constexpr (QUAD) {  // slices 60..63
        const f2x v = fma2(pk2(60.f, 62.f), dv2, fv02);
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
        const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
        f2x h[3];
#pragma unroll
        for (int r = 0; r < 3; ++r) {
            const f2x a = pk2(lds32(adA + r * S), lds32(adB + r * S));
            const f2x b = pk2(lds32(adA + r * S + 4), lds32(adB + r * S + 4));
            h[r] = fma2(du2, sub2(b, a), a);
        }
        const f2x d01 = sub2(h[1], h[0]), d12 = sub2(h[2], h[1]);
        const f2x g = add2(fr, dvm12);
        acc[3 * NQ] = fma2(W2, fma2(fr, d01, h[0]), acc[3 * NQ]);
        acc[3 * NQ + 1] = fma2(W2, fma2(g, sel2(d12, d01, g), h[1]), acc[3 * NQ + 1]);
    }
}

// The 64 accumulators of one thread: pair m = columns 2m, 2m + 1.  SUB = 4: sub-walks of four
// groups (pairs 0..11, 12..23) and the rest (24..31); SUB = 2: five sub-walks of two groups
// (pairs 0..5, .., 18..23) and the rest (24..31) -- fewer live accumulators, for 4 CTAs / SM.
template <int BW, bool ROWS3, int Q0, int NQ>
__device__ __forceinline__ void tmem_sub(uint32_t tacc, uint32_t a0, const ThreadInv& t)
{
    constexpr int NP = 3 * NQ;  // 12 or 6 pairs = 24 or 12 columns
    f2x acc[NP];
    if constexpr (NP == 12) {
        f2x x[8], y[4];
        tm_ld16(tacc + 6 * Q0, x);
        tm_ld8(tacc + 6 * Q0 + 16, y);
        tm_wait_ld();
#pragma unroll
        for (int m = 0; m < 8; ++m) acc[m] = x[m];
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[8 + m] = y[m];
    } else {
        f2x x[4], y[2];
        tm_ld8(tacc + 6 * Q0, x);
        tm_ld4(tacc + 6 * Q0 + 8, y);
        tm_wait_ld();
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[m] = x[m];
#pragma unroll
        for (int m = 0; m < 2; ++m) acc[4 + m] = y[m];
    }
    triple_groups<BW, ROWS3, Q0, NQ, false>(acc, a0, t);
    if constexpr (NP == 12) {
        f2x x[8], y[4];
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = acc[m];
#pragma unroll
        for (int m = 0; m < 4; ++m) y[m] = acc[8 + m];
        tm_st16(tacc + 6 * Q0, x);
        tm_st8(tacc + 6 * Q0 + 16, y);
    } else {
        f2x x[4], y[2];
#pragma unroll
        for (int m = 0; m < 4; ++m) x[m] = acc[m];
#pragma unroll
        for (int m = 0; m < 2; ++m) y[m] = acc[4 + m];
        tm_st8(tacc + 6 * Q0, x);
        tm_st4(tacc + 6 * Q0 + 8, y);
    }
}

template <int BW, bool ROWS3, int SUB>
__device__ __forceinline__ void walk_view_tmem(uint32_t tacc, uint32_t a0, const ThreadInv& t)
{
    tm_wait_st();  // the previous view's stores of these columns
    if constexpr (SUB == 4) {
        tmem_sub<BW, ROWS3, 0, 4>(tacc, a0, t);
        tmem_sub<BW, ROWS3, 4, 4>(tacc, a0, t);
    } else {
        tmem_sub<BW, ROWS3, 0, 2>(tacc, a0, t);
        tmem_sub<BW, ROWS3, 2, 2>(tacc, a0, t);
        tmem_sub<BW, ROWS3, 4, 2>(tacc, a0, t);
        tmem_sub<BW, ROWS3, 6, 2>(tacc, a0, t);
    }
    {
        f2x acc[8];
        tm_ld16(tacc + 48, acc);
        tm_wait_ld();
        triple_groups<BW, ROWS3, 8, 2, true>(acc, a0, t);
        tm_st16(tacc + 48, acc);
    }
}

// Flush: every slice's partial sum to the volume (mapping of flush_x2_triple), zeros back.
template <int KC, bool RED = true>
__device__ __forceinline__ void flush_tmem_triple_r(uint32_t tacc, const BPParams& p, int i, int j,
                                                  int kb, bool overwrite, bool inside)
{
    tm_wait_st();
    float* q0 = vol_voxel(p, kb, j, i);
    const long plane = (long)p.Ny * p.Nx;
    const f2x zero[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int part = 0; part < 4; ++part) {  // pairs 8 part .. 8 part + 7
        f2x a[8];
        tm_ld16(tacc + 16 * part, a);
        tm_wait_ld();
        if (inside) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int pi = 8 * part + m;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int kk = pi < 30 ? 6 * (pi / 3) + 3 * half + pi % 3
                                           : 60 + 2 * half + (pi - 30);
                    const float v = half ? hi2(a[m]) : lo2(a[m]);
                    put_voxel<RED>(p, q0 + kk * plane, kb + kk, j, i, v, overwrite);
                }
            }
        }
        tm_st16(tacc + 16 * part, zero);
    }
}

template <int KC>
__device__ __forceinline__ void flush_tmem_triple(uint32_t tacc, const BPParams& p, int i, int j,
                                                  int kb, bool overwrite, bool inside)
{
    flush_tmem_triple_r<KC, true>(tacc, p, i, j, kb, overwrite, inside);
}

// TRI 1: 4-row TRIPLE (walk 9), 2: 3-row TRIPLE (walk 10).  Three CTAs per SM (80 registers,
// 3 x 128 TMEM columns).  Measured alternatives (B200, config 4 / config 5 slab, 256 views):
// four CTAs per SM with 12-slice sub-walks (64 registers) 2078 / 2304 GUPS vs 2089 / 2311;
// no CTA barrier per view (the last warp out of a buffer refills it) 1908 / 2062 -- warps drift
// apart and the refill lands late (28.7 % long-scoreboard stalls on the box barrier).
template <int BW, int TRI, int MINB>
__global__ void __launch_bounds__(kThreads, MINB)
    bp_tmem_kernel(const __grid_constant__ BPParams p, const __grid_constant__ CUtensorMap tmap,
                   const __grid_constant__ PTable pt)
{
    constexpr int KC = 64;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile_i = (int)blockIdx.z * p.raster + (int)(blockIdx.x % (unsigned)p.raster);
    const int tile_j = (int)(blockIdx.x / (unsigned)p.raster);
    if (tile_i >= p.tiles_i) return;
    const int i = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
    const int j = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
    const int ic = min(i, p.Nx - 1), jc = min(j, p.Ny - 1);
    const int i_corner = (lane & 1) ? min(tile_i * kTI + kTI, p.Nx) - 1 : tile_i * kTI;
    const int j_corner = (lane & 2) ? min(tile_j * kTJ + kTJ, p.Ny) - 1 : tile_j * kTJ;
    const int kb = p.kb0 + (int)blockIdx.y * KC;
    if (kb < p.k0 || kb + KC > p.k0 + p.nk) __trap();  // whole chunks only (host)
    const int n = (int)p.n_views;

    unsigned char* const raw = smem;
    Meta* const meta = reinterpret_cast<Meta*>(raw + kRawBuf * p.raw_bytes);
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(meta + kMetaRing);
    uint32_t* const tslot = reinterpret_cast<uint32_t*>(mbar + kRawBuf);
    const uint32_t tx_bytes = (uint32_t)(BW * p.box_h * 4);
    const CUtensorMap* const tmap_ptr = &tmap;
    const PTable* const ptab = &pt;
    const uint32_t raw0 = smem_u32(raw);

    auto issue = [=](int t) {
        const Meta& m = meta[t & (kMetaRing - 1)];
        if (!m.fast) __trap();
        const int b = t % kRawBuf;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[b], tx_bytes);
        tma_load_3d(raw + b * p.raw_bytes, tmap_ptr, &mbar[b], m.u_org, m.v_org - p.v0, t);
    };
    auto metas = [=](int t0) {
        if (t0 + warp < n)
            compute_meta1<KC, 2>(meta, p, ptab->P[t0 + warp], t0 + warp, i_corner, j_corner, kb,
                                 0, KC);
    };

    if (warp == 0) {  // 128 TMEM columns: 64 per warp pair (w, w + 4) sharing a lane quarter
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                         smem_u32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int b = 0; b < kRawBuf; ++b) mbar_init(&mbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    metas(0);
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tacc = *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    if (tid == 0)
        for (int t = 0; t < kRawBuf && t < n; ++t) issue(t);
    {
        const f2x zero[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int part = 0; part < 4; ++part) tm_st16(tacc + 16 * part, zero);
    }

    // the host always sums in 128-view batches (p.vb): a power of two here, so the flush test is
    // a mask, not a division
    constexpr int VB = 128;
    if (p.vb != VB) __trap();
    const int first_flush = (int)(VB - 1 - (p.s0 % VB + VB) % VB);
    // the column's coordinates as doubles, hoisted (80 registers leave room for them)
    const double di = ic, dj = jc, dk = kb;
    for (int t = 0; t < n; ++t) {
        const ThreadInv ti = split(column_invariants(ptab->P[t], di, dj, dk));
        const int b = t % kRawBuf;
        mbar_wait(&mbar[b], (uint32_t)((t / kRawBuf) & 1));
        const Meta& m = meta[t & (kMetaRing - 1)];
        const int u_org = m.u_org, v_org = m.v_org;
        const uint32_t rb = raw0 + (uint32_t)(b * p.raw_bytes);
        const uint32_t a0 =
            rb + (uint32_t)(((ti.nv - v_org) * BW + (ti.nu - u_org)) * 4) + p.neg_magic;
        walk_view_tmem<BW, TRI == 2, MINB == 3 ? 4 : 2>(tacc, a0, ti);
        if ((t >= first_flush && ((t - first_flush) & (VB - 1)) == 0) || t == n - 1) {
            const int fi = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
            const int fj = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
            const bool ow = !p.accumulate && t <= first_flush;
            flush_tmem_triple<KC>(tacc, p, fi, fj, kb, ow, fi < p.Nx && fj < p.Ny);
        }
        if (((t + kRawBuf + 1) & 7) == 0) metas(t + kRawBuf + 1);
        __syncthreads();  // buffer b read out by every warp
        if (tid == 0 && t + kRawBuf < n) issue(t + kRawBuf);
    }
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tslot)
                     : "memory");
}

// Two views per step (walks 11 / 12 = 9 / 10 stepping two views at a time): every sub-walk
// loads its accumulators from TMEM once, adds view t's and then view t + 1's updates (the same
// per-voxel order, so bitwise the same sums) and stores them once.  The two views' tap loads and
// interpolations are independent, which doubles the work the scheduler can interleave, and the
// per-step costs (TMEM traffic, box barrier, CTA barrier, TMA issue) are shared by two views.
// (A one-view step -- view 0 when the first flush falls on it, or the last view -- walks the
// view a second time with weight 0, which adds +0 to each sum.)  Six boxes in flight (two steps
// of prefetch).  A step ends on every flush point of the two-level sum.
// Measured (B200, 256 views; config 4 / config 5 slab): 2220 / 2480 GUPS vs 2133 / 2345 for
// one view per step (walks 9 / 10); a generic V-view form was slower (V = 2: 2161 / 2378,
// V = 3: 2168 / 2407) -- its per-view padding and buffer bookkeeping cost more than V = 3 saves.
constexpr int kRawBuf2 = 6;

template <int BW, bool ROWS3, int Q0, int NQ>
__device__ __forceinline__ void tmem_sub2(uint32_t tacc, uint32_t a0, const ThreadInv& t,
                                          uint32_t a1, const ThreadInv& u)
{
    constexpr int NP = 3 * NQ;  // 6 pairs = 12 columns
    static_assert(NP == 6, "two-group sub-walks");
    f2x acc[NP];
    {
        f2x x[4], y[2];
        tm_ld8(tacc + 6 * Q0, x);
        tm_ld4(tacc + 6 * Q0 + 8, y);
        tm_wait_ld();
#pragma unroll
        for (int m = 0; m < 4; ++m) acc[m] = x[m];
#pragma unroll
        for (int m = 0; m < 2; ++m) acc[4 + m] = y[m];
    }
    triple_groups<BW, ROWS3, Q0, NQ, false>(acc, a0, t);
    triple_groups<BW, ROWS3, Q0, NQ, false>(acc, a1, u);
    {
        f2x x[4], y[2];
#pragma unroll
        for (int m = 0; m < 4; ++m) x[m] = acc[m];
#pragma unroll
        for (int m = 0; m < 2; ++m) y[m] = acc[4 + m];
        tm_st8(tacc + 6 * Q0, x);
        tm_st4(tacc + 6 * Q0 + 8, y);
    }
}

template <int BW, bool ROWS3>
__device__ __forceinline__ void walk_views_tmem2(uint32_t tacc, uint32_t a0, const ThreadInv& t,
                                                 uint32_t a1, const ThreadInv& u)
{
    tm_wait_st();
    tmem_sub2<BW, ROWS3, 0, 2>(tacc, a0, t, a1, u);
    tmem_sub2<BW, ROWS3, 2, 2>(tacc, a0, t, a1, u);
    tmem_sub2<BW, ROWS3, 4, 2>(tacc, a0, t, a1, u);
    tmem_sub2<BW, ROWS3, 6, 2>(tacc, a0, t, a1, u);
    {
        f2x acc[8];
        tm_ld16(tacc + 48, acc);
        tm_wait_ld();
        triple_groups<BW, ROWS3, 8, 2, true>(acc, a0, t);
        triple_groups<BW, ROWS3, 8, 2, true>(acc, a1, u);
        tm_st16(tacc + 48, acc);
    }
}

template <int BW, int TRI, bool RED = false>
__global__ void __launch_bounds__(kThreads, 3)
    bp_tmem2_kernel(const __grid_constant__ BPParams p, const __grid_constant__ CUtensorMap tmap,
                    const __grid_constant__ PTable pt)
{
    constexpr int KC = 64, NB = kRawBuf2, VB = 128;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile_i = (int)blockIdx.z * p.raster + (int)(blockIdx.x % (unsigned)p.raster);
    const int tile_j = (int)(blockIdx.x / (unsigned)p.raster);
    if (tile_i >= p.tiles_i) return;
    const int i = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
    const int j = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
    const int ic = min(i, p.Nx - 1), jc = min(j, p.Ny - 1);
    const int i_corner = (lane & 1) ? min(tile_i * kTI + kTI, p.Nx) - 1 : tile_i * kTI;
    const int j_corner = (lane & 2) ? min(tile_j * kTJ + kTJ, p.Ny) - 1 : tile_j * kTJ;
    const int kb = p.kb0 + (int)blockIdx.y * KC;
    if (kb < p.k0 || kb + KC > p.k0 + p.nk) __trap();  // whole chunks only (host)
    if (p.vb != VB) __trap();
    const int n = (int)p.n_views;

    unsigned char* const raw = smem;
    Meta* const meta = reinterpret_cast<Meta*>(raw + NB * p.raw_bytes);
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(meta + kMetaRing);
    uint32_t* const tslot = reinterpret_cast<uint32_t*>(mbar + NB);
    const uint32_t tx_bytes = (uint32_t)(BW * p.box_h * 4);
    const CUtensorMap* const tmap_ptr = &tmap;
    const PTable* const ptab = &pt;
    const uint32_t raw0 = smem_u32(raw);

    auto issue = [=](int t) {
        const Meta& m = meta[t & (kMetaRing - 1)];
        if (!m.fast) __trap();
        const int b = t % NB;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[b], tx_bytes);
        tma_load_3d(raw + b * p.raw_bytes, tmap_ptr, &mbar[b], m.u_org, m.v_org - p.v0, t);
    };
    auto metas = [=](int t0) {
        if (t0 + warp < n)
            compute_meta1<KC, 2>(meta, p, ptab->P[t0 + warp], t0 + warp, i_corner, j_corner, kb,
                                 0, KC);
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                         smem_u32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) mbar_init(&mbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    metas(0);
    int meta_next = 8;  // views with boxes computed: 0 .. meta_next - 1
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tacc = *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    if (tid == 0)
        for (int t = 0; t < NB && t < n; ++t) issue(t);
    {
        const f2x zero[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int part = 0; part < 4; ++part) tm_st16(tacc + 16 * part, zero);
    }

    const int first_flush = (int)(VB - 1 - (p.s0 % VB + VB) % VB);
    const double di = ic, dj = jc, dk = kb;
    const uint32_t nm = p.neg_magic;
    for (int t = 0; t < n;) {
        const bool two = t + 1 < n && !(t == 0 && (first_flush & 1) == 0);
        const int te = two ? t + 1 : t;
        const ThreadInv ti = split(column_invariants(ptab->P[t], di, dj, dk));
        ThreadInv tu = split(column_invariants(ptab->P[te], di, dj, dk));
        if (!two) tu.W = 0.f;
        mbar_wait(&mbar[t % NB], (uint32_t)((t / NB) & 1));
        if (two) mbar_wait(&mbar[te % NB], (uint32_t)((te / NB) & 1));
        const Meta& m0 = meta[t & (kMetaRing - 1)];
        const Meta& m1 = meta[te & (kMetaRing - 1)];
        const uint32_t a0 = raw0 + (uint32_t)((t % NB) * p.raw_bytes) +
                            (uint32_t)(((ti.nv - m0.v_org) * BW + (ti.nu - m0.u_org)) * 4) + nm;
        const uint32_t a1 = raw0 + (uint32_t)((te % NB) * p.raw_bytes) +
                            (uint32_t)(((tu.nv - m1.v_org) * BW + (tu.nu - m1.u_org)) * 4) + nm;
        walk_views_tmem2<BW, TRI == 2>(tacc, a0, ti, a1, tu);
        if ((te >= first_flush && ((te - first_flush) & (VB - 1)) == 0) || te == n - 1) {
            const int fi = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
            const int fj = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
            const bool ow = !p.accumulate && te <= first_flush;
            flush_tmem_triple_r<KC, RED>(tacc, p, fi, fj, kb, ow, fi < p.Nx && fj < p.Ny);
        }
        if (te + NB >= meta_next && meta_next < n) {  // boxes of the next eight views
            metas(meta_next);
            meta_next += 8;
        }
        __syncthreads();  // the step's buffers read out by every warp; new boxes written
        if (tid == 0)
            for (int v = t + NB; v <= te + NB; ++v)
                if (v < n) issue(v);
        t = te + 1;
    }
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tslot)
                     : "memory");
}

// ---------------------------------------------------------------------------------------------
// QUAD walk (walk 13, the default where 0.5 <= dv/dk < 1, configs 1-4): runs of four slices
// around a base slice b whose floor n = floor(v_b) serves all four.  Slice b + j sits at
// p = f_v + j dv from row n; for j = -1, 0, 1, 2 it lies within one row of row n + r_j
// (r = 0, 0, 1, 2): g_j = p - r_j is in [-1, 1) exactly when 0.5 <= dv <= 1 (the TRIPLE
// walk's condition), so every slice is Alg. alg:subpixel on the pair of rows around n + r_j,
// written from that row (h + g (g >= 0 ? h+ - h : h - h-)).  Five rows n-1 .. n+3 feed four
// slices: 10 LDS.32 per 4 updates and half, 2.5 per update (TRIPLE 2.67, PAIR 3), and 30 FP32x2
// + 12 selects + 2 IMAD per 8 updates (TRIPLE: 50 instructions per 6).  The walk is bounded by
// shared-memory wavefronts (LSU pipe 71 % for TRIPLE, r2x capture), so the 6 % fewer
// wavefronts and 4 % fewer instructions go straight to the rate.  The two FP32x2 halves carry
// the runs b = 8q + 1 (slices 8q .. 8q+3) and 8q + 5 (8q+4 .. 8q+7): eight groups tile the
// 64-slice chunk with no tail.  Row n-1 stays inside the staged box (its origin is
// floor(v_min) - 1, compute_meta1), row n+3 too (floor(v_63) + 2 >= floor(v_61) + 3).
// Partial chunks (slab ends inside a chunk) run the same walk over all 64 slices with the box of
// the whole chunk and write back only the slab's slices, so every slab split is bitwise one
// launch without a companion walk.
// The QUAD kernel's per-(column, view) invariants in fp32 from the tile corner's fp64 values
// (Meta, compute_meta1<.., 13>): with the column's offsets di, dj < 16 from the corner,
// x = x_c + dx, z = z_c + dz and u = x / z = u_c + (dx - u_c dz) / z, the correction a few
// pixels in size, so its fp32 rounding (~1e-6 px) stays far below the tolerance while x = u z
// itself (~1e6) would cancel (SURVEY c-N1).  Same for v(kb).  About 20 fp32 instructions per
// view instead of 7 DFMA, an fp64 reciprocal, 4 DMUL and 8 conversions (round 2: the per-view
// invariants were a fifth of the two-view step's instructions).
__device__ __forceinline__ float rcp_approx(float x)
{
    float r;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}
__device__ __forceinline__ ThreadInv quad_inv(const Meta& m, float fdi, float fdj)
{
    ThreadInv t;
    const float dx = fmaf(m.p0, fdi, m.p1 * fdj);
    const float dy = fmaf(m.p3, fdi, m.p4 * fdj);
    const float dz = fmaf(m.p7, fdi, m.p8 * fdj);
    const float f = rcp_approx(m.zc + dz);
    const f2x s2 = pk2(fmaf(fmaf(-m.uc, dz, dx), f, m.ucf), fmaf(fmaf(-m.vc, dz, dy), f, m.vcf));
    // floor by the round-down magic add of 1.5 * 2^23 (|s| < 2^22): bits - 0x4B400000 = floor(s)
    const f2x t2 = add2_rd(s2, pk2(12582912.0f, 12582912.0f));
    const f2x fr = sub2(s2, add2(t2, pk2(-12582912.0f, -12582912.0f)));
    t.nu = m.uci + (int)(__float_as_uint(lo2(t2)) - 0x4B400000u);
    t.nv = m.vci + (int)(__float_as_uint(hi2(t2)) - 0x4B400000u);
    t.du = lo2(fr);
    t.fv0 = hi2(fr);
    t.dv = m.p5 * f;
    t.dvm1 = t.dv - 1.f;
    t.W = f * f;
    t.dvi = 0;  // the QUAD / QUINT walks need dv < 1
    t.dvf = t.dv;
    return t;
}

// IFDK_BOUNDS_CHECK builds (tools/gpu_bounds.sh; compute-sanitizer is not available on the
// GPU pool): every tap the QUAD / QUINT walks read must lie in its staged box -- row below the
// box height, the column and its right neighbour inside the row -- or the kernel traps.
__device__ __forceinline__ void check_tap(uint32_t addr, uint32_t blo, int bw, int bh)
{
#ifdef IFDK_BOUNDS_CHECK
    const int idx = (int)(addr - blo) >> 2;
    if (addr < blo || idx / bw >= bh || idx % bw > bw - 2) __trap();
#endif
}

template <int BW, int Q0, int NQ>
__device__ __forceinline__ void quad_groups(f2x (&acc)[4 * NQ], uint32_t a0, const ThreadInv& t,
                                            uint32_t blo = 0, int bh = 0)
{
    constexpr uint32_t S = BW * 4;
    const f2x dv2 = pk2(t.dv, t.dv), dvm12 = pk2(t.dvm1, t.dvm1), W2 = pk2(t.W, t.W);
    const f2x du2 = pk2(t.du, t.du);
    const f2x magic2 = pk2(8388608.0f, 8388608.0f), nmagic2 = pk2(-8388608.0f, -8388608.0f);
    const f2x fv02 = pk2(t.fv0, t.fv0);
    f2x kvec = pk2((float)(8 * Q0 + 1), (float)(8 * Q0 + 5));  // the two runs' base slices
    asm volatile("mov.b64 %0, %0;" : "+l"(kvec));
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {
        const f2x v = fma2(kvec, dv2, fv02);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(kvec) : "l"(pk2(8.f, 8.f)));
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
        const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
        f2x h[5];  // rows n-1 .. n+3
#pragma unroll
        for (int r = 0; r < 5; ++r) {
            check_tap(adA + (r - 1) * S, blo, BW, bh);
            check_tap(adB + (r - 1) * S, blo, BW, bh);
            const f2x a = pk2(lds32(adA + (r - 1) * S), lds32(adB + (r - 1) * S));
            const f2x b = pk2(lds32(adA + (r - 1) * S + 4), lds32(adB + (r - 1) * S + 4));
            h[r] = fma2(du2, sub2(b, a), a);  // Alg. alg:subpixel lines 4-5
        }
        f2x d[4];
#pragma unroll
        for (int r = 0; r < 4; ++r) d[r] = sub2(h[r + 1], h[r]);
        const f2x gm = sub2(fr, dv2);       // slice b - 1 from row n
        const f2x g1 = add2(fr, dvm12);     // slice b + 1 from row n + 1
        const f2x g2 = add2(g1, dvm12);     // slice b + 2 from row n + 2
        acc[4 * qq] = fma2(W2, fma2(gm, sel2(d[1], d[0], gm), h[1]), acc[4 * qq]);  // line 6;
        acc[4 * qq + 1] = fma2(W2, fma2(fr, d[1], h[1]), acc[4 * qq + 1]);         // Alg. alg:bp
        acc[4 * qq + 2] = fma2(W2, fma2(g1, sel2(d[2], d[1], g1), h[2]), acc[4 * qq + 2]);
        acc[4 * qq + 3] = fma2(W2, fma2(g2, sel2(d[3], d[2], g2), h[3]), acc[4 * qq + 3]);
    }
}

// Two groups (16 TMEM columns: pair 4 q + m = slices 8 q + m / 8 q + 4 + m) of two views.
template <int BW, int Q0>
__device__ __forceinline__ void quad_sub2(uint32_t tacc, uint32_t a0, const ThreadInv& t,
                                          uint32_t a1, const ThreadInv& u, uint32_t b0,
                                          uint32_t b1, int bh)
{
    f2x acc[8];
    tm_ld16(tacc + 8 * Q0, acc);
    tm_wait_ld();
    quad_groups<BW, Q0, 2>(acc, a0, t, b0, bh);
    quad_groups<BW, Q0, 2>(acc, a1, u, b1, bh);
    tm_st16(tacc + 8 * Q0, acc);
}

template <int BW>
__device__ __forceinline__ void walk_views_quad2(uint32_t tacc, uint32_t a0, const ThreadInv& t,
                                                 uint32_t a1, const ThreadInv& u, uint32_t b0,
                                                 uint32_t b1, int bh)
{
    tm_wait_st();
    quad_sub2<BW, 0>(tacc, a0, t, a1, u, b0, b1, bh);
    quad_sub2<BW, 2>(tacc, a0, t, a1, u, b0, b1, bh);
    quad_sub2<BW, 4>(tacc, a0, t, a1, u, b0, b1, bh);
    quad_sub2<BW, 6>(tacc, a0, t, a1, u, b0, b1, bh);
}

// QUINT walk (walk 14, the default where dv/dk < 1/2, config 5): runs of five slices around a
// base floor n; slice b + j, j = -2..2, lies within one row of row n + r_j, r = (0, 0, 0, 1, 1),
// exactly when dv < 1/2 (g_j = f_v + j dv - r_j in [-1, 1)).  Four rows n-1 .. n+2 feed five
// slices: 1.6 LDS.32 per update (the 3-row TRIPLE: 2.0).  Halves at b = 10 q + 2 and 10 q + 7
// (slices 10 q .. 10 q + 9), six groups and a two-slice-pair tail (60, 61 | 62, 63) from rows
// n .. n+2.
// HI (walk 15, 0.5 <= dv/dk < 1): the same five-slice runs reach rows n-2 .. n+3, r = (-1, 0,
// 0, 1, 2) -- g_j in [-1, 1) exactly when 0.5 <= dv <= 1: six rows per five slices, 2.4 LDS.32
// per update (QUAD 2.5) but a 2+2 tail per chunk.
template <int BW, int Q0, int NQ, bool HI = false>
__device__ __forceinline__ void quint_groups(f2x (&acc)[5 * NQ], uint32_t a0, const ThreadInv& t,
                                             uint32_t blo = 0, int bh = 0)
{
    constexpr uint32_t S = BW * 4;
    const f2x dv2 = pk2(t.dv, t.dv), dvm12 = pk2(t.dvm1, t.dvm1), W2 = pk2(t.W, t.W);
    const f2x du2 = pk2(t.du, t.du);
    const f2x magic2 = pk2(8388608.0f, 8388608.0f), nmagic2 = pk2(-8388608.0f, -8388608.0f);
    const f2x fv02 = pk2(t.fv0, t.fv0);
    f2x kvec = pk2((float)(10 * Q0 + 2), (float)(10 * Q0 + 7));
    asm volatile("mov.b64 %0, %0;" : "+l"(kvec));
#pragma unroll
    for (int qq = 0; qq < NQ; ++qq) {
        const f2x v = fma2(kvec, dv2, fv02);
        asm("add.rn.f32x2 %0, %0, %1;" : "+l"(kvec) : "l"(pk2(10.f, 10.f)));
        const f2x tb = add2_rd(v, magic2);
        const f2x fr = sub2(v, add2(tb, nmagic2));
        const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
        const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
        constexpr int NR = HI ? 6 : 4, R0 = HI ? 2 : 1;  // rows n-R0 .. n-R0+NR-1
        f2x h[NR];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            check_tap(adA + (r - R0) * S, blo, BW, bh);
            check_tap(adB + (r - R0) * S, blo, BW, bh);
            const f2x a = pk2(lds32(adA + (r - R0) * S), lds32(adB + (r - R0) * S));
            const f2x b = pk2(lds32(adA + (r - R0) * S + 4), lds32(adB + (r - R0) * S + 4));
            h[r] = fma2(du2, sub2(b, a), a);  // Alg. alg:subpixel lines 4-5
        }
        f2x d[NR - 1];  // d[r] = h[r+1] - h[r]
#pragma unroll
        for (int r = 0; r < NR - 1; ++r) d[r] = sub2(h[r + 1], h[r]);
        constexpr int N0 = R0;  // index of row n in h
        const f2x gm1 = sub2(fr, dv2);    // slice b - 1 from row n
        const f2x g1 = add2(fr, dvm12);   // slice b + 1 from row n + 1
        if constexpr (HI) {
            const f2x gm2 = sub2(gm1, dvm12);  // slice b - 2 from row n - 1
            const f2x g2 = add2(g1, dvm12);    // slice b + 2 from row n + 2
            acc[5 * qq] = fma2(W2, fma2(gm2, sel2(d[N0 - 1], d[N0 - 2], gm2), h[N0 - 1]), acc[5 * qq]);
            acc[5 * qq + 4] = fma2(W2, fma2(g2, sel2(d[N0 + 2], d[N0 + 1], g2), h[N0 + 2]), acc[5 * qq + 4]);
        } else {
            const f2x gm2 = sub2(gm1, dv2);    // slice b - 2 from row n
            const f2x g2 = add2(g1, dv2);      // slice b + 2 from row n + 1
            acc[5 * qq] = fma2(W2, fma2(gm2, sel2(d[N0], d[N0 - 1], gm2), h[N0]), acc[5 * qq]);
            acc[5 * qq + 4] = fma2(W2, fma2(g2, sel2(d[N0 + 1], d[N0], g2), h[N0 + 1]), acc[5 * qq + 4]);
        }
        // line 6 (the row lerp), Alg. alg:bp line 10 (the accumulation)
        acc[5 * qq + 1] = fma2(W2, fma2(gm1, sel2(d[N0], d[N0 - 1], gm1), h[N0]), acc[5 * qq + 1]);
        acc[5 * qq + 2] = fma2(W2, fma2(fr, d[N0], h[N0]), acc[5 * qq + 2]);
        acc[5 * qq + 3] = fma2(W2, fma2(g1, sel2(d[N0 + 1], d[N0], g1), h[N0 + 1]), acc[5 * qq + 3]);
    }
}

// Slices 60, 61 (low half) and 62, 63 (high half) from rows n .. n+2 of their floors.
template <int BW>
__device__ __forceinline__ void quint_tail(f2x (&acc)[2], uint32_t a0, const ThreadInv& t,
                                           uint32_t blo = 0, int bh = 0)
{
    constexpr uint32_t S = BW * 4;
    const f2x dv2 = pk2(t.dv, t.dv), dvm12 = pk2(t.dvm1, t.dvm1), W2 = pk2(t.W, t.W);
    const f2x du2 = pk2(t.du, t.du);
    const f2x magic2 = pk2(8388608.0f, 8388608.0f), nmagic2 = pk2(-8388608.0f, -8388608.0f);
    const f2x v = fma2(pk2(60.f, 62.f), dv2, pk2(t.fv0, t.fv0));
    const f2x tb = add2_rd(v, magic2);
    const f2x fr = sub2(v, add2(tb, nmagic2));
    const uint32_t adA = __float_as_uint(lo2(tb)) * S + a0;
    const uint32_t adB = __float_as_uint(hi2(tb)) * S + a0;
    f2x h[3];
#pragma unroll
    for (int r = 0; r < 3; ++r) {
        check_tap(adA + r * S, blo, BW, bh);
        check_tap(adB + r * S, blo, BW, bh);
        const f2x a = pk2(lds32(adA + r * S), lds32(adB + r * S));
        const f2x b = pk2(lds32(adA + r * S + 4), lds32(adB + r * S + 4));
        h[r] = fma2(du2, sub2(b, a), a);
    }
    const f2x d01 = sub2(h[1], h[0]), d12 = sub2(h[2], h[1]);
    const f2x g = add2(fr, dvm12);
    acc[0] = fma2(W2, fma2(fr, d01, h[0]), acc[0]);
    acc[1] = fma2(W2, fma2(g, sel2(d12, d01, g), h[1]), acc[1]);
}

// Two QUINT groups (20 TMEM columns: pair 5 q + m = slices 10 q + m / 10 q + 5 + m) of two views.
template <int BW, int Q0, bool HI>
__device__ __forceinline__ void quint_sub2(uint32_t tacc, uint32_t a0, const ThreadInv& t,
                                           uint32_t a1, const ThreadInv& u, uint32_t b0,
                                           uint32_t b1, int bh)
{
    f2x acc[10];
    {
        f2x x[8], y[2];
        tm_ld16(tacc + 10 * Q0, x);
        tm_ld4(tacc + 10 * Q0 + 16, y);
        tm_wait_ld();
#pragma unroll
        for (int m = 0; m < 8; ++m) acc[m] = x[m];
        acc[8] = y[0];
        acc[9] = y[1];
    }
    quint_groups<BW, Q0, 2, HI>(acc, a0, t, b0, bh);
    quint_groups<BW, Q0, 2, HI>(acc, a1, u, b1, bh);
    {
        f2x x[8], y[2];
#pragma unroll
        for (int m = 0; m < 8; ++m) x[m] = acc[m];
        y[0] = acc[8];
        y[1] = acc[9];
        tm_st16(tacc + 10 * Q0, x);
        tm_st4(tacc + 10 * Q0 + 16, y);
    }
}

template <int BW, bool HI>
__device__ __forceinline__ void walk_views_quint2(uint32_t tacc, uint32_t a0, const ThreadInv& t,
                                                  uint32_t a1, const ThreadInv& u, uint32_t b0,
                                                  uint32_t b1, int bh)
{
    tm_wait_st();
    quint_sub2<BW, 0, HI>(tacc, a0, t, a1, u, b0, b1, bh);
    quint_sub2<BW, 2, HI>(tacc, a0, t, a1, u, b0, b1, bh);
    quint_sub2<BW, 4, HI>(tacc, a0, t, a1, u, b0, b1, bh);
    f2x acc[2];
    tm_ld4(tacc + 60, acc);
    tm_wait_ld();
    quint_tail<BW>(acc, a0, t, b0, bh);
    quint_tail<BW>(acc, a1, u, b1, bh);
    tm_st4(tacc + 60, acc);
}

// Flush of the QUAD accumulators: slices of the slab only (a partial chunk's other slices
// were walked but are not written), zeros back.
template <bool RED, int RUN>
__device__ __forceinline__ void flush_quad(uint32_t tacc, const BPParams& p, int i, int j, int kb,
                                           bool overwrite, bool inside)
{
    tm_wait_st();
    float* q0 = vol_voxel(p, kb, j, i);
    const long plane = (long)p.Ny * p.Nx;
    const int klo = p.k0 - kb, khi = p.k0 + p.nk - kb;  // slab slices of this chunk: [klo, khi)
    const f2x zero[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int part = 0; part < 4; ++part) {  // pairs 8 part .. 8 part + 7
        f2x a[8];
        tm_ld16(tacc + 16 * part, a);
        tm_wait_ld();
        if (inside) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const int pi = 8 * part + m;
#pragma unroll
                for (int half = 0; half < 2; ++half) {
                    const int kk = RUN == 4 ? 8 * (pi / 4) + 4 * half + pi % 4
                                   : pi < 30 ? 10 * (pi / 5) + 5 * half + pi % 5
                                             : 60 + 2 * half + (pi - 30);
                    const float v = half ? hi2(a[m]) : lo2(a[m]);
                    if (kk >= klo && kk < khi)
                        put_voxel<RED>(p, q0 + kk * plane, kb + kk, j, i, v, overwrite);
                }
            }
        }
        tm_st16(tacc + 16 * part, zero);
    }
}

// The two-views-per-step TMEM kernel (bp_tmem2_kernel's pipeline) with the QUAD walk; whole and
// partial chunks alike.
template <int BW, bool RED = false, int RUN = 4>
__global__ void __launch_bounds__(kThreads, 3)
    bp_quad2_kernel(const __grid_constant__ BPParams p, const __grid_constant__ CUtensorMap tmap,
                    const __grid_constant__ PTable pt)
{
    constexpr int KC = 64, NB = kRawBuf2, VB = 128;
    extern __shared__ __align__(128) unsigned char smem[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int tile_i = (int)blockIdx.z * p.raster + (int)(blockIdx.x % (unsigned)p.raster);
    const int tile_j = (int)(blockIdx.x / (unsigned)p.raster);
    if (tile_i >= p.tiles_i) return;
    const int i = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
    const int j = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
    const int ic = min(i, p.Nx - 1), jc = min(j, p.Ny - 1);
    const int i_corner = (lane & 1) ? min(tile_i * kTI + kTI, p.Nx) - 1 : tile_i * kTI;
    const int j_corner = (lane & 2) ? min(tile_j * kTJ + kTJ, p.Ny) - 1 : tile_j * kTJ;
    const int kb = p.kb0 + (int)blockIdx.y * KC;
    if (p.vb != VB) __trap();
    const int n = (int)p.n_views;

    unsigned char* const raw = smem;
    Meta* const meta = reinterpret_cast<Meta*>(raw + NB * p.raw_bytes);
    uint64_t* const mbar = reinterpret_cast<uint64_t*>(meta + kMetaRing);
    uint32_t* const tslot = reinterpret_cast<uint32_t*>(mbar + NB);
    const uint32_t tx_bytes = (uint32_t)(BW * p.box_h * 4);
    const CUtensorMap* const tmap_ptr = &tmap;
    const PTable* const ptab = &pt;
    const uint32_t raw0 = smem_u32(raw);

    auto issue = [=](int t) {
        const Meta& m = meta[t & (kMetaRing - 1)];
        if (!m.fast) __trap();
        const int b = t % NB;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&mbar[b], tx_bytes);
        tma_load_3d(raw + b * p.raw_bytes, tmap_ptr, &mbar[b], m.u_org, m.v_org - p.v0, t);
    };
    auto metas = [=](int t0) {  // boxes of the whole chunk (partial chunks too), 8 views
        if (warp == ((t0 >> 3) & 7))
            compute_meta8<KC, RUN == 6 ? 15 : 13>(meta, p, ptab, t0, n, tile_i, tile_j, kb);
    };

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
                         smem_u32(tslot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) {
        for (int b = 0; b < NB; ++b) mbar_init(&mbar[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    metas(0);
    int meta_next = 8;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tacc = *tslot + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(64 * (warp >> 2));
    if (tid == 0)
        for (int t = 0; t < NB && t < n; ++t) issue(t);
    {
        const f2x zero[8] = {0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int part = 0; part < 4; ++part) tm_st16(tacc + 16 * part, zero);
    }

    const int first_flush = (int)(VB - 1 - (p.s0 % VB + VB) % VB);
    const float fdi = (float)(ic - tile_i * kTI), fdj = (float)(jc - tile_j * kTJ);
    const uint32_t nm = p.neg_magic;
    // box ring position of view t (buffer, mbarrier phase), stepped without divisions
    int bt = 0;
    uint32_t pt0 = 0;
    for (int t = 0; t < n;) {
        const bool two = t + 1 < n && !(t == 0 && (first_flush & 1) == 0);
        const int te = two ? t + 1 : t;
        int be = bt;
        uint32_t pe = pt0;
        if (two && ++be == NB) {
            be = 0;
            pe ^= 1u;
        }
        const Meta& m0 = meta[t & (kMetaRing - 1)];
        const Meta& m1 = meta[te & (kMetaRing - 1)];
        const ThreadInv ti = quad_inv(m0, fdi, fdj);
        ThreadInv tu = quad_inv(m1, fdi, fdj);
        if (!two) tu.W = 0.f;
        mbar_wait(&mbar[bt], pt0);
        if (two) mbar_wait(&mbar[be], pe);
        const int bt0 = bt;
        const uint32_t a0 = raw0 + (uint32_t)(bt * p.raw_bytes) +
                            (uint32_t)(((ti.nv - m0.v_org) * BW + (ti.nu - m0.u_org)) * 4) + nm;
        const uint32_t a1 = raw0 + (uint32_t)(be * p.raw_bytes) +
                            (uint32_t)(((tu.nv - m1.v_org) * BW + (tu.nu - m1.u_org)) * 4) + nm;
        bt = be + 1;  // the view after te
        pt0 = pe;
        if (bt == NB) {
            bt = 0;
            pt0 ^= 1u;
        }
        const uint32_t b0 = raw0 + (uint32_t)(bt0 * p.raw_bytes), b1 = raw0 + (uint32_t)(be * p.raw_bytes);
        if constexpr (RUN == 4)
            walk_views_quad2<BW>(tacc, a0, ti, a1, tu, b0, b1, p.box_h);
        else
            walk_views_quint2<BW, RUN == 6>(tacc, a0, ti, a1, tu, b0, b1, p.box_h);
        if ((te >= first_flush && ((te - first_flush) & (VB - 1)) == 0) || te == n - 1) {
            const int fi = tile_i * kTI + (warp & 1) * 8 + (lane & 7);
            const int fj = tile_j * kTJ + (warp >> 1) * 4 + (lane >> 3);
            const bool ow = !p.accumulate && te <= first_flush;
            flush_quad<RED, RUN>(tacc, p, fi, fj, kb, ow, fi < p.Nx && fj < p.Ny);
        }
        if (te + NB >= meta_next && meta_next < n) {
            metas(meta_next);
            meta_next += 8;
        }
        __syncthreads();
        if (tid == 0)
            for (int v = t + NB; v <= te + NB; ++v)
                if (v < n) issue(v);
        t = te + 1;
    }
    tm_wait_st();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(*tslot)
                     : "memory");
}

// Opt-in dynamic shared memory per CTA of the current device.
int max_dyn_smem()
{
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) != cudaSuccess ||
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess) {
        cudaGetLastError();
        return 48 * 1024;
    }
    return v;
}

PFN_cuTensorMapEncodeTiled_v12000 get_encode()
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void* ptr = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    }
    return fn;
}

template <int KC, int P2, int WALK>
ifdk_status launch_t(const BPParams& p, const CUtensorMap& map, const PTable& pt, bool tma,
                     dim3 grid, size_t smem, cudaStream_t st)
{
    cudaError_t e;
    if (tma) {
        auto k = bp_kernel<KC, P2, true, WALK>;
        e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(bp)");
        k<<<grid, kThreads, smem, st>>>(p, map, pt);
    } else {
        auto k = bp_kernel<KC, P2, false, (WALK >= 2 ? 2 : 1)>;
        k<<<grid, kThreads, 0, st>>>(p, map, pt);
    }
    e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "bp_kernel launch");
    count_launch();
    return IFDK_OK;
}

// PAIR walk: two slices per floor; valid while dv/dk = (D/Dv) Dz / z < 1 for every z.
bool use_pair(const ifdk_geometry* g)
{
    const double dv_max = g->D / g->Dv * g->Dz / g->zmin;
    return dv_max < 0.999;
}

// Tuning hook (ifdk_set_bp_variant): a walk of the automatic choice's family gives bitwise its
// result (the QUAD / QUINT kernels are families of their own, equal to the others to fp32
// rounding); the raster only reorders CTAs.
std::atomic<int> g_walk_override{0}, g_raster_override{0};

// Slices per floor of the k-walk.  Default where dv/dk < 1 for every z (all five configs):
// the TRIPLE walks with TMEM accumulators, two views per step -- 4-row (11) where
// 0.5 <= dv/dk (configs 1-4), 3-row (12) where dv/dk < 0.5 everywhere (config 5); measured on
// config 4 / the config-5 slab (256 views): 2220 / 2480 GUPS vs 2133 / 2345 for one view per
// step (9 / 10) and 2022 / 2197 for the register walks (6 / 7; 2000 vs 1884 for PAIR RAW 5) --
// and the PAIR RAW walk (5) in between; their partial chunks run on the pair-patch companions
// 3, 8 and 4, bitwise equal.  dv/dk >= 1 somewhere: one floor per slice (walk 1, 32-slice
// chunks).  The override (ifdk_set_bp_variant) picks among the bitwise-equal walks of the
// geometry's family: 2, 4, 5 (PAIR), 3, 6, 9, 11 (4-row TRIPLE), 7, 8, 10, 12 (3-row TRIPLE).
int choose_walk(const ifdk_geometry* g)
{
    if (!use_pair(g)) return 1;
    const double dv_min = g->D / g->Dv * g->Dz / g->zmax;
    const double dv_max = g->D / g->Dv * g->Dz / g->zmin;
    int w = dv_min >= 0.5001 && dv_max < 0.9999 ? 13 : dv_max < 0.4999 ? 14 : 5;
    const int v = g_walk_override.load(std::memory_order_relaxed);
    if (v == 2 || v == 4 || v == 5) w = v;
    if ((v == 3 || v == 6 || v == 9 || v == 11) && dv_min >= 0.5001) w = v;
    if (v == 13 && dv_min >= 0.5001 && dv_max < 0.9999) w = v;
    if (v == 14 && dv_max < 0.4999) w = v;
    if (v == 15 && dv_min >= 0.5001 && dv_max < 0.9999) w = v;
    if ((v == 7 || v == 8 || v == 10 || v == 12) && dv_max < 0.4999) w = v;
    return w;
}

// Slices per k-chunk (= register accumulators per thread).  The choice depends on the geometry
// only, never on the slab, so every decomposition of a volume walks identical chunks.
// Measured on B200 (config 4): PAIR with 64 slices (2 CTAs/SM, 128 registers) 1724 GUPS vs
// 32 slices (3 CTAs/SM, 80 registers) 1586; without PAIR 32 slices win.
int choose_kc(const ifdk_geometry* g) { return use_pair(g) ? 64 : 32; }

}  // namespace

namespace {

// One launch over views s0 .. s0+n_views-1 (n_views <= kMaxViewsPerLaunch).
ifdk_status launch_range(const ifdk_geometry* g, const float* Q, long s0, long n_views, int v0,
                         int n_rows, float* vol, int k0, int nk, int accumulate, cudaStream_t st,
                         const RedDest* red)
{
    // Per-view projection matrices (fp64), passed in the kernel's parameter space.
    PTable pt;
    fill_ptable(g, s0, n_views, pt);

    BPParams p{};
    p.Q = Q;
    p.vol = vol;
    p.n_views = n_views;
    p.s0 = s0;
    p.Nu = g->Nu; p.Nv = g->Nv; p.Nx = g->Nx; p.Ny = g->Ny;
    p.v0 = v0; p.n_rows = n_rows;
    p.k0 = k0; p.nk = nk;
    const int KC = choose_kc(g);
    p.kb0 = (k0 / KC) * KC;
    p.tiles_i = (g->Nx + kTI - 1) / kTI;
    const int tiles_j = (g->Ny + kTJ - 1) / kTJ;
    const int n_chunks = (k0 + nk - p.kb0 + KC - 1) / KC;
    p.vb = 128;
    p.accumulate = accumulate;
    if (red) {
        p.red = red->mode + 1;
        p.n_dest = red->n;
        for (int d = 0; d < red->n; ++d) {
            p.dest_k0[d] = red->k0[d];
            p.dest[d] = red->base[d];
        }
    }

    // Box of the staged patch from the conservative geometric bound.
    double wb, hb;
    patch_bound(g, kTI, kTJ, KC, &wb, &hb);
    p.pair = use_pair(g) ? 1 : 0;
    int walk = KC == 64 ? choose_walk(g) : (p.pair ? 2 : 1);
    const int box_h = (int)std::ceil(hb) + 6 + p.pair + (walk == 15 ? 1 : 0);
    const int box_w0 = std::max(8, ((int)std::ceil(wb) + 9 + 3) / 4 * 4);  // +3: 16-B origin
    // Raster band of 16 tile columns: measured on B200 (config 4, one 256-view launch) DRAM
    // traffic 49 GB (algorithmic 39 GB) and L2 hit rate 95 %, vs 354 GB and 65 % for the
    // row-major raster, at the same speed (the kernel is shared-memory bound).
    // ifdk_set_bp_variant(.., n) overrides (n >= tiles_i: row-major).
    p.raster = std::min(kRasterTiles, p.tiles_i);
    if (const int r = g_raster_override.load(std::memory_order_relaxed))
        p.raster = (r > 0 && r < p.tiles_i) ? r : p.tiles_i;
    const bool tma_ok = box_h <= 256 && (g->Nu % 4) == 0 &&
                        (reinterpret_cast<uintptr_t>(Q) % 16) == 0 && get_encode() != nullptr;

    // One launch of chunks kb .. kb + nch KC - 1 with walk w (5 = RAW staging, full chunks only).
    auto run = [&](int w, int kb, int nch) -> ifdk_status {
        BPParams q = p;
        q.kb0 = kb;
        q.walk = w;
        int box_w = box_w0, P2 = 0, BW = 0;
        for (int c : {24, 40, 56, 72})
            if (c >= box_w - 1) { P2 = c; break; }
        if (w == 5 || w == 6 || w == 7 || (w >= 9 && w <= 15)) {
            for (int c : {40, 72})  // row pitch = 8 mod 32 words: conflict-free LDS.32 taps
                if (c >= box_w) { BW = c; break; }
            box_w = BW;
        }
        bool tma = tma_ok && P2 != 0;
        CUtensorMap map;
        std::memset(&map, 0, sizeof(map));
        size_t smem = 0;
        if (tma) {
            q.box_w = box_w;
            q.box_h = box_h;
            q.raw_bytes = (box_w * box_h * 4 + 127) / 128 * 128;
            auto raw_smem = [&](int nbuf) {
                return nbuf * (size_t)q.raw_bytes + kMetaRing * sizeof(Meta) + 8 * nbuf + 16;
            };
            // two views per step want six boxes; where those do not fit three CTAs per SM
            // (tall or wide boxes) the one-view step (four boxes) is the faster choice
            if (w >= 11 && w <= 12 && 3 * (raw_smem(kRawBuf2) + 1024) > 228 * 1024) w = w % 2 ? 9 : 10;
            const int nbuf = w >= 11 ? kRawBuf2 : kRawBuf;
            smem = BW ? raw_smem(nbuf)
                      : 2 * (size_t)q.raw_bytes + 2 * sizeof(float2) * box_h * P2 +
                            kMetaRing * sizeof(Meta) + 16;
            cuuint64_t dims[3] = {(cuuint64_t)g->Nu, (cuuint64_t)n_rows, (cuuint64_t)n_views};
            cuuint64_t strides[2] = {(cuuint64_t)g->Nu * 4, (cuuint64_t)g->Nu * 4 * n_rows};
            cuuint32_t box[3] = {(cuuint32_t)box_w, (cuuint32_t)box_h, 1};
            cuuint32_t estr[3] = {1, 1, 1};
            CUresult r = get_encode()(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, (void*)Q, dims,
                                      strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                      CU_TENSOR_MAP_SWIZZLE_NONE,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) tma = false;
            // a box too large for the opt-in shared memory takes the global-memory walk
            if (smem > (size_t)max_dyn_smem()) tma = false;
        }
        if (!tma) {
            P2 = 24;
            BW = 0;
            q.box_w = q.box_h = 0;
            q.raw_bytes = 0;
        }
        q.neg_magic = 0u - 0x4B000000u * (uint32_t)(BW ? BW * 4 : P2 * 8);
        dim3 grid((unsigned)(q.raster * tiles_j), (unsigned)nch,
                  (unsigned)((q.tiles_i + q.raster - 1) / q.raster));
        if (BW && (w == 13 || w == 14 || w == 15)) {
            auto k = w == 13 ? (q.red ? (BW == 40 ? bp_quad2_kernel<40, true> : bp_quad2_kernel<72, true>)
                                      : (BW == 40 ? bp_quad2_kernel<40> : bp_quad2_kernel<72>))
                   : w == 14 ? (q.red ? (BW == 40 ? bp_quad2_kernel<40, true, 5> : bp_quad2_kernel<72, true, 5>)
                                      : (BW == 40 ? bp_quad2_kernel<40, false, 5> : bp_quad2_kernel<72, false, 5>))
                             : (q.red ? (BW == 40 ? bp_quad2_kernel<40, true, 6> : bp_quad2_kernel<72, true, 6>)
                                      : (BW == 40 ? bp_quad2_kernel<40, false, 6> : bp_quad2_kernel<72, false, 6>));
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(bp quad)");
            k<<<grid, kThreads, smem, st>>>(q, map, pt);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "bp_quad2_kernel launch");
            count_launch();
            return IFDK_OK;
        }
        if (BW && w >= 9 && w <= 12) {
            auto k = w == 9    ? (BW == 40 ? bp_tmem_kernel<40, 1, 3> : bp_tmem_kernel<72, 1, 3>)
                     : w == 10 ? (BW == 40 ? bp_tmem_kernel<40, 2, 3> : bp_tmem_kernel<72, 2, 3>)
                     : w == 11 ? (q.red ? (BW == 40 ? bp_tmem2_kernel<40, 1, true> : bp_tmem2_kernel<72, 1, true>)
                                        : (BW == 40 ? bp_tmem2_kernel<40, 1> : bp_tmem2_kernel<72, 1>))
                               : (q.red ? (BW == 40 ? bp_tmem2_kernel<40, 2, true> : bp_tmem2_kernel<72, 2, true>)
                                        : (BW == 40 ? bp_tmem2_kernel<40, 2> : bp_tmem2_kernel<72, 2>));
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(bp tmem)");
            k<<<grid, kThreads, smem, st>>>(q, map, pt);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "bp_tmem_kernel launch");
            count_launch();
            return IFDK_OK;
        }
        if (BW) {
            auto k = w == 6   ? (BW == 40 ? bp_raw_kernel<64, 40, 1> : bp_raw_kernel<64, 72, 1>)
                     : w == 7 ? (BW == 40 ? bp_raw_kernel<64, 40, 2> : bp_raw_kernel<64, 72, 2>)
                              : (BW == 40 ? bp_raw_kernel<64, 40> : bp_raw_kernel<64, 72>);
            cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 (int)smem);
            if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(bp raw)");
            k<<<grid, kThreads, smem, st>>>(q, map, pt);
            e = cudaGetLastError();
            if (e != cudaSuccess) return cuda_fail(e, "bp_raw_kernel launch");
            count_launch();
            return IFDK_OK;
        }
        if (w == 5) w = 4;
        if (w == 6 || (w >= 9 && w % 2 == 1)) w = 3;
        if (w == 7 || (w >= 9 && w % 2 == 0)) w = 8;
        if (w == 8) {
            switch (P2) {
                case 24: return launch_t<64, 24, 8>(q, map, pt, tma, grid, smem, st);
                case 40: return launch_t<64, 40, 8>(q, map, pt, tma, grid, smem, st);
                case 56: return launch_t<64, 56, 8>(q, map, pt, tma, grid, smem, st);
                default: return launch_t<64, 72, 8>(q, map, pt, tma, grid, smem, st);
            }
        }
        if (w == 3) {
            switch (P2) {
                case 24: return launch_t<64, 24, 3>(q, map, pt, tma, grid, smem, st);
                case 40: return launch_t<64, 40, 3>(q, map, pt, tma, grid, smem, st);
                case 56: return launch_t<64, 56, 3>(q, map, pt, tma, grid, smem, st);
                default: return launch_t<64, 72, 3>(q, map, pt, tma, grid, smem, st);
            }
        } else if (w == 4) {
            switch (P2) {
                case 24: return launch_t<64, 24, 4>(q, map, pt, tma, grid, smem, st);
                case 40: return launch_t<64, 40, 4>(q, map, pt, tma, grid, smem, st);
                case 56: return launch_t<64, 56, 4>(q, map, pt, tma, grid, smem, st);
                default: return launch_t<64, 72, 4>(q, map, pt, tma, grid, smem, st);
            }
        } else if (w == 2 && KC == 64) {
            switch (P2) {
                case 24: return launch_t<64, 24, 2>(q, map, pt, tma, grid, smem, st);
                case 40: return launch_t<64, 40, 2>(q, map, pt, tma, grid, smem, st);
                case 56: return launch_t<64, 56, 2>(q, map, pt, tma, grid, smem, st);
                default: return launch_t<64, 72, 2>(q, map, pt, tma, grid, smem, st);
            }
        } else if (w == 2) {
            switch (P2) {
                case 24: return launch_t<32, 24, 2>(q, map, pt, tma, grid, smem, st);
                case 40: return launch_t<32, 40, 2>(q, map, pt, tma, grid, smem, st);
                case 56: return launch_t<32, 56, 2>(q, map, pt, tma, grid, smem, st);
                default: return launch_t<32, 72, 2>(q, map, pt, tma, grid, smem, st);
            }
        }
        switch (P2) {
            case 24: return launch_t<32, 24, 1>(q, map, pt, tma, grid, smem, st);
            case 40: return launch_t<32, 40, 1>(q, map, pt, tma, grid, smem, st);
            case 56: return launch_t<32, 56, 1>(q, map, pt, tma, grid, smem, st);
            default: return launch_t<32, 72, 1>(q, map, pt, tma, grid, smem, st);
        }
    };

    if ((walk != 5 && walk != 6 && walk != 7 && (walk < 9 || walk > 15)) || !tma_ok || box_w0 > 72)
        return run(walk, p.kb0, n_chunks);
    if (walk >= 13 && walk <= 15) {
        // the QUAD kernel walks partial chunks itself (one launch for the slab) when its six
        // boxes fit three CTAs per SM; otherwise the TRIPLE family (walk 11 + companions)
        const int bw = box_w0 <= 40 ? 40 : 72;
        const size_t raw_bytes = ((size_t)bw * box_h * 4 + 127) / 128 * 128;
        const size_t smem6 = kRawBuf2 * raw_bytes + kMetaRing * sizeof(Meta) + 8 * kRawBuf2 + 16;
        if (3 * (smem6 + 1024) <= 228 * 1024) return run(walk, p.kb0, n_chunks);
        walk = walk == 14 ? 12 : 11;
    }
    // RAW staging runs the whole chunks; a partial chunk at either slab end (its masked slices
    // would read rows outside the box) takes the x2 pair walk, bitwise the same values.
    const bool head = (k0 % KC) != 0, tail = ((k0 + nk) % KC) != 0;
    const int c0 = head ? 1 : 0, c1 = tail ? n_chunks - 1 : n_chunks;
    ifdk_status s = IFDK_OK;
    if (c1 > c0) s = run(walk, p.kb0 + c0 * KC, c1 - c0);
    // partial chunks: walk 4 for walk 5, 3 for 6, 8 for 7 (bitwise the same arithmetic)
    const int wp = (walk == 6 || (walk >= 9 && walk % 2 == 1)) ? 3
                   : (walk == 7 || (walk >= 9 && walk % 2 == 0)) ? 8 : 4;
    if (s == IFDK_OK && head) s = run(wp, p.kb0, 1);
    if (s == IFDK_OK && tail && (n_chunks - 1 > 0 || !head)) s = run(wp, p.kb0 + (n_chunks - 1) * KC, 1);
    return s;
}

}  // namespace

// Lazy module loading loads a kernel at its first launch, which waits for the context to go
// idle: a kernel that spins on a peer's signal (ifdk_wait) would then deadlock against the
// first launch of any kernel behind it.  ifdk_wait calls this first (cudaFuncGetAttributes
// loads the function).
template <typename K>
static void touch_kernel(K k)
{
    cudaFuncAttributes a;
    if (cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k)) != cudaSuccess)
        cudaGetLastError();
}

template <int P2>
static void preload_bp_p2()
{
    touch_kernel(bp_kernel<64, P2, true, 2>);
    touch_kernel(bp_kernel<64, P2, true, 3>);
    touch_kernel(bp_kernel<64, P2, true, 4>);
    touch_kernel(bp_kernel<64, P2, true, 8>);
    touch_kernel(bp_kernel<32, P2, true, 2>);
    touch_kernel(bp_kernel<32, P2, true, 1>);
    touch_kernel(bp_kernel<64, P2, false, 2>);
    touch_kernel(bp_kernel<32, P2, false, 2>);
    touch_kernel(bp_kernel<32, P2, false, 1>);
}

void preload_bp_kernels()
{
    preload_bp_p2<24>();
    preload_bp_p2<40>();
    preload_bp_p2<56>();
    preload_bp_p2<72>();
    touch_kernel(bp_raw_kernel<64, 40, 0>);
    touch_kernel(bp_raw_kernel<64, 72, 0>);
    touch_kernel(bp_raw_kernel<64, 40, 1>);
    touch_kernel(bp_raw_kernel<64, 72, 1>);
    touch_kernel(bp_raw_kernel<64, 40, 2>);
    touch_kernel(bp_raw_kernel<64, 72, 2>);
    touch_kernel(bp_tmem_kernel<40, 1, 3>);
    touch_kernel(bp_tmem_kernel<72, 1, 3>);
    touch_kernel(bp_tmem_kernel<40, 2, 3>);
    touch_kernel(bp_tmem_kernel<72, 2, 3>);
    touch_kernel(bp_tmem2_kernel<40, 1>);
    touch_kernel(bp_tmem2_kernel<72, 1>);
    touch_kernel(bp_tmem2_kernel<40, 2>);
    touch_kernel(bp_tmem2_kernel<72, 2>);
    touch_kernel(bp_tmem2_kernel<40, 1, true>);
    touch_kernel(bp_tmem2_kernel<72, 1, true>);
    touch_kernel(bp_tmem2_kernel<40, 2, true>);
    touch_kernel(bp_tmem2_kernel<72, 2, true>);
    touch_kernel(bp_quad2_kernel<40>);
    touch_kernel(bp_quad2_kernel<72>);
    touch_kernel(bp_quad2_kernel<40, true>);
    touch_kernel(bp_quad2_kernel<72, true>);
    touch_kernel(bp_quad2_kernel<40, false, 5>);
    touch_kernel(bp_quad2_kernel<72, false, 5>);
    touch_kernel(bp_quad2_kernel<40, true, 5>);
    touch_kernel(bp_quad2_kernel<72, true, 5>);
    touch_kernel(bp_quad2_kernel<40, false, 6>);
    touch_kernel(bp_quad2_kernel<72, false, 6>);
    touch_kernel(bp_quad2_kernel<40, true, 6>);
    touch_kernel(bp_quad2_kernel<72, true, 6>);
}

void set_bp_variant(int walk, int raster)
{
    g_walk_override.store(walk, std::memory_order_relaxed);
    g_raster_override.store(raster, std::memory_order_relaxed);
}

ifdk_status launch_backproject(const ifdk_geometry* g, const float* Q, long s0, long n_views,
                               int v0, int n_rows, float* vol, int k0, int nk, int accumulate,
                               cudaStream_t st, const RedDest* red)
{
    if (n_views == 0 && red) return IFDK_OK;  // nothing to add
    if (n_views == 0) {
        if (!accumulate) {
            cudaError_t e =
                cudaMemsetAsync(vol, 0, sizeof(float) * (size_t)nk * g->Ny * g->Nx, st);
            if (e != cudaSuccess) return cuda_fail(e, "cudaMemsetAsync");
        }
        return IFDK_OK;
    }
    // Launches end at global view indices that are multiples of kMaxViewsPerLaunch (and so of
    // the summation batch): every voxel sees the same sums in the same order as one launch.
    const size_t view_elems = (size_t)n_rows * g->Nu;
    long t = 0;
    while (t < n_views) {
        const long s = s0 + t;
        long stop = (s >= 0 ? s / kMaxViewsPerLaunch + 1 : -((-s - 1) / kMaxViewsPerLaunch))
                    * kMaxViewsPerLaunch;  // next multiple strictly above s
        long n = stop - s;
        if (n > n_views - t) n = n_views - t;
        ifdk_status r = launch_range(g, Q + (size_t)t * view_elems, s, n, v0, n_rows, vol, k0, nk,
                                     (accumulate || t > 0) ? 1 : 0, st, red);
        if (r != IFDK_OK) return r;
        t += n;
    }
    return IFDK_OK;
}

}  // namespace ifdk
