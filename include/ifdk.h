/*
 * ifdk.h -- C ABI of the B200-native iFDK hot path (libifdk.so).
 *
 * The library computes FDK cone-beam reconstruction as the paper states the
 * problem: "N_u x N_v x N_p -> N_x x N_y x N_z" (section
 * "Terminology"), with the parameters of Table tbl:cbct-param.
 *   Filtering (Alg. alg:filter):  Q_s = (E_s . F_cos) (x) F_ramp, row by row.
 *   Back-projection (Alg. alg:bp, Alg. alg:subpixel P:431-447):
 *     I(i,j,k) += sum_s f^2 . interp2(Q_s, x f, y f),  [x,y,z] = P_s [i,j,k,1], f = 1/z,
 *     with P_s = (M1 . Mrot . M0)[0:3] of the appendix, beta_s = s . theta.
 * Readings of the passages the paper leaves silent (F_cos formula, Ram-Lak
 * ramp, FDK constant folded into Q, floor + per-tap zero border) are listed in
 * DESIGN.md; the ids c-A5 .. c-A9 below refer to that list.
 *
 * Conventions (all entry points):
 *   - Every function returns ifdk_status; nothing throws across the ABI.
 *     ifdk_last_error() returns a thread-local message for the last failure.
 *   - Units: pitches Du, Dv, Dx, Dy, Dz and distances D, d in mm (reading
 *     c-A2); theta in radians; u, v in detector pixels.
 *   - Layouts (row-major, fp32, x/u fastest):
 *       projections  [n_views][n_rows][Nu]   rows v0 .. v0+n_rows-1 of each view
 *       volume slab  [nk][Ny][Nx]            k = k0 .. k0+nk-1  ("i-major", P:800 slices)
 *   - Ownership: the geometry handle is created and freed by the library.  All
 *     data buffers are owned by the caller; the library never frees them.
 *     Pointers named *_dev are CUDA device pointers on the current device;
 *     pointers named *_host are host pointers.  Only ifdk_reconstruct and
 *     ifdk_reconstruct_host allocate scratch: stream-ordered, from a memory pool
 *     owned by the geometry that keeps its memory between calls (so repeated
 *     reconstructions do not remap tens of GiB) and is released by
 *     ifdk_geometry_destroy.
 *   - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy
 *     default stream).  Device work is enqueued asynchronously on it; the
 *     status reports argument and launch errors only.  Asynchronous faults
 *     surface at the caller's next synchronisation.
 *   - There is no CPU fallback: without a CUDA device every compute entry point
 *     returns IFDK_ERR_CUDA.
 */
#ifndef IFDK_H
#define IFDK_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    IFDK_OK = 0,
    IFDK_ERR_INVALID_ARGUMENT = 1,   /* bad dimension/pitch/pointer/flag */
    IFDK_ERR_DEGENERATE_GEOMETRY = 2,/* some voxel could reach z <= 0 (volume not inside the source circle) */
    IFDK_ERR_SHAPE = 3,              /* slab/band outside range, band not covering the taps, n_views < 0 */
    IFDK_ERR_CUDA = 4,               /* CUDA runtime / launch error (incl. no device) */
    IFDK_ERR_OUT_OF_MEMORY = 5       /* scratch allocation failed */
} ifdk_status;

typedef struct ifdk_geometry ifdk_geometry; /* opaque, library-owned */

/* Create a geometry from Table tbl:cbct-param: detector Nu x Nv
 * pixels of pitch Du x Dv; volume Nx x Ny x Nz voxels of pitch Dx x Dy x Dz;
 * source-to-axis distance d and source-to-detector distance D; angle step
 * theta (beta_s = s*theta; the paper's theta = 2 pi / N_p).
 * N_p is not a geometry argument: any global view index s is allowed.
 * Errors: INVALID_ARGUMENT if a dimension < 1, a pitch <= 0, D <= d, d <= 0,
 * theta <= 0 or not finite (the rotation sense is fixed by Mrot,
 * P:556-570), or out == NULL; DEGENERATE_GEOMETRY if the volume's
 * circumscribed radius in the rotation plane is >= d. */
ifdk_status ifdk_geometry_create(int Nu, int Nv, int Nx, int Ny, int Nz, double Du, double Dv,
                                 double Dx, double Dy, double Dz, double D, double d,
                                 double theta, ifdk_geometry** out);

/* Free a geometry (NULL-safe), the per-device tables it owns and its scratch pool. */
void ifdk_geometry_destroy(ifdk_geometry* g);

/* P_s as a row-major 3x4 fp64 matrix (appendix; 3x4 per reading c-A1).
 * Host-only; works without a GPU. */
ifdk_status ifdk_projection_matrix(const ifdk_geometry* g, long s, double P[12]);

/* Detector rows [*v_lo, *v_hi] (inclusive, clipped to [0, Nv-1]) that the
 * interpolation taps of every voxel of slab k0..k0+nk-1 can touch in view s,
 * with a one-row safety margin on each side.  *v_lo > *v_hi means "none".
 * Host-only.  Errors: SHAPE if the slab is outside [0, Nz). */
ifdk_status ifdk_band_rows(const ifdk_geometry* g, int k0, int nk, long s, int* v_lo, int* v_hi);

/* Alg. alg:filter: filtered_dev = C . ((raw_dev . F_cos) (x) h1)
 * row by row for rows v0..v0+n_rows-1 of n_views views, where F_cos is the
 * cosine weight (reading c-A5), h1 the unit-spacing Ram-Lak kernel applied as
 * a full-length linear convolution (reading c-A6) and C = theta d D / (2 Du)
 * the FDK constant (reading c-A7).  Both buffers [n_views][n_rows][Nu] fp32,
 * device; raw_dev == filtered_dev (in place) is allowed.
 * Errors: INVALID_ARGUMENT (NULL pointers), SHAPE (rows outside [0, Nv), n_views < 0). */
ifdk_status ifdk_filter(const ifdk_geometry* g, const float* raw_dev, float* filtered_dev,
                        long n_views, int v0, int n_rows, void* stream);

/* One destination of ifdk_filter_scatter: rows v_lo..v_hi (inclusive) of every
 * filtered view t are written to base[(t (v_hi - v_lo + 1) + v - v_lo) Nu + u].
 * base is a device pointer on the current device or a peer device's memory mapped
 * into this one (CUDA IPC / symmetric memory over NVLink); caller-owned. */
typedef struct {
    float* base;
    int v_lo, v_hi;
} ifdk_band_dest;

/* Alg. alg:filter exactly as ifdk_filter (bitwise the same values), fused with the
 * row-band exchange of the k-slab split: instead of one output array,
 * each filtered row is stored straight into every destination band that contains
 * it (n_dest <= 16; dests is a host array, copied at launch).  With peer-mapped
 * bases (ifdk_peer_open) the NVLink transfer of a row overlaps the filtering of the
 * next ones.
 * Completion signal (n_flags > 0): flags is a host array of n_flags <= 16 device
 * pointers (words in local or peer-mapped memory); once every row of this launch has
 * been stored, each word is incremented by 1 with a system-scope atomic that is
 * ordered after all those stores (__threadfence_system by every thread, then the
 * "last block" ticket; see csrc/peer.cu).  ticket_dev is a caller-owned device word
 * that must be 0 at launch; the kernel leaves it 0 (launches sharing a ticket must be
 * stream-ordered).  With n_views == 0 the flags are still incremented.  n_flags = 0:
 * no signal (flags, ticket_dev may be NULL); the caller then orders the
 * destinations' later reads itself.
 * Errors: INVALID_ARGUMENT (NULL pointers, n_dest < 1 or > 16, a band outside
 * [0, Nv) or empty, n_flags outside 0..16, a NULL flag or ticket), SHAPE (rows
 * outside [0, Nv), n_views < 0). */
ifdk_status ifdk_filter_scatter(const ifdk_geometry* g, const float* raw_dev, long n_views,
                                int v0, int n_rows, int n_dest, const ifdk_band_dest* dests,
                                int n_flags, unsigned int* const* flags, unsigned int* ticket_dev,
                                void* stream);

/* ---- peer memory and device-side signals of the fused exchange (csrc/peer.cu) ---- */

/* cudaMalloc of `bytes` (a whole allocation, so its IPC handle maps offset 0) and its
 * 64-byte CUDA IPC handle, to be sent to the other ranks (one process per GPU).
 * Free with ifdk_peer_free.  Errors: INVALID_ARGUMENT (NULL, 0 bytes), CUDA,
 * OUT_OF_MEMORY. */
ifdk_status ifdk_peer_alloc(size_t bytes, void** dev_ptr, unsigned char handle[64]);

/* Map another process's ifdk_peer_alloc buffer into this one (cudaIpcOpenMemHandle
 * with lazy peer access: NVLink P2P between GPUs, or the same GPU).  *dev_ptr is valid
 * on the current device until ifdk_peer_close.  Errors: INVALID_ARGUMENT, CUDA. */
ifdk_status ifdk_peer_open(const unsigned char handle[64], void** dev_ptr);
ifdk_status ifdk_peer_close(void* dev_ptr);   /* NULL-safe */
ifdk_status ifdk_peer_free(void* dev_ptr);    /* NULL-safe */

/* After all earlier work on `stream`, increment each of the n_flags <= 16 device words
 * flags[i] (host array of local or peer-mapped device pointers) by 1 with a
 * system-scope atomic (used to release a receive buffer once the back-projection that
 * read it has completed).  Errors: INVALID_ARGUMENT (n_flags outside 0..16, NULL). */
ifdk_status ifdk_signal(int n_flags, unsigned int* const* flags, void* stream);

/* Later work on `stream` waits until each of the n consecutive device words at
 * flags_dev (local memory) has reached `target` (compared modulo 2^32, so the
 * counters may wrap), read with ld.acquire.sys.  A word that never reaches the target
 * (a dead peer) traps after timeout_ms (0: 300 s) instead of hanging the GPU.
 * Errors: INVALID_ARGUMENT (NULL, n outside 1..1024). */
ifdk_status ifdk_wait(const unsigned int* flags_dev, int n, unsigned int target,
                      unsigned int timeout_ms, void* stream);

/* Alg. alg:bp + alg:subpixel for views s0..s0+n_views-1 into the
 * slab k0..k0+nk-1:  vol_dev[k-k0][j][i] (=|+=) sum_s f^2 . interp2(Q_s, u, v).
 * filtered_dev holds detector rows v0..v0+n_rows-1 of each view
 * ([n_views][n_rows][Nu], device); those rows must cover ifdk_band_rows(k0,nk,s)
 * for every view, else SHAPE (a silently zero tap would corrupt the result).
 * Taps off the detector read 0 (reading c-A9).  accumulate = 0 overwrites the
 * slab, 1 adds to it.  The fp64 P_s of the views ride in constant memory (the
 * kernel's parameter space, <= 256 views per launch; longer ranges launch once
 * per 256-view block of the global index, which leaves the result unchanged).  Per-voxel summation is in view order, fp32, with the
 * per-column invariants z, u, 1/z^2 and the k-walk base of v in fp64
 * (DESIGN.md "Numerics").
 * Errors: INVALID_ARGUMENT (NULL, accumulate not 0/1), SHAPE (slab outside
 * [0, Nz), band outside [0, Nv) or not covering, n_views < 0). */
ifdk_status ifdk_backproject(const ifdk_geometry* g, const float* filtered_dev, long s0,
                             long n_views, int v0, int n_rows, float* vol_dev, int k0, int nk,
                             int accumulate, void* stream);

/* Fused projection-split back-projection (the paper's single
 * MPI_Reduce of partial volumes, done inside the back-projection's
 * write-back instead of a separate reduce-scatter).  Views s0..s0+n_views-1 (filtered_dev
 * as for ifdk_backproject) are back-projected over slices k0..k0+nk-1, and every 128-view
 * partial sum of a voxel is ADDED to the destination slab holding its slice: dest[d]
 * ([..][Ny][Nx] fp32, device memory of this GPU or a peer mapping -- ifdk_peer_open --
 * reached over NVLink) holds slices dest_k0[d] .. dest_k0[d+1]-1 (the last one through
 * k0+nk-1).  mode 0: red.global.add.f32 (relaxed, system scope); mode 1:
 * multimem.red.add.f32, dest[] being multicast mappings (NVLS: the switch adds).  The
 * caller zeroes the slabs first and orders the adds of all ranks before reading them
 * (stream / device synchronisation, or ifdk_signal + ifdk_wait).  Sum order across ranks is
 * not fixed, so results agree with ifdk_backproject to fp32 rounding, not bitwise.
 * Errors: INVALID_ARGUMENT (NULL, n_dest outside 1..16, mode not 0/1), SHAPE (slab or band
 * as for ifdk_backproject; dest_k0 not strictly increasing or dest_k0[0] > k0). */
ifdk_status ifdk_backproject_reduce(const ifdk_geometry* g, const float* filtered_dev, long s0,
                                    long n_views, int v0, int n_rows, int k0, int nk, int n_dest,
                                    float* const* dest, const int* dest_k0, int mode,
                                    void* stream);

/* Whole FDK on device: filter views 0..n_views-1 of raw_dev ([n_views][Nv][Nu])
 * into stream-ordered scratch and back-project them into vol_dev ([Nz][Ny][Nx]),
 * overwriting it.  raw_dev is left unchanged. */
ifdk_status ifdk_reconstruct(const ifdk_geometry* g, const float* raw_dev, long n_views,
                             float* vol_dev, void* stream);

/* End-to-end FDK from HOST memory: raw_host ([n_views][Nv][Nu] fp32) is copied
 * to the device in view batches (overlapped with filtering), filtered,
 * back-projected, and the volume is copied back into vol_host ([Nz][Ny][Nx]).
 * Host buffers should be page-locked (cudaHostAlloc / cudaHostRegister) for
 * full PCIe bandwidth.  Synchronous: returns after vol_host is written. */
ifdk_status ifdk_reconstruct_host(const ifdk_geometry* g, const float* raw_host, long n_views,
                                  float* vol_host, void* stream);

/* MEASURED BASELINE, not the production path: the paper's
 * straightforward kernel -- Alg. alg:bp per voxel with fp32
 * coordinates [x,y,z] = P_s [i,j,k,1] -- with the bilinear sample of Alg.
 * alg:subpixel taken by the texture unit (texture = 1: cudaFilterModeLinear,
 * 8-bit fixed-point weights, border mode = per-tap zero border) or in software
 * from global memory (texture = 0).  filtered_dev holds all Nv rows of each view
 * ([n_views][Nv][Nu]); vol_dev is the slab k0..k0+nk-1 ([nk][Ny][Nx]),
 * overwritten (accumulate = 0) or added to (1).  Its error against the fp64
 * oracle exceeds the tolerance ifdk_backproject meets.
 * texture = 1 allocates a layered CUDA array per 256 views and synchronises
 * `stream` before returning.  Errors as ifdk_backproject. */
ifdk_status ifdk_backproject_alg2(const ifdk_geometry* g, const float* filtered_dev, long s0,
                                  long n_views, float* vol_dev, int k0, int nk, int accumulate,
                                  int texture, void* stream);

/* The k-slab split without any exchange ("zero-exchange"): the volume slab
 * k0..k0+nk-1 reconstructed from host views by copying only the detector row band the slab
 * needs (ifdk_band_rows over all views; filtering is row-separable, Alg. alg:filter line 3,
 * P:396), filtering it and back-projecting it -- what one GPU of an N-GPU split does with no
 * inter-GPU traffic at all.  raw_host: [n_views][Nv][Nu] fp32 host (pinned for overlap);
 * vol_host: [nk][Ny][Nx] fp32 host.  Pipelined like ifdk_reconstruct_host; synchronous.
 * Values equal ifdk_reconstruct's slab within fp32 rounding (rows pair up differently in the
 * filter's complex transforms).  Errors: INVALID_ARGUMENT (NULL), SHAPE (slab outside
 * [0, Nz), n_views < 0), OUT_OF_MEMORY. */
ifdk_status ifdk_reconstruct_slab_host(const ifdk_geometry* g, const float* raw_host,
                                       long n_views, int k0, int nk, float* vol_host,
                                       void* stream);

/* MEASURED BASELINE (not the production path): the paper's proposed Alg. alg:bp-v1
 * as printed, in fp32 like the paper: per column and view the two
 * inner products x, z, then per k < N_z/2 the one inner product y and the mirrored
 * sample for slice N_z-1-k (Theorem 1, v~ = N_v-1-v).  Whole volume only ([Nz][Ny][Nx]);
 * filtered_dev as for ifdk_backproject_alg2 (all N_v rows); texture = 1 samples through
 * the texture unit.  Kept to re-measure the paper's claimed speed-up of Alg. alg:bp-v1
 * over Alg. alg:bp on B200.  Errors as ifdk_backproject_alg2. */
ifdk_status ifdk_backproject_alg4(const ifdk_geometry* g, const float* filtered_dev, long s0,
                                  long n_views, float* vol_dev, int accumulate, int texture,
                                  void* stream);

/* ---- iterative reconstruction (SART / SIRT) ---- */

/* The matched forward projector: the exact transpose of ifdk_backproject
 * (Alg. alg:bp + alg:subpixel; reading c-I1).  For views s0..s0+n_views-1,
 *   proj_dev[t][v-v0][u] (=|+=) sum over the slab k0..k0+nk-1 of
 *                               f^2 . w_(u,v)(x f, y f) . vol_dev[k-k0][j][i],
 * [x,y,z] = P_s.[i,j,k,1], f = 1/z, w the bilinear weight of detector tap (u,v) in
 * Alg. alg:subpixel (0 unless (u,v) is one of the four taps).  Taps off the
 * detector are dropped (reading c-A9).  vol_dev: [nk][Ny][Nx] fp32 device;
 * proj_dev: [n_views][n_rows][Nu] fp32 device holding rows v0..v0+n_rows-1, which
 * must cover ifdk_band_rows(k0,nk,s) for every view, else SHAPE (a dropped tap
 * would break the adjoint).  accumulate = 0 overwrites the band, 1 adds to it.
 * The sums are order-dependent fp32 atomics: not bitwise reproducible.
 * Errors: INVALID_ARGUMENT (NULL, accumulate not 0/1), SHAPE (as ifdk_backproject). */
ifdk_status ifdk_forward_project(const ifdk_geometry* g, const float* vol_dev, int k0, int nk,
                                 long s0, long n_views, float* proj_dev, int v0, int n_rows,
                                 int accumulate, void* stream);

/* SART residual step (reading c-I2): out[e] = (b[e] - ax[e]) / R[e], 0 where
 * R[e] <= 0 (rays no voxel reaches, reading c-I3).  R = forward projection of a
 * volume of ones.  n elements, fp32 device; out may alias ax.
 * Errors: INVALID_ARGUMENT (NULL), SHAPE (n < 0). */
ifdk_status ifdk_sart_ratio(const float* b_dev, const float* ax_dev, const float* R_dev,
                            float* out_dev, long n, void* stream);

/* SART update step (reading c-I2): x[e] += lambda c[e] / C[e], unchanged where
 * C[e] <= 0 (voxels no ray sees, reading c-I3); nonneg = 1 then clamps x at 0.
 * c = back-projection of the residual ratio, C = back-projection of ones.
 * Errors: INVALID_ARGUMENT (NULL, lambda outside (0, 2), nonneg not 0/1), SHAPE. */
ifdk_status ifdk_sart_update(float* x_dev, const float* c_dev, const float* C_dev, float lambda,
                             long n, int nonneg, void* stream);

/* MLEM / OS-EM ratio step (Shepp & Vardi, cited at P:266; reading c-I4):
 * out[e] = b[e] / ax[e] where ax[e] > 0, else 0.  ax = forward projection of the current
 * estimate; out may alias ax.  Errors: INVALID_ARGUMENT (NULL), SHAPE (n < 0). */
ifdk_status ifdk_mlem_ratio(const float* b_dev, const float* ax_dev, float* out_dev, long n,
                            void* stream);

/* MLEM / OS-EM multiplicative update (reading c-I4): x[e] = x[e] c[e] / C[e] where
 * C[e] > 0 (C = back-projection of ones), else x[e] unchanged.  c = back-projection of
 * the ratio.  Errors: INVALID_ARGUMENT (NULL), SHAPE (n < 0). */
ifdk_status ifdk_mlem_update(float* x_dev, const float* c_dev, const float* C_dev, long n,
                             void* stream);

/* x[e] = value for n fp32 device elements (normaliser inputs of SART).
 * Errors: INVALID_ARGUMENT (NULL), SHAPE (n < 0). */
ifdk_status ifdk_fill(float* x_dev, float value, long n, void* stream);

/* Speed-tuning hook for A/B measurements and tests, not needed in normal use:
 * walk selects the back-projection k-walk; within a family the variants give
 * BITWISE the same result (PAIR family 2, 4, 5; 4-row TRIPLE family 3, 6, 9, 11
 * where 0.5 <= dv/dk; 3-row TRIPLE family 7, 8, 10, 12 where dv/dk < 0.5; 9-12
 * keep the accumulators in tensor memory, 11 / 12 step two views at a time), and
 * the QUAD walk 13 (the automatic choice where 0.5 <= dv/dk < 1: four slices per
 * floor, tensor-memory accumulators, two views per step, partial chunks in the
 * same kernel), the QUINT walk 14 (five slices per floor, the automatic choice
 * where dv/dk < 0.5) and QUINT-HI 15 (five slices where 0.5 <= dv/dk < 1) are
 * families of their own -- they agree with the others to fp32 rounding, not
 * bitwise.  A walk outside the geometry's range, or 0,
 * means automatic.
 * raster sets the CTA raster band in tiles (0 = automatic; >= the tile count =
 * row-major); it only reorders CTAs.  Process-wide; affects later launches. */
ifdk_status ifdk_set_bp_variant(int walk, int raster);

/* Number of device kernels the last successful call on this thread launched. */
int ifdk_last_launch_count(void);

/* Thread-local message describing the last non-OK status ("" if none). */
const char* ifdk_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* IFDK_H */
