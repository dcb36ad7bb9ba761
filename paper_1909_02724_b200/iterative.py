"""SART / SIRT on the GPU from the library's operators.

The paper's back-projection "can be adopted by iterative reconstruction methods, in which
the back-projection is required to be repeated dozens of times, e.g. ART, SART, MLEM"
(P:266).  This driver reuses BP-sm100 (``ifdk_backproject``, Alg. alg:bp) as M^T
and its exact transpose ``ifdk_forward_project`` as M (reading c-I1), with the textbook
SART update of Andersen & Kak (cited at P:266; reading c-I2) over ordered subsets of
consecutive views:

    x <- x + lam * M_S^T((b_S - M_S x) / R_S) / C_S,   R_S = M_S 1,  C_S = M_S^T 1,

terms with a zero normaliser left out (reading c-I3).  One subset holding every view is
SIRT.  MLEM / OS-EM (Shepp & Vardi, also cited at P:266; reading c-I4) uses the same two
operators with the multiplicative update  x <- x * M_S^T(b_S / M_S x) / C_S.  Every arithmetic
step runs in libifdk kernels; torch only allocates the buffers.
"""
from __future__ import annotations

from .ifdk import (
    Geometry,
    ifdk_backproject,
    ifdk_fill,
    ifdk_forward_project,
    ifdk_mlem_ratio,
    ifdk_mlem_update,
    ifdk_sart_ratio,
    ifdk_sart_update,
)


class SART:
    """Reusable SART state for one geometry and one set of measured projections.

    b: [Np][Nv][Nu] float32 CUDA tensor, views 0..Np-1.  block: views per subset (None = all
    views, i.e. SIRT).  The normalisers R_S (projection-sized) and C_S (volume-sized) of every
    subset are computed once and kept when `cache_C` (memory: one volume per subset)."""

    def __init__(self, g: Geometry, b, block: int | None = None, cache_C: bool = True):
        import torch

        self.g, self.b = g, b
        Np = b.shape[0]
        self.block = block or Np
        self.subsets = [(s0, min(self.block, Np - s0)) for s0 in range(0, Np, self.block)]
        dev = b.device
        vol_shape = (g.Nz, g.Ny, g.Nx)
        self.ax = torch.empty((self.block, g.Nv, g.Nu), device=dev)
        self.c = torch.empty(vol_shape, device=dev)
        ones_vol = torch.empty(vol_shape, device=dev)
        ifdk_fill(ones_vol, 1.0)
        # R = M 1 for all views at once (projection-sized, sliced per subset)
        self.R = torch.empty_like(b)
        ifdk_forward_project(g, ones_vol, 0, self.R)
        del ones_vol
        self.ones_proj = torch.empty((self.block, g.Nv, g.Nu), device=dev)
        ifdk_fill(self.ones_proj, 1.0)
        self.cache_C = cache_C
        self.C = [self._column_sums(s0, n) for s0, n in self.subsets] if cache_C else None

    def _column_sums(self, s0: int, n: int):
        import torch

        C = torch.empty((self.g.Nz, self.g.Ny, self.g.Nx), device=self.b.device)
        ifdk_backproject(self.g, self.ones_proj[:n], s0, C)
        return C

    def iterate(self, x, n_iter: int = 1, lam: float = 1.0, nonneg: bool = False):
        """n_iter passes over all subsets, updating x ([Nz][Ny][Nx], float32 CUDA) in place."""
        g = self.g
        for _ in range(n_iter):
            for q, (s0, n) in enumerate(self.subsets):
                ax = self.ax[:n]
                ifdk_forward_project(g, x, s0, ax)                            # M_S x
                ifdk_sart_ratio(self.b[s0:s0 + n], ax, self.R[s0:s0 + n], ax)  # (b - Mx) / R
                ifdk_backproject(g, ax, s0, self.c)                           # M_S^T (...)
                C = self.C[q] if self.cache_C else self._column_sums(s0, n)
                ifdk_sart_update(x, self.c, C, lam, nonneg)                    # x += lam c / C
        return x


def sart(g: Geometry, b, n_iter: int, lam: float = 1.0, block: int | None = None, x0=None,
         nonneg: bool = False):
    """SART (block views per subset) or SIRT (block=None) from x0 (default 0)."""
    import torch

    x = torch.empty((g.Nz, g.Ny, g.Nx), device=b.device)
    if x0 is None:
        ifdk_fill(x, 0.0)
    else:
        x.copy_(x0)
    return SART(g, b, block).iterate(x, n_iter, lam, nonneg)


def mlem(g: Geometry, b, n_iter: int, block: int | None = None, x0=None):
    """MLEM (block=None) or OS-EM (block views per subset) from x0 (default 1 everywhere):
    x <- x * M_S^T(b_S / M_S x) / M_S^T 1 per subset (reading c-I4)."""
    import torch

    Np = b.shape[0]
    block = block or Np
    subsets = [(s0, min(block, Np - s0)) for s0 in range(0, Np, block)]
    dev = b.device
    x = torch.empty((g.Nz, g.Ny, g.Nx), device=dev)
    if x0 is None:
        ifdk_fill(x, 1.0)
    else:
        x.copy_(x0)
    ax = torch.empty((block, g.Nv, g.Nu), device=dev)
    c = torch.empty_like(x)
    ones_proj = torch.empty((block, g.Nv, g.Nu), device=dev)
    ifdk_fill(ones_proj, 1.0)
    C = []
    for s0, n in subsets:
        Cq = torch.empty_like(x)
        ifdk_backproject(g, ones_proj[:n], s0, Cq)
        C.append(Cq)
    for _ in range(n_iter):
        for q, (s0, n) in enumerate(subsets):
            a = ax[:n]
            ifdk_forward_project(g, x, s0, a)              # M_S x
            ifdk_mlem_ratio(b[s0:s0 + n], a, a)            # b / M_S x
            ifdk_backproject(g, a, s0, c)                  # M_S^T (...)
            ifdk_mlem_update(x, c, C[q])                   # x * c / C
    return x
