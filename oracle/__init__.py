"""Double-precision CPU oracle for the iFDK hot path (arXiv 1909.02724).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import,
call, link or execute anything under ``oracle/``.  The product package
``paper_1909_02724_b200`` never imports it and shares no code with it.

What it computes (all fp64; the only fp32 quantity is the raw input E):

* ``projection_matrix``  -- P_s = (M1 . Mrot . M0)[0:3], appendix P:15-82.
* ``cos_weight``, ``ramp_h1``, ``fdk_scale`` -- F_cos, F_ramp and the FDK
  constant (readings c-A5, c-A6, c-A7 in DESIGN.md).
* ``filter_direct``      -- Alg. alg:filter, direct linear
  convolution written out as the sum.
* ``filter_fft``         -- the same convolution through the convolution
  theorem with a library fp64 FFT; pinned to ``filter_direct``.
* ``interp2``            -- Alg. alg:subpixel, floor + per-tap
  zero border (readings c-A8, c-A9).
* ``backproject``        -- Alg. alg:bp on a voxel list or a
  k-slab of the volume.
* ``reconstruct``        -- filter then back-project (the FDK of P:366-454).
* ``forward_project``    -- the matched forward projector, the transpose of
  Alg. alg:bp + alg:subpixel (reading c-I1); pinned by the adjoint identity
  against ``backproject_volume`` and by closed forms.
* ``sart``               -- SART / SIRT (Andersen & Kak, cited at P:266;
  readings c-I2, c-I3) built from the two operators.
* ``mlem``               -- MLEM / OS-EM (Shepp & Vardi, cited at P:266; reading
  c-I4), the multiplicative update from the same operators.

Parity pins live in ``tests/test_oracle_pins.py``.  Functions whose result
the paper does not fix (the F_cos formula, the ramp shape, the constant C,
the detector-edge rule) are conventions: "parity unpinned" by the paper, see
DESIGN.md section "Readings".
"""
from .oracle import (  # noqa: F401
    OracleGeometry,
    backproject,
    backproject_volume,
    build,
    cos_weight,
    fdk_scale,
    filter_direct,
    filter_fft,
    forward_project,
    interp2,
    mlem,
    num_threads,
    projection_matrix,
    ramp_h1,
    reconstruct,
    sart,
)
