"""Pins of the iterative-reconstruction oracle (DESIGN.md readings
c-I1..c-I4): the matched forward projector, SART / SIRT and MLEM / OS-EM, checked against what the
mathematics fixes -- the adjoint identity with the (independently pinned) back-projector,
a brute-force ray construction of every splat, closed forms on the rotation axis and
Eq. equ:z, the exact one-step solution of a single-voxel system, and the monotone decrease
of SIRT's weighted residual and of MLEM's Kullback-Leibler divergence."""
import math

import numpy as np

import oracle
from oracle import OracleGeometry
from test_oracle_pins import _random_geom, _ray_uvz


def _small(rng):
    g = _random_geom(rng, small=True)
    # keep the volume inside the source circle (as the BP brute-force pin does)
    return OracleGeometry(g.Nu, g.Nv, g.Nx, g.Ny, g.Nz, g.Du, g.Dv, 1.0, 1.0, 1.0, 30.0, 20.0,
                          g.theta)


def test_forward_projector_is_the_adjoint_of_backprojection():
    """<M x, y> = <x, M^T y> with M^T = Alg. alg:bp (oracle.backproject_volume, pinned in
    test_oracle_pins.py) for random volumes, projections, view offsets and slabs: a dropped
    tap, a wrong weight or a transposed index breaks it."""
    rng = np.random.default_rng(7)
    for _ in range(20):
        g = _small(rng)
        n = int(rng.integers(1, 6))
        s0 = int(rng.integers(0, 50))
        k0 = int(rng.integers(0, g.Nz))
        nk = int(rng.integers(1, g.Nz - k0 + 1))
        x = rng.standard_normal((nk, g.Ny, g.Nx))
        y = rng.standard_normal((n, g.Nv, g.Nu))
        lhs = float((oracle.forward_project(g, x, s0, n, k0=k0) * y).sum())
        rhs = float((x * oracle.backproject_volume(g, y, s0=s0, k0=k0, nk=nk)).sum())
        assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs)), (lhs, rhs)


def test_forward_projector_bruteforce_ray_splat():
    """Every voxel of a tiny volume splatted by hand: (u, v, z) from the independent
    ray-plane construction of the scanner (reading c-A15), four bilinear taps with weights
    (1-du)(1-dv), du(1-dv), (1-du)dv, du dv times W = 1/z^2, taps off the detector dropped."""
    rng = np.random.default_rng(11)
    for _ in range(8):
        g = _small(rng)
        n = int(rng.integers(1, 4))
        s0 = int(rng.integers(0, 40))
        x = rng.standard_normal((g.Nz, g.Ny, g.Nx))
        got = oracle.forward_project(g, x, s0, n)
        ref = np.zeros((n, g.Nv, g.Nu))
        for t in range(n):
            for k in range(g.Nz):
                for j in range(g.Ny):
                    for i in range(g.Nx):
                        u, v, z = _ray_uvz(g, s0 + t, i, j, k)
                        nu, nv = math.floor(u), math.floor(v)
                        du, dv = u - nu, v - nv
                        for a, b, w in ((nu, nv, (1 - du) * (1 - dv)), (nu + 1, nv, du * (1 - dv)),
                                        (nu, nv + 1, (1 - du) * dv), (nu + 1, nv + 1, du * dv)):
                            if 0 <= a < g.Nu and 0 <= b < g.Nv:
                                ref[t, b, a] += w * x[k, j, i] / (z * z)
        assert np.max(np.abs(got - ref)) <= 1e-12 * max(1.0, np.max(np.abs(ref)))


def test_forward_projector_center_voxel_on_axis():
    """Odd volume and detector: the centre voxel sits on the rotation axis, so z = d for
    every view (Eq. equ:z with X = Y = 0) and it projects onto the detector centre
    (c_u, c_v), an integer pixel: one non-zero tap of value x / d^2 per view."""
    d = 20.0
    g = OracleGeometry(9, 7, 5, 5, 5, 1.0, 1.0, 1.0, 1.0, 1.0, 40.0, d, 2 * math.pi / 10)
    x = np.zeros((5, 5, 5))
    x[2, 2, 2] = 3.0
    F = oracle.forward_project(g, x, 0, 10)
    for t in range(10):
        nz = np.argwhere(np.abs(F[t]) > 1e-14)
        assert nz.tolist() == [[3, 4]]
        assert abs(F[t, 3, 4] - 3.0 / d ** 2) < 1e-15


def test_forward_projector_mass_equals_equ_z_weights():
    """When every tap of every voxel lands on the detector, the bilinear weights of a voxel
    sum to 1, so sum over the detector of (M x)_s = sum_voxels x / z_s^2 with the depth z
    from Eq. equ:z (z = d + sin(b) X - cos(b) Y), computed here independently of P."""
    rng = np.random.default_rng(5)
    g = OracleGeometry(64, 64, 6, 7, 5, 1.0, 1.0, 1.0, 1.0, 1.0, 60.0, 30.0, 0.29)
    x = rng.standard_normal((5, 7, 6))
    F = oracle.forward_project(g, x, 2, 4)
    for t in range(4):
        b = (2 + t) * g.theta
        ref = 0.0
        for k in range(5):
            for j in range(7):
                for i in range(6):
                    X = g.Dx * (i - (g.Nx - 1) / 2)
                    Y = g.Dy * (j - (g.Ny - 1) / 2)
                    z = g.d + math.sin(b) * X - math.cos(b) * Y
                    ref += x[k, j, i] / z ** 2
        assert abs(F[t].sum() - ref) <= 1e-12 * max(1.0, abs(ref))


def test_sart_single_voxel_exact_in_one_step():
    """One voxel, any views: M is one column a, R_i = a_i, C = sum a_i, so one SART step
    from 0 with lambda = 1 gives sum_i a_i (b_i / a_i) / sum_i a_i = sum b / sum a, which is
    x_true exactly for consistent data b = a x_true (reading c-I2)."""
    g = OracleGeometry(7, 6, 1, 1, 1, 1.0, 1.0, 1.0, 1.0, 1.0, 40.0, 20.0, 0.7)
    b = oracle.forward_project(g, np.full((1, 1, 1), 2.5), 0, 5)
    x = oracle.sart(g, b, 1, lam=1.0)
    assert abs(x[0, 0, 0] - 2.5) < 1e-13


def test_sirt_weighted_residual_decreases_monotonically():
    """SIRT (one subset = all views) with 0 < lambda < 2 is a gradient step on the
    R-weighted residual sum_i (b_i - (Mx)_i)^2 / R_i in the C-weighted metric, which
    therefore decreases monotonically on consistent data; OS-SART reaches a small residual."""
    rng = np.random.default_rng(3)
    g = OracleGeometry(16, 12, 6, 6, 5, 1.0, 1.0, 1.0, 1.0, 1.0, 50.0, 25.0, 2 * math.pi / 12)
    x_true = rng.uniform(0, 1, (5, 6, 6))
    b = oracle.forward_project(g, x_true, 0, 12)
    R = oracle.forward_project(g, np.ones((5, 6, 6)), 0, 12)

    def wres(x):
        r = b - oracle.forward_project(g, x, 0, 12)
        return float(np.sum(np.where(R > 0, r * r / np.where(R > 0, R, 1.0), 0.0)))

    x = np.zeros((5, 6, 6))
    prev = wres(x)
    for _ in range(8):
        x = oracle.sart(g, b, 1, lam=1.5, x0=x)
        cur = wres(x)
        assert cur < prev
        prev = cur
    xo = oracle.sart(g, b, 10, lam=1.0, block=3)
    assert wres(xo) < 1e-3 * wres(np.zeros_like(xo))


def test_mlem_single_voxel_exact_in_one_step():
    """One voxel: x1 = x0 / sum a * sum_i a_i b_i / (a_i x0) = sum b / sum a, which is x_true for
    consistent data, from any positive start (reading c-I4)."""
    g = OracleGeometry(7, 6, 1, 1, 1, 1.0, 1.0, 1.0, 1.0, 1.0, 40.0, 20.0, 0.7)
    b = oracle.forward_project(g, np.full((1, 1, 1), 2.5), 0, 5)
    for x0 in (1.0, 0.3):
        x = oracle.mlem(g, b, 1, x0=np.full((1, 1, 1), x0))
        assert abs(x[0, 0, 0] - 2.5) < 1e-13


def test_mlem_keeps_positivity_and_decreases_kl():
    """MLEM on consistent non-negative data keeps the estimate positive and decreases the
    Kullback-Leibler divergence KL(b || M x) = sum b log(b / Mx) - b + Mx monotonically
    (the EM property); OS-EM reaches a small divergence."""
    rng = np.random.default_rng(9)
    g = OracleGeometry(16, 12, 6, 6, 5, 1.0, 1.0, 1.0, 1.0, 1.0, 50.0, 25.0, 2 * math.pi / 12)
    x_true = rng.uniform(0.2, 1, (5, 6, 6))
    b = oracle.forward_project(g, x_true, 0, 12)

    def kl(x):
        ax = oracle.forward_project(g, x, 0, 12)
        m = b > 0
        return float(np.sum(b[m] * np.log(b[m] / ax[m])) - b.sum() + ax.sum())

    x = np.ones((5, 6, 6))
    prev = kl(x)
    for _ in range(6):
        x = oracle.mlem(g, b, 1, x0=x)
        assert x.min() > 0
        cur = kl(x)
        assert cur < prev
        prev = cur
    xo = oracle.mlem(g, b, 10, block=3)
    assert kl(xo) < 1e-2 * kl(np.ones((5, 6, 6)))
