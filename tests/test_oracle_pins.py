"""Pins of the fp64 oracle against what the paper and mathematics fix.

Each test pins the oracle to something other than itself: a hand expansion of
the printed matrices, an independent ray construction of the scanner, the
closed form of Eq. equ:z, Theorems 1-3, the Ram-Lak Fourier series, the
convolution theorem, worked interpolation examples, brute force on tiny
inputs, the paper's own Alg. alg:bp-v1, and the analytic Shepp-Logan phantom.
"""
import math
import os

import numpy as np
import pytest

import oracle
import synth
from oracle import OracleGeometry

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    out = []
    with open(os.path.join(GOLD, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                out.append([float(x) for x in line.split()])
    return out


def _geom(Nu, Nv, Nx, Ny, Nz, Du, Dv, Dx, Dy, Dz, D, d, theta):
    return OracleGeometry(int(Nu), int(Nv), int(Nx), int(Ny), int(Nz), Du, Dv, Dx, Dy, Dz, D, d, theta)


def _random_geom(rng, small=False):
    N = rng.integers(3, 9) if small else rng.integers(4, 300)
    Nx, Ny, Nz = (int(rng.integers(3, 9)) for _ in range(3)) if small else (
        int(N), int(rng.integers(4, 300)), int(rng.integers(4, 300)))
    Nu, Nv = (int(rng.integers(4, 12)) for _ in range(2)) if small else (
        int(rng.integers(8, 600)), int(rng.integers(8, 600)))
    d = float(rng.uniform(200, 1500))
    D = d * float(rng.uniform(1.1, 2.5))
    Dx, Dy = float(rng.uniform(0.05, 1.0)), float(rng.uniform(0.05, 1.0))
    Dz = float(rng.uniform(0.05, 1.0))
    Du, Dv = float(rng.uniform(0.1, 1.5)), float(rng.uniform(0.1, 1.5))
    theta = float(rng.uniform(0.001, 1.0))
    return _geom(Nu, Nv, Nx, Ny, Nz, Du, Dv, Dx, Dy, Dz, D, d, theta)


def _ray_uvz(g, s, i, j, k):
    """Independent scanner construction (reading c-A15): source at
    (-d sin b, -d cos b, 0), detector plane at distance D with centre on the
    central ray, u axis (cos b, -sin b, 0), v axis (0, 0, -1); voxel (i,j,k) at
    (Dx(i-cx), -Dy(j-cy), -Dz(k-cz)).  Ray-plane intersection -> (u, v, z)."""
    b = s * g.theta
    cb, sb = math.cos(b), math.sin(b)
    S = np.array([-g.d * sb, -g.d * cb, 0.0])
    n = np.array([sb, cb, 0.0])
    Dc = S + g.D * n
    eu = np.array([cb, -sb, 0.0])
    ev = np.array([0.0, 0.0, -1.0])
    p = np.array([g.Dx * (i - (g.Nx - 1) / 2), -g.Dy * (j - (g.Ny - 1) / 2),
                  -g.Dz * (k - (g.Nz - 1) / 2)])
    z = float((p - S) @ n)
    q = S + (p - S) * (g.D / z)
    u = (g.Nu - 1) / 2 + float((q - Dc) @ eu) / g.Du
    v = (g.Nv - 1) / 2 + float((q - Dc) @ ev) / g.Dv
    return u, v, z


def _P_uvz(P, i, j, k):
    x, y, z = P @ np.array([i, j, k, 1.0])
    return x / z, y / z, z


# ------------------------------------------------------------------ geometry
def test_projection_matrix_hand_expansion():
    rows = _rows("projection_matrix_tiny.txt")
    gvals, P_exp = rows[0], np.array(rows[1:4])
    g = _geom(*gvals[:13])
    P = oracle.projection_matrix(g, int(gvals[13]))
    np.testing.assert_allclose(P, P_exp, rtol=0, atol=1e-13)


def test_projection_matrix_matches_ray_construction():
    rng = np.random.default_rng(7)
    worst = 0.0
    for _ in range(300):
        g = _random_geom(rng)
        s = int(rng.integers(-50, 5000))
        P = oracle.projection_matrix(g, s)
        for _ in range(5):
            i, j, k = (float(rng.integers(0, n)) for n in (g.Nx, g.Ny, g.Nz))
            u1, v1, z1 = _P_uvz(P, i, j, k)
            u2, v2, z2 = _ray_uvz(g, s, i, j, k)
            worst = max(worst, abs(u1 - u2), abs(v1 - v2), abs(z1 - z2) / z2)
    assert worst < 1e-9


def test_depth_closed_form_equ_z():
    """Eq. equ:z: z = d + sin(b)(i-cx)Dx - cos(b)(j-cy)Dy, any k."""
    rng = np.random.default_rng(3)
    for _ in range(200):
        g = _random_geom(rng)
        s = int(rng.integers(0, 10000))
        P = oracle.projection_matrix(g, s)
        b = s * g.theta
        for _ in range(5):
            i, j, k = (float(rng.integers(0, n)) for n in (g.Nx, g.Ny, g.Nz))
            z = P[2] @ np.array([i, j, k, 1.0])
            zc = g.d + math.sin(b) * (i - (g.Nx - 1) / 2) * g.Dx - math.cos(b) * (j - (g.Ny - 1) / 2) * g.Dy
            assert abs(z - zc) <= 1e-12 * abs(zc)


def test_theorems_1_2_3():
    """Theorem-2/3: u and z constant along k; Theorem-1:
    v(k) + v(Nz-1-k) = Nv - 1."""
    rng = np.random.default_rng(11)
    for _ in range(100):
        g = _random_geom(rng)
        s = int(rng.integers(0, 4096))
        P = oracle.projection_matrix(g, s)
        assert P[0, 2] == 0.0 and P[2, 2] == 0.0
        i, j = float(rng.integers(0, g.Nx)), float(rng.integers(0, g.Ny))
        ks = np.arange(g.Nz, dtype=np.float64)
        uvz = np.array([_P_uvz(P, i, j, k) for k in ks])
        assert np.ptp(uvz[:, 2]) <= 1e-12 * abs(uvz[0, 2])
        assert np.ptp(uvz[:, 0]) <= 1e-9
        vs = uvz[:, 1]
        np.testing.assert_allclose(vs + vs[::-1], g.Nv - 1, rtol=0, atol=1e-9)


def test_special_cases_center_and_z13():
    """beta=0 centre voxel -> z=d, (u,v) = detector centre.
    S:73: beta=pi/2, d=10, Dx=1, i=cx+3 -> z = 13."""
    g = _geom(9, 7, 5, 5, 5, 0.7, 0.9, 1, 1, 1, 20.0, 10.0, math.pi / 2)
    P = oracle.projection_matrix(g, 0)
    u, v, z = _P_uvz(P, 2, 2, 2)
    assert abs(z - 10.0) < 1e-14 and abs(u - 4.0) < 1e-13 and abs(v - 3.0) < 1e-13
    g2 = _geom(8, 8, 7, 7, 7, 1, 1, 1, 1, 1, 20.0, 10.0, math.pi / 2)
    P = oracle.projection_matrix(g2, 1)
    for j in range(7):
        assert abs(_P_uvz(P, 3 + 3, j, 0)[2] - 13.0) < 1e-13


# ------------------------------------------------------------------ filter
def test_cos_weight_examples_and_symmetry():
    for D, Du, Dv, Nu, Nv, m, v, exp in _rows("cos_weight.txt"):
        g = _geom(Nu, Nv, 4, 4, 4, Du, Dv, 1, 1, 1, D, D / 2, 0.1)
        assert abs(oracle.cos_weight(g, int(m), int(v)) - exp) < 1e-14
    g = _geom(13, 10, 4, 4, 4, 0.3, 0.45, 1, 1, 1, 300.0, 200.0, 0.1)
    for m in range(13):
        for v in range(10):
            w = oracle.cos_weight(g, m, v)
            assert 0 < w <= 1
            assert abs(w - oracle.cos_weight(g, 12 - m, 9 - v)) < 1e-15


def test_ramp_taps_and_frequency_response():
    for n, exp in _rows("ramp_taps.txt"):
        assert abs(oracle.ramp_h1(int(n)) - exp) < 1e-16
    # DTFT of h1 is |w|/(2 pi) on [-pi, pi]: sum_{n odd} cos(n w)/n^2 = pi(pi-2|w|)/8.
    N = 20001
    n = np.arange(-N, N + 1)
    h = np.array([oracle.ramp_h1(int(t)) for t in n])
    for w in (0.0, 0.3, 1.0, 2.0, 3.0, math.pi):
        Hw = float(np.sum(h * np.cos(n * w)))
        assert abs(Hw - abs(w) / (2 * math.pi)) < 2.0 / (math.pi ** 2 * N)


def test_filter_impulse_response():
    """A single unit sample at m0 filters to C * F_cos(m0, v) * h1[n - m0]."""
    g = _geom(37, 5, 8, 8, 8, 0.8, 0.6, 0.5, 0.5, 0.5, 900.0, 600.0, 2 * math.pi / 90)
    E = np.zeros((1, 5, 37), np.float32)
    E[0, 3, 11] = 1.0
    Q = oracle.filter_direct(g, E)
    C = oracle.fdk_scale(g)
    assert abs(C - g.theta * g.d * g.D / (2 * g.Du)) < 1e-12 * C
    exp = np.array([C * oracle.cos_weight(g, 11, 3) * oracle.ramp_h1(n - 11) for n in range(37)])
    np.testing.assert_allclose(Q[0, 3], exp, rtol=1e-14, atol=1e-14 * C)
    assert np.all(Q[0, [0, 1, 2, 4]] == 0)


def test_filter_fft_equals_direct_and_linearity():
    rng = np.random.default_rng(5)
    for Nu, Nv, v0 in ((64, 6, 0), (33, 4, 10), (200, 3, 7)):
        g = _geom(Nu, Nv + v0 + 2, 8, 8, 8, 0.4, 0.3, 0.5, 0.5, 0.5, 700.0, 500.0, 0.05)
        E = rng.standard_normal((2, Nv, Nu)).astype(np.float32)
        Qd = oracle.filter_direct(g, E, v0=v0)
        Qf = oracle.filter_fft(g, E, v0=v0)
        assert np.max(np.abs(Qd - Qf)) <= 1e-12 * np.max(np.abs(Qd))
        Q2 = oracle.filter_direct(g, (2 * E).astype(np.float32), v0=v0)
        np.testing.assert_allclose(Q2, 2 * Qd, rtol=1e-14, atol=1e-14 * np.max(np.abs(Qd)))
    assert np.all(oracle.filter_direct(g, np.zeros((1, 2, Nu), np.float32)) == 0)


# ------------------------------------------------------------------ interpolation
def test_interp2_worked_examples_and_border():
    g = _geom(2, 2, 4, 4, 4, 1, 1, 1, 1, 1, 20, 10, 0.1)
    Q = np.array([[0.0, 1.0], [2.0, 3.0]])
    for u, v, exp in _rows("interp2_2x2.txt"):
        val, miss = oracle.interp2(g, Q, u, v)
        assert abs(val - exp) < 1e-15 and not miss
    # per-tap zero border (reading c-A9): continuous across the edge
    assert oracle.interp2(g, Q, -1.0, 0.0)[0] == 0.0
    assert abs(oracle.interp2(g, Q, -0.5, 0.0)[0] - 0.0) < 1e-15  # 0.5*0 + 0.5*X(0,0)
    assert abs(oracle.interp2(g, Q, 1.5, 1.0)[0] - 1.5) < 1e-15  # 0.5*3 + 0.5*0
    assert abs(oracle.interp2(g, Q, 1.0 + 1e-9, 1.0)[0] - 3.0) < 1e-8
    # floor, not truncation (reading c-A8): u = -0.25 is 0.75 of X(0, .)
    assert abs(oracle.interp2(g, Q, -0.25, 1.0)[0] - 0.75 * 2.0) < 1e-15


# ------------------------------------------------------------------ back-projection
def test_bp_uniform_projection_center_voxel():
    """Q = 1, odd N, centre voxel on the rotation axis: z = d for every view and
    the tap lands on the detector centre, so V = Np / d^2."""
    Np, d = 12, 20.0
    g = _geom(9, 9, 5, 5, 5, 1, 1, 1, 1, 1, 40.0, d, 2 * math.pi / Np)
    Q = np.ones((Np, 9, 9))
    V = oracle.backproject(g, Q, np.array([[2, 2, 2]]))
    assert abs(V[0] - Np / d ** 2) < 1e-15


def _bilinear_by_hand(Q, u, v):
    nu, nv = math.floor(u), math.floor(v)
    du, dv = u - nu, v - nv

    def T(a, b):
        return Q[b][a] if 0 <= a < len(Q[0]) and 0 <= b < len(Q) else 0.0

    return ((1 - dv) * ((1 - du) * T(nu, nv) + du * T(nu + 1, nv))
            + dv * ((1 - du) * T(nu, nv + 1) + du * T(nu + 1, nv + 1)))


def test_bp_bruteforce_ray_driven_tiny():
    rng = np.random.default_rng(19)
    for _ in range(12):
        g = _random_geom(rng, small=True)
        # keep the volume inside the source circle
        g = OracleGeometry(g.Nu, g.Nv, g.Nx, g.Ny, g.Nz, g.Du, g.Dv, 1.0, 1.0, 1.0, 30.0, 20.0, g.theta)
        nv = int(rng.integers(1, 8))
        s0 = int(rng.integers(0, 100))
        Q = rng.standard_normal((nv, g.Nv, g.Nu))
        V = oracle.backproject_volume(g, Q, s0=s0)
        for k in range(g.Nz):
            for j in range(g.Ny):
                for i in range(g.Nx):
                    acc = 0.0
                    for t in range(nv):
                        u, v, z = _ray_uvz(g, s0 + t, i, j, k)
                        acc += _bilinear_by_hand(Q[t], u, v) / (z * z)
                    assert abs(V[k, j, i] - acc) <= 1e-12 * max(1.0, abs(acc))


def test_bp_equals_paper_alg_bp_v1():
    """Alg. alg:bp-v1: 2 inner products per column, 1 per k, the
    mirror k~ = Nz-1-k with v~ = Nv-1-v, transposed Q~ read as interp2(Q~, v, u).
    In fp64 it must equal Alg. alg:bp (the oracle)."""
    rng = np.random.default_rng(23)
    for _ in range(8):
        Nz = 2 * int(rng.integers(2, 4))
        g = OracleGeometry(int(rng.integers(5, 11)), int(rng.integers(5, 11)), int(rng.integers(3, 6)),
                           int(rng.integers(3, 6)), Nz, 0.9, 0.8, 1.0, 1.0, 1.0, 40.0, 25.0, 0.37)
        nv = 3
        Q = rng.standard_normal((nv, g.Nv, g.Nu))
        It = np.zeros((g.Nx, g.Ny, g.Nz))  # k-major I~(k, j, i) stored as [i][j][k]
        for s in range(nv):
            P = oracle.projection_matrix(g, s)
            Qt = Q[s].T  # line 3: Q~ = Q^T  ([u][v])
            for j in range(g.Ny):
                for i in range(g.Nx):
                    t = np.array([i, j, 0, 1.0])
                    x, z = P[0] @ t, P[2] @ t
                    f = 1.0 / z
                    u = x * f
                    W = f * f
                    for k in range(Nz // 2):
                        y = P[1] @ np.array([i, j, k, 1.0])
                        v = y * f
                        It[i, j, k] += W * _bilinear_by_hand(Qt.T, u, v)
                        kt, vt = Nz - 1 - k, g.Nv - 1 - v
                        It[i, j, kt] += W * _bilinear_by_hand(Qt.T, u, vt)
        V = oracle.backproject_volume(g, Q)
        np.testing.assert_allclose(V, np.transpose(It, (2, 1, 0)), rtol=1e-12, atol=1e-13)


def test_bp_band_coverage_error():
    g = _geom(16, 16, 4, 4, 4, 1, 1, 1, 1, 1, 40.0, 25.0, 0.2)
    Q = np.ones((2, 4, 16))  # rows 0..3 only, the volume projects to the middle rows
    with pytest.raises(oracle.oracle.BandError):
        oracle.backproject(g, Q, np.array([[2, 2, 2]]), v0=0)


# ------------------------------------------------------------------ whole FDK
def test_fdk_reproduces_phantom_densities():
    """Analytic Shepp-Logan projections -> oracle FDK -> interior means equal
    the phantom densities (pins F_cos, F_ramp and the constant C up to the
    method's discretisation error)."""
    from scipy import ndimage

    spec = synth.config(1)
    g = OracleGeometry(**spec.geometry_args())
    ell = synth.default_ellipsoids(spec)
    E = synth.project(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, 0, spec.Np)
    V = oracle.reconstruct(g, E)
    kk, jj, ii = np.meshgrid(np.arange(spec.Nz), np.arange(spec.Ny), np.arange(spec.Nx), indexing="ij")
    X, Y, Z = synth.voxel_world(spec, ii, jj, kk)
    truth = synth.density(ell, np.stack([X, Y, Z], -1)).reshape(V.shape)
    checked = 0
    for val in (0.2, 0.3, 0.0):
        mask = ndimage.binary_erosion(np.isclose(truth, val), iterations=3)
        if mask.sum() < 50:
            continue
        mean = float(V[mask].mean())
        assert abs(mean - val) < 0.01, (val, mean, int(mask.sum()))
        checked += 1
    assert checked >= 2


def test_fdk_sphere_center_density():
    spec = synth.ConfigSpec("sphere", 90, 96, 96, 64, 64, 64)
    g = OracleGeometry(**spec.geometry_args())
    ell = synth.ellipsoids(1.0, table=((40.0, 40.0, 40.0, 0, 0, 0, 0, 1.0),))
    E = synth.project(spec.Nu, spec.Nv, spec.Du, spec.Dv, spec.D, spec.d, spec.theta, ell, 0, spec.Np)
    Q = oracle.filter_fft(g, E)
    c = np.array([[i, j, k] for i in (30, 31, 32, 33) for j in (30, 31, 32, 33) for k in (30, 31, 32, 33)])
    V = oracle.backproject(g, Q, c)
    assert abs(V.mean() - 1.0) < 0.01
