"""Shared helpers for the GPU-vs-oracle parity tests (tolerances from north_star)."""
import numpy as np

# BASELINE.json north_star: "max |d| <= 1e-4 . max|V| and relative RMSE <= 1e-5".
VOL_MAX_REL = 1e-4
VOL_RMSE = 1e-5
# Filter: the same bounds on Q; an fp32 radix-4 FFT of length L has
# a relative RMS error of ~ eps sqrt(log2 L) ~ 2e-7, far inside both.
Q_MAX_REL = 1e-4
Q_RMSE = 1e-5


def metrics(got, ref):
    got = np.asarray(got, np.float64)
    ref = np.asarray(ref, np.float64)
    d = got - ref
    den = float(np.sqrt(np.sum(ref * ref)))
    rel_rmse = float(np.sqrt(np.sum(d * d)) / den) if den > 0 else float(np.sqrt(np.sum(d * d)))
    mx = float(np.abs(ref).max()) if ref.size else 0.0
    max_rel = float(np.abs(d).max() / mx) if mx > 0 else float(np.abs(d).max() if d.size else 0)
    return rel_rmse, max_rel


def assert_parity(got, ref, rmse_tol, max_tol, what=""):
    r, m = metrics(got, ref)
    print(f"PARITY {what}: relRMSE {r:.3e}  max|d|/max|ref| {m:.3e}  (n={np.size(ref)})")
    assert r <= rmse_tol and m <= max_tol, f"{what}: relRMSE {r:.3e} (tol {rmse_tol}), max|d|/max|ref| {m:.3e} (tol {max_tol})"
    return r, m


_POOL = None


def filter_fft_threads(og, E, v0=0):
    """oracle.filter_fft over row ranges on host threads (rows are independent in Alg.
    alg:filter, so the values are bitwise those of one call)."""
    import concurrent.futures as cf
    import os

    import oracle

    global _POOL
    nt = os.cpu_count() or 1
    if _POOL is None:
        _POOL = cf.ThreadPoolExecutor(nt)
    n_rows = E.shape[1]
    parts = min(n_rows, 2 * nt)
    cuts = [n_rows * i // parts for i in range(parts + 1)]
    Q = np.empty(E.shape, np.float64)

    def job(a, b):
        Q[:, a:b] = oracle.filter_fft(og, E[:, a:b], v0=v0 + a, workers=1)

    for f in [_POOL.submit(job, a, b) for a, b in zip(cuts[:-1], cuts[1:]) if b > a]:
        f.result()
    return Q
