"""GPU-vs-oracle tolerances (north_star).

* predicted errors: 1e-3 relative on the error norm sqrt(err^2), i.e.
  |e2_gpu - e2_ora| <= 2e-3 * e2_ora, plus an fp32-resolution floor of
  1e-7 * total in the squared domain (the inputs and the projection GEMMs are
  fp32: an exact-zero error comes back as O(u_fp32 * ||M||_F^2));
* singular values: 1e-4 relative plus 1e-6 * sigma_1 of the same spectrum
  (reading A13);
* energies: 1e-12 relative (fp64 accumulation of exact fp32 products).
"""
import numpy as np


def err2_ok(e2_gpu, e2_ora, total):
    e2_gpu = np.asarray(e2_gpu); e2_ora = np.asarray(e2_ora); total = np.asarray(total)
    return np.abs(e2_gpu - e2_ora) <= 2e-3 * e2_ora + 1e-7 * total


def sigma_ok(s_gpu, s_ora, s1):
    s_gpu = np.asarray(s_gpu, np.float64); s_ora = np.asarray(s_ora, np.float64)
    return np.abs(s_gpu - s_ora) <= 1e-4 * s_ora + 1e-6 * np.asarray(s1)[..., None]


def assert_err2(e2_gpu, e2_ora, total, what=""):
    ok = err2_ok(e2_gpu, e2_ora, total)
    if not ok.all():
        idx = np.argwhere(~ok)[:5]
        rows = [(tuple(i), float(np.asarray(e2_gpu)[tuple(i)]), float(np.asarray(e2_ora)[tuple(i)])) for i in idx]
        raise AssertionError(f"{what}: {int((~ok).sum())} err2 outside tolerance, e.g. {rows}")


def assert_sigma(s_gpu, s_ora, s1, what=""):
    ok = sigma_ok(s_gpu, s_ora, s1)
    if not ok.all():
        idx = np.argwhere(~ok)[:5]
        rows = [(tuple(i), float(np.asarray(s_gpu)[tuple(i)]), float(np.asarray(s_ora)[tuple(i)])) for i in idx]
        raise AssertionError(f"{what}: {int((~ok).sum())} singular values outside tolerance, e.g. {rows}")
