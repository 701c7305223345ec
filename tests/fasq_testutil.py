"""Shared test helpers (tolerances from BASELINE.json north_star)."""
import numpy as np


def parity_ok(y, y_ref, x, F_in, rel_l2=1e-3, abs_coef=5e-3):
    """north_star: ||y - y_ref||_2 / ||y_ref||_2 <= 1e-3 and
    max|y - y_ref| <= 5e-3 * ||x||_inf * sqrt(K), K = F_in, against fp64."""
    y = np.asarray(y, np.float64)
    y_ref = np.asarray(y_ref, np.float64)
    err = y - y_ref
    nref = np.linalg.norm(y_ref)
    rel = np.linalg.norm(err) / nref if nref > 0 else np.linalg.norm(err)
    xinf = float(np.max(np.abs(np.asarray(x, np.float64)))) if np.size(x) else 0.0
    amax = float(np.max(np.abs(err))) if err.size else 0.0
    bound = abs_coef * xinf * np.sqrt(F_in)
    return (rel <= rel_l2 and amax <= bound + 1e-30), {"rel_l2": rel, "max_abs": amax, "abs_bound": bound}
