"""Shared test helpers: small seeded scenes and parity metrics."""
import numpy as np


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def cosine(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(a @ b / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-300))


def field_rel(a, b, n):
    """|f_gpu - f_ref| / max(|f_ref|, 1e-6 sqrt(N))."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-6 * np.sqrt(n))


def random_block(rng, n, lo, hi, vs=0.3, fs=0.02, cs=0.5, groups=1):
    x = lo + (hi - lo) * rng.random((n, 3))
    v = vs * rng.standard_normal((n, 3))
    F = np.tile(np.eye(3).ravel(), (n, 1)) + fs * rng.standard_normal((n, 9))
    C = cs * rng.standard_normal((n, 9))
    return {"x": x, "v": v, "F": F, "C": C, "material": np.zeros(n, np.int32),
            "group": rng.integers(0, groups, n).astype(np.int32)}


def to_f32_state(st):
    return {k: (np.asarray(v, np.float32).astype(np.float64) if k in "xvFC" else v) for k, v in st.items()}
