"""Seeded synthetic input generators shared by the oracle tests and the GPU
parity tests.  Holds none of the method's arithmetic: only random numbers of a
given shape / dtype / distribution (SURVEY 8d input recipe)."""
import numpy as np


def rng(seed: int) -> np.random.Generator:
    return np.random.default_rng(seed)


def uniform_field(shape, seed: int, dtype=np.float64, lo=-1.0, hi=1.0) -> np.ndarray:
    """Uniform[lo, hi) values, generated in binary64 and then cast (RN) to dtype."""
    return rng(seed).uniform(lo, hi, size=shape).astype(dtype)


def uniform_global(n: int, seed: int) -> np.ndarray:
    return rng(seed).uniform(-1.0, 1.0, size=n)


def lognormal_terms(n: int, seed: int, sigma: float = 8.0, cancel: bool = False) -> np.ndarray:
    """Terms spanning many binades; with cancel=True, signs are mixed and a
    large cancelling pair is planted (heavy cancellation)."""
    g = rng(seed)
    t = np.exp(g.normal(0.0, sigma, size=n))
    if cancel:
        t *= g.choice([-1.0, 1.0], size=n)
        if n >= 2:
            big = 2.0 ** 60
            t[0] += big
            t[n // 2] -= big
    return t
