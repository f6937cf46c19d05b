"""Seeded synthetic inputs standing in for the five BASELINE.json configs.

BASELINE.json names no public dataset; these generators follow SURVEY.md
Appendix A (builder conventions where BASELINE.json is silent):

* ``rng = np.random.default_rng(SEED[cfg])`` (PCG64, as simulate.py:178);
* draw order: perturbation axis (cfg4 only), then band parameters in the
  listed order, then noise ``rng.normal(0, sigma, (m, n))`` row-major
  (cfg2: all set-1 parameters, all set-2 parameters, set-1 noise, set-2 noise);
* Lorentzian ``w^2/((nu-c)^2+w^2)`` (w = HWHM) and Gaussian
  ``exp(-(nu-c)^2/(2 s^2))`` as simulate.py:84-88;
* intensities = amplitudes (m x B) @ profiles (B x n) in float64 with BLAS
  pinned to one thread, so the bits do not depend on the host.

Each generator returns a :class:`ConfigCase` with the raw spectral datasets
(float64 arrays; cfg5 additionally rounds to float32 as the fp32 config
prescribes), the preprocessing recipe and the compute dtype.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

SEED = {1: 101, 2: 202, 3: 303, 4: 404, 5: 505}


@dataclass
class RawSet:
    spectral_axis: np.ndarray
    perturbation_axis: np.ndarray
    intensities: np.ndarray


@dataclass
class ConfigCase:
    cfg: int
    name: str
    set1: RawSet
    set2: RawSet | None
    resample: int | None = None
    interpolant: str = "linear"
    alpha: float = 0.0
    dtype: str = "float64"
    notes: dict = field(default_factory=dict)

    @property
    def m(self) -> int:
        return self.resample or self.set1.perturbation_axis.size

    @property
    def n1(self) -> int:
        return self.set1.spectral_axis.size

    @property
    def n2(self) -> int:
        return (self.set2 or self.set1).spectral_axis.size

    @property
    def homo(self) -> bool:
        return self.set2 is None


def _lorentz(nu, c, w):
    w2 = (w * w)[:, None]
    return w2 / ((nu[None, :] - c[:, None]) ** 2 + w2)


def _gauss(nu, c, s):
    return np.exp(-((nu[None, :] - c[:, None]) ** 2) / (2.0 * (s * s)[:, None]))


def _matmul1(a, b):
    try:
        from threadpoolctl import threadpool_limits
        with threadpool_limits(limits=1):
            return a @ b
    except ImportError:  # pragma: no cover
        return a @ b


def cfg1() -> ConfigCase:
    """11 spectra (t = 20..70 step 5) x 1000 points over 800-1800, 3 Lorentzians."""
    rng = np.random.default_rng(SEED[1])
    t = 20.0 + 5.0 * np.arange(11)
    nu = np.linspace(800.0, 1800.0, 1000)
    s = (t - 20.0) / 50.0
    w = np.array([15.0])
    base = _lorentz(nu, np.array([1000.0, 1300.0]), np.array([15.0, 15.0]))  # 2 x n
    amp = np.stack([1.0 + s, 1.0 - 0.7 * s], axis=1)  # m x 2
    inten = _matmul1(amp, base)
    c3 = 1600.0 - 0.2 * (t - 20.0)
    for j in range(t.size):
        inten[j] += 0.5 * _lorentz(nu, c3[j:j + 1], w)[0]
    inten += rng.normal(0.0, 0.01, (t.size, nu.size))
    return ConfigCase(1, "cfg1_homo_11x1000_f64", RawSet(nu, t, inten), None,
                      notes={"bands": "L 1000,1300,1600(t) HWHM 15", "noise": 0.01})


def cfg2() -> ConfigCase:
    """Hetero: 21x2000 Gaussians (sigmoid amps) vs 21x1500 Lorentzians (exp decay)."""
    rng = np.random.default_rng(SEED[2])
    t = np.linspace(0.0, 100.0, 21)
    nu1 = np.linspace(400.0, 2400.0, 2000)
    nu2 = np.linspace(0.0, 1500.0, 1500)
    c1 = rng.uniform(400.0, 2400.0, 5)
    s1 = rng.uniform(8.0, 25.0, 5)
    t0 = rng.uniform(0.0, 100.0, 5)
    c2 = rng.uniform(0.0, 1500.0, 4)
    w2 = rng.uniform(2.0, 20.0, 4)
    tau = rng.uniform(10.0, 100.0, 4)
    amp1 = 1.0 / (1.0 + np.exp(-(t[:, None] - t0[None, :]) / 10.0))
    amp2 = np.exp(-t[:, None] / tau[None, :])
    i1 = _matmul1(amp1, _gauss(nu1, c1, s1))
    i2 = _matmul1(amp2, _lorentz(nu2, c2, w2))
    i1 += rng.normal(0.0, 0.005, i1.shape)
    i2 += rng.normal(0.0, 0.005, i2.shape)
    return ConfigCase(2, "cfg2_hetero_21x2000_21x1500_f64", RawSet(nu1, t, i1),
                      RawSet(nu2, t.copy(), i2), notes={"noise": 0.005})


def cfg3() -> ConfigCase:
    """64 x 16384, 200 Lorentzians with amplitude g t / 63."""
    rng = np.random.default_rng(SEED[3])
    t = np.arange(64, dtype=float)
    nu = np.arange(16384, dtype=float)
    c = rng.uniform(0.0, 16383.0, 200)
    w = rng.uniform(2.0, 20.0, 200)
    g = rng.normal(0.0, 1.0, 200)
    amp = (t[:, None] / 63.0) * g[None, :]
    inten = _matmul1(amp, _lorentz(nu, c, w))
    inten += rng.normal(0.0, 0.01, inten.shape)
    return ConfigCase(3, "cfg3_homo_64x16384_f64", RawSet(nu, t, inten), None,
                      notes={"noise": 0.01})


def cfg4() -> ConfigCase:
    """37 sorted U[0,100] perturbations -> linear 64, 8192 points, alpha 0.5."""
    rng = np.random.default_rng(SEED[4])
    t = np.sort(rng.uniform(0.0, 100.0, 37))
    nu = np.arange(8192, dtype=float)
    c = rng.uniform(0.0, 8191.0, 50)
    s = rng.uniform(5.0, 50.0, 50)
    a = rng.normal(0.0, 1.0, 50)
    b = rng.normal(0.0, 1.0, 50)
    amp = t[:, None] * a[None, :] + (t * t)[:, None] * b[None, :]
    inten = _matmul1(amp, _gauss(nu, c, s))
    inten += rng.normal(0.0, 0.02, inten.shape)
    return ConfigCase(4, "cfg4_homo_37to64x8192_linear_alpha0.5_f64", RawSet(nu, t, inten), None,
                      resample=64, interpolant="linear", alpha=0.5,
                      notes={"noise": 0.02, "beta": 0.0})


def cfg5() -> ConfigCase:
    """512 x 32768, 1000 Lorentzians with 3-sinusoid amplitudes; fp32."""
    rng = np.random.default_rng(SEED[5])
    t = np.arange(512, dtype=float)
    nu = np.arange(32768, dtype=float)
    c = rng.uniform(0.0, 32767.0, 1000)
    w = rng.uniform(2.0, 20.0, 1000)
    a = rng.normal(0.0, 1.0, (1000, 3))
    f = rng.uniform(1.0, 32.0, (1000, 3))
    ph = rng.uniform(0.0, 2.0 * np.pi, (1000, 3))
    amp = np.zeros((t.size, 1000))
    for k in range(3):
        amp += a[None, :, k] * np.sin(2.0 * np.pi * f[None, :, k] * t[:, None] / 512.0 + ph[None, :, k])
    inten = _matmul1(amp, _lorentz(nu, c, w))
    inten += rng.normal(0.0, 0.01, inten.shape)
    inten = inten.astype(np.float32)  # both GPU and oracle see the fp32-rounded data
    return ConfigCase(5, "cfg5_homo_512x32768_f32", RawSet(nu, t, inten), None,
                      dtype="float32", notes={"noise": 0.01, "rounded": "float32"})


GENERATORS = {1: cfg1, 2: cfg2, 3: cfg3, 4: cfg4, 5: cfg5}


def make(cfg: int) -> ConfigCase:
    return GENERATORS[int(cfg)]()
