"""Seeded synthetic fields for the five BASELINE.json configs.

The paper's SDRBench datasets (Hurricane, CESM-ATM, ...) are not available
offline; these generators stand in for them with the shapes, spectra and value
distributions BASELINE.json names.  Parity never depends on
the generator: the same array feeds the GPU path and the oracle.

* config 1 -- 1-D sinusoid mix, 2^20 values, seed 0, rel eps 1e-3
* config 2 -- 100x500x500 GRF, P(k) ~ k^-11/3, mean 280 std 15, seed 1, rel 1e-4
* config 3 -- 1800x3600 sum of 64 Fourier modes x a 40% rectangular mask, seed 2
* config 4 -- 512^3 lognormal exp(1.5 G), G a GRF with P(k) ~ k^-2, seed 3, rel 1e-3
* config 5 -- 2048^3 as config 2, generated as 8 slabs of 256x2048x2048, slab s
  from seed (4, s), so the field is identical for any GPU count

GRFs: white Gaussian noise -> rFFT -> amplitude k^(-alpha/2) (DC zeroed) ->
inverse rFFT -> standardise.  Small fields use scipy on the host; large ones
use torch.fft on the GPU when ``device`` is given.
"""

from __future__ import annotations

import os

import numpy as np

CONFIGS = {
    1: dict(dims=(1 << 20,), rel_eps=1e-3, sadd=3.5, smul=-1.25),
    2: dict(dims=(100, 500, 500), rel_eps=1e-4, sadd=3.5, smul=-1.25),
    3: dict(dims=(1800, 3600), rel_eps=1e-4, rel_sweep=(1e-3, 1e-4, 1e-5), sadd=3.5, smul=-1.25),
    # config 4: eps ~ 4.16, so scalars must exceed 2 eps
    4: dict(dims=(512, 512, 512), rel_eps=1e-3, sadd=100.0, smul=-12.5),
    5: dict(dims=(2048, 2048, 2048), rel_eps=1e-4, sadd=3.5, smul=-1.25, slabs=8),
}


def config1(seed: int = 0) -> np.ndarray:
    rng = np.random.default_rng(seed)
    n = 1 << 20
    a = rng.uniform(0.5, 2.0, 8)
    f = rng.uniform(1.0, 200.0, 8)
    ph = rng.uniform(0.0, 2 * np.pi, 8)
    i = np.arange(n, dtype=np.float64)
    x = np.zeros(n)
    for j in range(8):
        x += a[j] * np.sin(2 * np.pi * f[j] * i / n + ph[j])
    x += rng.normal(0.0, 0.01, n)
    return x.astype(np.float32)


def _kgrid_np(shape):
    axes = [np.fft.fftfreq(s) for s in shape[:-1]] + [np.fft.rfftfreq(shape[-1])]
    k2 = np.zeros([len(a) for a in axes], dtype=np.float64)
    for d, a in enumerate(axes):
        sh = [1] * len(axes)
        sh[d] = len(a)
        k2 = k2 + (a.reshape(sh) ** 2)
    return np.sqrt(k2)


def grf_host(shape, alpha: float, seed) -> np.ndarray:
    """Standardised Gaussian random field, P(k) ~ k^-alpha (float64 host)."""
    import scipy.fft as sfft

    rng = np.random.default_rng(seed)
    white = rng.standard_normal(shape, dtype=np.float32)
    spec = sfft.rfftn(white, workers=os.cpu_count())
    k = _kgrid_np(shape).astype(np.float32)
    with np.errstate(divide="ignore"):
        amp = np.where(k > 0, k ** (-alpha / 2.0), 0.0).astype(np.float32)
    spec *= amp
    field = sfft.irfftn(spec, s=shape, workers=os.cpu_count()).astype(np.float64)
    field -= field.mean()
    field /= field.std()
    return field


def grf_device(shape, alpha: float, seed, device="cuda"):
    """Same construction on the GPU with torch (for the 512^3 / 2048^3 fields)."""
    import torch

    gen = torch.Generator(device=device)
    s = seed if isinstance(seed, int) else int(np.random.SeedSequence(seed).generate_state(1)[0])
    gen.manual_seed(s)
    white = torch.randn(shape, generator=gen, device=device, dtype=torch.float32)
    spec = torch.fft.rfftn(white)
    del white
    axes = [torch.fft.fftfreq(n, device=device) for n in shape[:-1]]
    axes.append(torch.fft.rfftfreq(shape[-1], device=device))
    k2 = None
    for d, a in enumerate(axes):
        sh = [1] * len(axes)
        sh[d] = a.numel()
        term = (a.reshape(sh) ** 2)
        k2 = term if k2 is None else k2 + term
    amp = torch.where(k2 > 0, k2.clamp_min(1e-30) ** (-alpha / 4.0), torch.zeros((), device=device))
    spec *= amp
    del amp, k2
    field = torch.fft.irfftn(spec, s=shape)
    del spec
    field = field - field.mean()
    field = field / field.std()
    return field


def config2(seed: int = 1, device=None):
    shape = CONFIGS[2]["dims"]
    if device is not None:
        return (grf_device(shape, 11.0 / 3.0, seed, device) * 15.0 + 280.0).reshape(-1).float()
    return (grf_host(shape, 11.0 / 3.0, seed) * 15.0 + 280.0).astype(np.float32).ravel()


def config3(seed: int = 2) -> np.ndarray:
    ny, nx = CONFIGS[3]["dims"]
    rng = np.random.default_rng(seed)
    y = np.linspace(0.0, 1.0, ny, endpoint=False)[:, None]
    x = np.linspace(0.0, 1.0, nx, endpoint=False)[None, :]
    field = np.zeros((ny, nx))
    for _ in range(64):
        kx, ky = rng.integers(1, 12, 2)
        amp = rng.uniform(0.2, 1.0)
        ph = rng.uniform(0, 2 * np.pi)
        # cos(a + b) = cos a cos b - sin a sin b, with a over x and b over y
        ax = 2 * np.pi * kx * x + ph
        by = 2 * np.pi * ky * y
        field += amp * (np.cos(by) * np.cos(ax) - np.sin(by) * np.sin(ax))
    mask = np.ones((ny, nx), dtype=bool)
    target = 0.40 * ny * nx
    while (~mask).sum() < target:
        h, w = rng.integers(ny // 20, ny // 4), rng.integers(nx // 20, nx // 4)
        y0, x0 = rng.integers(0, ny - h), rng.integers(0, nx - w)
        mask[y0:y0 + h, x0:x0 + w] = False
    field[~mask] = 0.0
    return field.astype(np.float32).ravel()


def config4(seed: int = 3, device=None):
    shape = CONFIGS[4]["dims"]
    if device is not None:
        import torch

        return torch.exp(1.5 * grf_device(shape, 2.0, seed, device)).reshape(-1).float()
    return np.exp(1.5 * grf_host(shape, 2.0, seed)).astype(np.float32).ravel()


def config5_slab(slab: int, seed: int = 4, device="cuda"):
    """Slab `slab` (0..7) of config 5: 256 x 2048 x 2048 values (2^30)."""
    shape = (256, 2048, 2048)
    return (grf_device(shape, 11.0 / 3.0, (seed, slab), device) * 15.0 + 280.0).reshape(-1).float()


CONFIG5_SLAB = 1 << 30          # values per slab (256 x 2048 x 2048)
CONFIG5_N = 8 * CONFIG5_SLAB    # the whole 2048^3 field


def config5_range(e0: int, e1: int, seed: int = 4, device="cuda", out=None):
    """Elements [e0, e1) of the ONE 2048^3 config-5 field (flat row-major),
    assembled from the slabs they overlap -- identical for any partition, so
    a rank owning a contiguous block range generates exactly its share of
    the same field.  `out` (optional) receives the values in place."""
    import torch

    if not (0 <= e0 <= e1 <= CONFIG5_N):
        raise ValueError(f"config 5 range [{e0}, {e1}) outside [0, 2^33)")
    if out is None:
        out = torch.empty(e1 - e0, dtype=torch.float32, device=device)
    s0, s1 = e0 // CONFIG5_SLAB, -(-e1 // CONFIG5_SLAB)
    for s in range(s0, s1):
        a = max(e0, s * CONFIG5_SLAB)
        b = min(e1, (s + 1) * CONFIG5_SLAB)
        if a >= b:
            continue
        slab = config5_slab(s, seed=seed, device=device)
        out[a - e0:b - e0].copy_(slab[a - s * CONFIG5_SLAB:b - s * CONFIG5_SLAB])
        del slab
        torch.cuda.empty_cache()
    return out


def field(config: int, device=None):
    if config == 1:
        return config1()
    if config == 2:
        return config2(device=device)
    if config == 3:
        return config3()
    if config == 4:
        return config4(device=device)
    raise ValueError(f"config {config}: use config5_slab for the sharded config")
