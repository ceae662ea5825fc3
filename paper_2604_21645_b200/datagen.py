"""Seeded synthetic inputs standing in for BASELINE.json's datasets.

BASELINE.json specifies Gaussian-mixture data and no public dataset: means
mu_k ~ N(0, 4 I) (sigma 2 per coordinate), per-component isotropic sigma_k ~
U(0.5, 1.5), equal component weights; rows x = mu_c +
sigma_c * z, z ~ N(0, I), computed in fp64 and stored as fp32.  Queries reuse
the same mixture with an independent stream.  numpy's PCG64 makes the bytes
identical on every host, so the oracle and the GPU always see the same input.
"""
from __future__ import annotations

import numpy as np


def mixture_params(dims: int, components: int, seed: int):
    rng = np.random.Generator(np.random.PCG64(seed))
    means = rng.normal(0.0, 2.0, size=(components, dims))
    sigmas = rng.uniform(0.5, 1.5, size=components)
    return means, sigmas


def gaussian_mixture(rows: int, dims: int, components: int, seed: int, stream: int = 0,
                     chunk: int = 1 << 20) -> np.ndarray:
    """rows x dims float32 drawn from the seeded mixture.  ``stream`` selects an
    independent row stream over the same mixture (0 = base rows, 1 = queries,
    2+r = shard r when rows are generated per shard)."""
    means, sigmas = mixture_params(dims, components, seed)
    rng = np.random.Generator(np.random.PCG64([seed, stream + 1]))
    out = np.empty((rows, dims), np.float32)
    for b in range(0, rows, chunk):
        e = min(rows, b + chunk)
        comp = rng.integers(0, components, size=e - b)
        z = rng.standard_normal(size=(e - b, dims))
        out[b:e] = means[comp] + sigmas[comp, None] * z
    return out


def strided_sample(n_rows: int, n_sample: int, seed: int) -> np.ndarray:
    """The seeded S-row training sample of SURVEY.md 8(d): rows
    {i : (i + off) mod (N/S) == 0}, off = seed mod (N/S), ascending; the first
    n_sample of them.  Deterministic and independent of the GPU count."""
    if n_sample >= n_rows:
        return np.arange(n_rows, dtype=np.int64)
    stride = n_rows // n_sample
    off = seed % stride
    first = (stride - off) % stride
    return (first + stride * np.arange(n_sample, dtype=np.int64))


def device_mixture(rows: int, dims: int, components: int, seed: int, gen_seed: int, out=None,
                   chunk: int = 1 << 20):
    """rows x dims float32 drawn on the GPU from the same seeded mixture
    (mixture_params(dims, components, seed)), rows from a torch CUDA (Philox)
    generator seeded with gen_seed -- BASELINE configs[4]'s "generated per
    shard from seed + rank"; also used for configs[3]'s 10M
    rows.  x = mu_c + sigma_c * z in fp64, stored fp32.  ``out`` (optional) is
    a preallocated rows x dims CUDA tensor to fill."""
    import torch
    means, sigmas = mixture_params(dims, components, seed)
    mu = torch.from_numpy(means.astype(np.float64)).cuda()
    sg = torch.from_numpy(sigmas.astype(np.float64)).cuda()
    g = torch.Generator(device="cuda")
    g.manual_seed(gen_seed)
    x = out if out is not None else torch.empty((rows, dims), dtype=torch.float32, device="cuda")
    for r0 in range(0, rows, chunk):
        r1 = min(rows, r0 + chunk)
        comp = torch.randint(0, components, (r1 - r0,), generator=g, device="cuda")
        z = torch.randn((r1 - r0, dims), generator=g, device="cuda", dtype=torch.float64)
        x[r0:r1] = (mu[comp] + sg[comp, None] * z).float()
    return x
