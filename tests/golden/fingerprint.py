"""Size-independent fingerprints of full-size reference outputs.

Shared by make_golden.py (which runs the reference here) and the GPU tests
(which run on a box without the reference).  A full 256^3 render or a
2.1M-Gaussian gradient is too large to commit, so the goldens keep:
  * values at seeded sample indices (regenerated from the seed);
  * sha256 of arrays that must match exactly (coverage masks);
  * sign-hash sketches <r_k, x>, k < SKETCH_K, with r_k[i] = +-1 from an
    integer hash of (i, k).  For e = x_gpu - x_ref, E[<r_k, e>^2] = |e|^2,
    so the RMS of the sketch differences estimates |e|_2 without storing x.
The hash uses only int64 multiplies whose low 32 bits are kept, so numpy
(here) and torch (on the GPU) produce the same signs bit for bit.
"""

from __future__ import annotations

import numpy as np

SKETCH_K = 32
HR_SAMPLES = 65536
GRAD_SAMPLES = 16384
_M32 = 0xFFFFFFFF


def _hash_bits(i, k: int):
    """Low bit of a 32-bit mix of (i, k); i is an int64 numpy or torch array."""
    h = (i * 2654435761 + (k + 1) * 97531) & _M32
    h = ((h ^ (h >> 15)) * 2246822519) & _M32
    h = ((h ^ (h >> 13)) * 3266489917) & _M32
    h = h ^ (h >> 16)
    return h & 1


def sketch_signs(n: int, k: int) -> np.ndarray:
    return (1 - 2 * _hash_bits(np.arange(n, dtype=np.int64), k)).astype(np.int8)


def sketch(x) -> list:
    """numpy: [<r_k, x> for k < SKETCH_K] in float64 (x flattened C-order)."""
    x = np.asarray(x, dtype=np.float64).reshape(-1)
    return [float(np.dot(sketch_signs(x.shape[0], k).astype(np.float64), x))
            for k in range(SKETCH_K)]


def sketch_torch(x) -> list:
    """The same sketch of a torch tensor, computed on its device."""
    import torch
    x = x.reshape(-1).to(torch.float64)
    i = torch.arange(x.shape[0], dtype=torch.int64, device=x.device)
    out = []
    for k in range(SKETCH_K):
        r = (1 - 2 * _hash_bits(i, k)).to(torch.float64)
        out.append(float(torch.dot(r, x)))
    return out


def sketch_rms_error(got: list, ref: list) -> float:
    """Estimate of |x_gpu - x_ref|_2 from the two sketches."""
    d = np.asarray(got) - np.asarray(ref)
    return float(np.sqrt(np.mean(d * d)))


def hr_sample_idx(nvox: int, cid: int) -> np.ndarray:
    return np.random.default_rng(1000 + cid).choice(nvox, size=min(HR_SAMPLES, nvox),
                                                    replace=False)


def grad_sample_idx(n: int, cid: int) -> np.ndarray:
    return np.random.default_rng(2000 + cid).choice(n, size=min(GRAD_SAMPLES, n),
                                                    replace=False)
