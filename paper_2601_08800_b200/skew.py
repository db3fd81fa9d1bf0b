"""Skewed routers (BASELINE config E) and the host-load skew term.

The reference cost model prices the MoE all-to-all on the MEAN per-rank
volume ``(b/t) * s * h * k * bytes`` (costmodel.py:129-133): it assumes every
expert host receives the same share of slots.  Under a skewed router (Zipf
expert popularity) the hottest host receives more, and the layer waits for
it.  This module adds that term without touching the reference's arithmetic:

* :func:`zipf_popularity` -- expert popularity ``p_e ∝ rank^-s`` with the
  rank order permuted by a seed;
* :func:`zipf_logits` -- gate logits ``N(0,1) + log p_e`` fed to the router;
* :func:`host_loads` / :func:`host_skew` -- slots per expert-parallel host
  under the reference's contiguous placement ``e * d // E``
  (simcluster.py:210-212) and ``kappa = max / mean``;
* ``costmodel.comm_terms(..., expert_load=...)`` scales the A2A volume by
  ``kappa(moe_ep)``.  ``expert_load=None`` or a balanced load gives
  ``kappa == 1.0`` exactly, so the ranking degenerates to the reference's.
"""
from __future__ import annotations

import numpy as np

__all__ = ["zipf_popularity", "zipf_logits", "host_loads", "host_skew", "expert_counts"]


def zipf_popularity(num_experts: int, s: float, seed: int = 0) -> np.ndarray:
    """``p_e ∝ rank(e)^-s`` normalised, popularity order permuted by ``seed``."""
    if num_experts < 1:
        raise ValueError("num_experts must be positive")
    if s < 0:
        raise ValueError("Zipf exponent must be nonnegative")
    ranks = np.arange(1, num_experts + 1, dtype=np.float64)
    p = ranks ** (-float(s))
    p /= p.sum()
    perm = np.random.default_rng(seed).permutation(num_experts)
    out = np.empty_like(p)
    out[perm] = p
    return out


def zipf_logits(tokens: int, num_experts: int, s: float, seed: int = 0, *, device=None,
                generator=None):
    """fp32 gate logits ``N(0,1) + log p_e`` (torch tensor ``[tokens, E]``).

    ``generator`` drives the N(0,1) draw (torch); the popularity order comes
    from ``seed`` so every group of a run shares it."""
    import torch

    logp = torch.from_numpy(np.log(zipf_popularity(num_experts, s, seed))).float()
    base = torch.randn(tokens, num_experts, generator=generator, device=device or "cpu")
    return base + logp.to(base.device)


def expert_counts(ids, num_experts: int) -> np.ndarray:
    """Slots per expert of a routed batch (``bincount`` of the top-k ids)."""
    a = np.asarray(ids).reshape(-1)
    return np.bincount(a, minlength=num_experts).astype(np.float64)


def host_loads(expert_load, ep: int) -> np.ndarray:
    """Sum of ``expert_load`` per host, experts placed contiguously
    (``home = e * ep // E``, simcluster.py:210-212)."""
    load = np.asarray(expert_load, dtype=np.float64).reshape(-1)
    E = load.size
    if ep < 1:
        raise ValueError(f"ep={ep} must be positive")
    home = (np.arange(E) * ep) // E
    return np.bincount(home, weights=load, minlength=ep)


def host_skew(expert_load, ep: int) -> float:
    """``max / mean`` host load at expert-parallel degree ``ep`` (>= 1),
    over the hosts that own at least one expert.

    Returns exactly 1.0 for ``ep == 1``, for ``expert_load is None`` and
    whenever every host carries the same load, so the skew-aware ranking
    reduces to the reference's on balanced routers."""
    if expert_load is None or ep == 1:
        return 1.0
    loads = host_loads(expert_load, ep)
    # ep > E leaves hosts without experts; the mean runs over hosts that own one
    owns = np.bincount((np.arange(np.size(expert_load)) * ep) // np.size(expert_load),
                       minlength=ep) > 0
    loads = loads[owns]
    ep = loads.size
    if loads.max() == loads.min():
        return 1.0
    total = loads.sum()
    if total <= 0:
        return 1.0
    return float(loads.max() / (total / ep))
