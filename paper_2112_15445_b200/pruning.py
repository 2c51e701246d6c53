"""Pruned-weight generation: the mask arithmetic of the reference's pruning module
(/root/reference/pkg/src/unsparse/pruning.py:131-209) and the bench's synthetic
masked weights (bench.py:84-95), plus the paper's *unified* per-output-channel
sparsity (every output channel keeps the same number of nonzeros, so the
encoder adds no padding entries -- PAPER.md:314).

The evolutionary search itself (prune_loop and its retraining) is training
machinery outside the inference hot path and is not rebuilt here.
"""

from __future__ import annotations

import numpy as np

from .tensor import ConvGeometry, DenseTensor4, PrecisionMode


def apply_mask(weights: np.ndarray, mask: np.ndarray) -> np.ndarray:
    """theta <- theta * M (pruning.py:131-141), on arrays."""
    if mask.shape != weights.shape:
        raise ValueError(f"mask shape {mask.shape} != weight shape {weights.shape}")
    return weights * mask.astype(weights.dtype)


def layer_sparsity(mask) -> float:
    """pruning.py:150-153."""
    if mask.size == 0:
        raise ValueError("empty mask")
    return float((mask.size - int(mask.sum())) / mask.size)


def weighted_sparsity(masks) -> float:
    """pruning.py:156-163: size-weighted mean over layers (iterable of masks)."""
    total, zeros = 0, 0.0
    for mask in masks:
        total += mask.size
        zeros += mask.size * layer_sparsity(mask)
    return zeros / total


def importance(theta, grad_stat, alpha: float):
    """pruning.py:185-189: g = alpha*|G| + (1-alpha)*|theta|."""
    if theta.shape != grad_stat.shape:
        raise ValueError(f"shape mismatch {theta.shape} vs {grad_stat.shape}")
    return alpha * np.abs(grad_stat) + (1.0 - alpha) * np.abs(theta)


def mask_for_target(g, target: float):
    """pruning.py:192-200: exactly floor(target*size) zeros at the smallest
    importance values, ties toward the lower flat index."""
    k = int(np.floor(target * g.size))
    mask = np.ones(g.size, dtype=np.uint8)
    if k > 0:
        order = np.argsort(g.ravel(), kind="stable")
        mask[order[:k]] = 0
    return mask.reshape(g.shape)


def random_mask(shape, sparsity: float, rng):
    """pruning.py:203-209."""
    size = int(np.prod(shape))
    k = int(np.floor(sparsity * size))
    mask = np.ones(size, dtype=np.uint8)
    if k > 0:
        mask[rng.choice(size, size=k, replace=False)] = 0
    return mask.reshape(shape)


def unified_mask(shape, sparsity: float, rng):
    """Unified sparsity: each output channel (axis 0) keeps exactly
    round((1-s) * C*Kh*Kw) (at least 1) nonzeros."""
    d = shape[0]
    per = int(np.prod(shape[1:]))
    keep = max(1, int(round((1.0 - sparsity) * per)))
    mask = np.zeros((d, per), dtype=np.uint8)
    for i in range(d):
        mask[i, rng.choice(per, size=keep, replace=False)] = 1
    return mask.reshape(shape)


def synthesize_masked_weights(geometry: ConvGeometry, sparsity: float, rng,
                              precision=PrecisionMode.BINARY32, unified: bool = False) -> DenseTensor4:
    """bench.py:84-95: N(0,1) weights with exactly floor(s*size) zeros chosen
    uniformly over the layer (same RNG draws as the reference); `unified=True`
    prunes per output channel instead."""
    shape = (geometry.out_channels, geometry.in_channels, geometry.filter_h, geometry.filter_w)
    w = rng.standard_normal(shape).astype(np.float32)
    if unified:
        w *= unified_mask(shape, sparsity, rng).astype(np.float32)
        return DenseTensor4.from_array(w, precision)
    size = w.size
    k = int(np.floor(sparsity * size))
    if k:
        flat = w.reshape(-1)
        flat[rng.choice(size, size=k, replace=False)] = 0.0
    return DenseTensor4.from_array(w, precision)
