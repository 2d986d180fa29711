"""Corpus helpers the training path needs (reference icetrain/data.py)."""
from __future__ import annotations

import numpy as np


def train_val_split(pairs: list, val_fraction: float, seed: int) -> tuple:
    """data.py:125-136: seeded permutation; validation = the first round(n * f) indices
    (never the whole corpus), training keeps the original order."""
    if not 0.0 <= val_fraction < 1.0:
        raise ValueError(f"val_fraction out of range: {val_fraction}")
    order = np.random.default_rng(seed).permutation(len(pairs))
    n_val = min(int(round(len(pairs) * val_fraction)), len(pairs) - 1)
    val_idx = set(order[:n_val].tolist())
    train = [pairs[i] for i in range(len(pairs)) if i not in val_idx]
    val = [pairs[i] for i in sorted(val_idx)]
    return train, val
