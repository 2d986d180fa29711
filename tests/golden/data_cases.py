"""Seeded inputs for the data-path golden cases (cut / stitch / codec / confusion / report)."""
import numpy as np

SIZES = [(300, 517), (256, 256), (17, 40), (513, 255)]
TILE = 256
# train_val_split cases (n, val_fraction, seed): BASELINE corpus, tiny corpora, zero fraction
SPLITS = [(4224, 0.2, 0), (64, 0.2, 0), (10, 0.2, 9), (3, 0.5, 1), (1, 0.2, 0), (50, 0.0, 3), (97, 0.35, 7)]


def scene(h, w, seed=5):
    return np.random.default_rng([seed, h, w]).integers(0, 256, (h, w, 3), dtype=np.uint8)


def mask(h, w, seed=6):
    return np.random.default_rng([seed, h, w]).integers(0, 3, (h, w)).astype(np.uint8)


def pred_ref(seed=7, n=4096):
    rng = np.random.default_rng(seed)
    ref = rng.integers(0, 3, (64, n // 64)).astype(np.uint8)
    pred = ref.copy()
    flip = rng.random(ref.shape) < 0.3
    pred[flip] = rng.integers(0, 3, int(flip.sum())).astype(np.uint8)
    return pred, ref
