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


def noisy_colors(h, w, seed=8):
    """Colormap colours with +-60 per-channel noise (parse_labels snap=True / error cases)."""
    rng = np.random.default_rng([seed, h, w])
    cols = np.array([(255, 0, 0), (0, 0, 255), (0, 255, 0)], np.int16)
    img = cols[rng.integers(0, 3, (h, w))] + rng.integers(-60, 61, (h, w, 3))
    img[0, :3] = [(128, 128, 0), (0, 128, 128), (128, 0, 128)]  # equidistant ties
    return np.clip(img, 0, 255).astype(np.uint8)


def ssim_pairs():
    """(name, a, b) u8 images for SSIM: identical, noisy copy, unrelated, minimum size."""
    a = scene(64, 80, seed=11)
    rng = np.random.default_rng(12)
    noisy = np.clip(a.astype(np.int16) + rng.integers(-20, 21, a.shape), 0, 255).astype(np.uint8)
    smooth = np.repeat(np.repeat(scene(8, 10, seed=13), 8, axis=0), 8, axis=1)
    return [("same", a, a.copy()), ("noisy", a, noisy), ("unrelated", a, scene(64, 80, seed=14)),
            ("smooth", smooth, np.clip(smooth.astype(np.int16) + 3, 0, 255).astype(np.uint8)),
            ("min", scene(11, 11, seed=15), scene(11, 11, seed=16))]
