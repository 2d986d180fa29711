"""The bench corpora, bit-exact: K1 (the fused auto-labeler) on every tile the bench labels --
the 4224-tile T-gray corpus of BASELINE configs[1] (the 100k-tile config is tile i = corpus[i
mod 4224], so this covers it), plus T-tint and T-rand tiles -- against the
reference algorithm on its own calls (oracle/autolabel_cv.py: OpenCV medianBlur/dilate +
NumPy, pinned to the reference's digests by tests/test_oracle_golden.py), run on all host
cores.  Filtered tiles, labels, masked-pixel counts and per-class counts must be identical.
"""
import multiprocessing as mp
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _oracle_chunk(tiles):
    import cv2
    cv2.setNumThreads(1)
    from oracle import autolabel_cv
    out = []
    for t in tiles:
        f, lbl, aff, first = autolabel_cv.process_tile(t)
        out.append((f, lbl, int(aff), first))
    return out


def _oracle(tiles):
    procs = os.cpu_count() or 1
    chunks = [tiles[i::procs] for i in range(procs)]
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_oracle_chunk, chunks)
    res = [None] * len(tiles)
    for i, part in enumerate(parts):
        res[i::procs] = part
    return res


def _check(tiles):
    from paper_2403_13135_b200 import icelabel as il
    got = il.autolabel(torch.from_numpy(tiles).cuda())
    filt, lab = got["filtered"].cpu().numpy(), got["label"].cpu().numpy()
    aff, counts = got["affected"].cpu().numpy(), got["counts"].cpu().numpy()
    unmatched = got["unmatched"].cpu().numpy()
    bad = []
    for i, (f, lbl, a, first) in enumerate(_oracle(list(tiles))):
        ok = (np.array_equal(filt[i], f) and np.array_equal(lab[i], lbl) and int(aff[i]) == a
              and counts[i].tolist() == np.bincount(lbl.ravel(), minlength=3)[:3].tolist()
              and int(unmatched[i]) == first)
        if not ok:
            bad.append(i)
    assert not bad, f"{len(bad)} tiles differ, first {bad[:10]}"


def test_bench_corpus_t_gray_4224_bit_exact():
    import bench
    _check(bench.make_corpus(4224))


def test_t_tint_and_t_rand_bit_exact():
    import bench
    gray = bench.make_corpus(1024)
    _check(bench.tint_corpus(gray))
    _check(bench.rand_corpus(512))
