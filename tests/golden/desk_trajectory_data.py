"""Inputs of the desk-scale 200-step trajectory golden, shared by the
generator (make_desk_trajectory.py, run against /root/reference) and the GPU test.

Corpus: the first N_TILES T-gray scenes of generate_corpus(101, N_TILES, 0.3) (our byte-
identical restatement lives in tests/fixtures/synth.py), labelled by the auto-labeler; batch
order: seeded reshuffles per epoch, batch 8.
"""
import torch

SPEC = dict(input_size=256, base_channels=16, depth=5, dropout=0.0)
N_TILES, BATCH, STEPS, SEED = 256, 8, 200, 0


def batch_order():
    g = torch.Generator().manual_seed(SEED)
    out = []
    while len(out) < STEPS:
        perm = torch.randperm(N_TILES, generator=g)
        out += [perm[i:i + BATCH] for i in range(0, N_TILES, BATCH)]
    return out[:STEPS]
