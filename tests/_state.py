"""Test helpers: synthetic logical state from the input module (plexgen)."""
from collections import OrderedDict

import numpy as np

from plexgen import manifest, gen_tensor


def full_state(model, seed=0, kinds=(0, 1, 2, 3), special_bits=0):
    """{(key, kind): full logical tensor bits} in manifest order."""
    out = OrderedDict()
    for k, s in manifest(model):
        for kd in kinds:
            out[(k, kd)] = gen_tensor(seed, k, kd, s, special_bits if kd else 0)
    return out


def fsdp_shards(full, world, rank, fsdp_rows):
    out = OrderedDict()
    for (k, kd), x in full.items():
        r0, r1 = fsdp_rows(x.shape[0], world, rank)
        out[(k, kd)] = x[r0:r1]
    return out


def master_shards(full, world, fsdp_rows):
    out = OrderedDict()
    for (k, kd), x in full.items():
        if kd != 1:
            continue
        out[k] = [x[slice(*fsdp_rows(x.shape[0], world, r))] for r in range(world)]
    return out
