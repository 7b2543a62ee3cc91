"""Pin for the oracle's multiplex replay (o10): the replayed state of each job
equals its initial state with exactly its own visits' mutations applied (XOR
masks commute, so the closed form is the XOR of all of that job's masks), and
the op list follows PAPER.md:555 / SPEC.md:361-363."""
import numpy as np

from oracle import plex_oracle as O
from plexgen import manifest, mutation_bits

from _state import full_state, fsdp_shards


def _mut(seeds):
    def f(job, step, key, kind, bits, base):
        idx = np.arange(base, base + bits.size, dtype=np.uint64)
        return bits ^ mutation_bits(seeds[job], step, key, kind, idx).reshape(bits.shape)
    return f


def test_multiplex_closed_form():
    W = 4
    models = ["toy", "toy-tied", "toy-moe", "toy-odd"]
    seeds = [0, 1, 2, 3]
    layouts = [(2, 2, 1), (1, 4, 1), (2, 2, 2), (1, 4, 1)]
    jobs, fulls = [], []
    for m, sd, (tp, dp, ep) in zip(models, seeds, layouts):
        full = full_state(m, seed=sd)
        fulls.append(full)
        jobs.append({"manifest": manifest(m), "tp": tp, "dp": dp, "ep": ep,
                     "shards": [fsdp_shards(full, W, r, O.fsdp_rows) for r in range(W)]})
    schedule = [0, 1, 2, 3] * 3 + [3, 0]
    visits, final = O.multiplex_replay(jobs, schedule, W, _mut(seeds))
    assert len(visits) == len(schedule)
    assert visits[0][0] == [(O.OP_ONLOAD, 0)]
    assert visits[1][0] == [(O.OP_OFFLOAD, 0), (O.OP_ONLOAD, 1)]
    assert visits[12][0] == []          # 3 -> 3: no switch
    n_visits = [schedule.count(j) for j in range(4)]
    for j, full in enumerate(fulls):
        for (key, kind), x in full.items():
            want = x.copy().reshape(-1)
            idx = np.arange(want.size, dtype=np.uint64)
            for step in range(n_visits[j]):
                want ^= mutation_bits(seeds[j], step, key, kind, idx)
            got = np.concatenate([final[j][r][(key, kind)].reshape(-1) for r in range(W)])
            assert np.array_equal(got, want)
    # the last visit's sync equals a fresh sync of the final master state
    j = schedule[-1]
    ms = {k: [final[j][r][(k, 1)] for r in range(W)] for k, _ in manifest(models[j])}
    again = O.weight_sync(ms, *layouts[j])
    for a, b in zip(again, visits[-1][1]):
        for k in a:
            assert np.array_equal(a[k], b[k])
