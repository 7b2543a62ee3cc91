"""NEXT-4 HRRS (Alg. 1 / Eq. 3-4): the oracle pinned to the textbook HRRN it
extends and to Eq. 4's closed form; the product scheduler == the oracle."""
import random

import pytest

from oracle import plex_oracle as O
from paper_2605_20863_b200.scheduler import Req, Setup, priority, schedule


def test_eq4_closed_form():
    # P = 1 + W / (E + 1_switch * C_setup)   (Eq. 4)
    run = O.Request(0, 0.0, 5.0, remaining=2.0)
    a = O.Request(1, 1.0, 4.0)        # other job: switch
    b = O.Request(0, 3.0, 4.0)        # same job: no switch
    now, tl, to = 10.0, 1.5, 2.5
    assert O.hrrs_score(a, now, run, tl, to) == pytest.approx(1 + 9.0 / (4.0 + 4.0))
    assert O.hrrs_score(b, now, run, tl, to) == pytest.approx(1 + 7.0 / 4.0)
    assert O.hrrs_score(run, now, run, tl, to) == pytest.approx(1 + 10.0 / 2.0)


def test_reduces_to_hrrn_without_setup_cost():
    """C_setup = 0: classic HRRN (highest (W+E)/E first), brute force."""
    rng = random.Random(0)
    for _ in range(50):
        reqs = [O.Request(rng.randrange(4), rng.uniform(0, 10), rng.uniform(0.1, 5)) for _ in range(6)]
        now = 12.0
        tl = O.hrrs_schedule(now, reqs[0], None, reqs[1:], 0.0, 0.0)
        hrrn = sorted(reqs, key=lambda r: -((now - r.arrival + r.exec_time) / r.exec_time))
        assert [r for r, _, _ in tl] == hrrn
        # contiguous timeline from now
        t = now
        for r, s, e in tl:
            assert s == pytest.approx(t) and e == pytest.approx(s + r.exec_time)
            t = e


def test_setup_cost_batches_same_job_and_inserts_gaps():
    run = O.Request(0, 0.0, 5.0, remaining=1.0)
    same = O.Request(0, 2.0, 3.0)
    other = O.Request(1, 2.0, 3.0)
    tl = O.hrrs_schedule(4.0, other, run, [same], 1.0, 1.0)
    jobs = [r.job for r, _, _ in tl]
    assert jobs == [0, 0, 1]                       # batching of the resident job
    (_, s0, e0), (_, s1, e1), (_, s2, e2) = tl
    assert s0 == 4.0 and s1 == e0 and s2 == pytest.approx(e1 + 2.0)   # one switch gap


def test_no_starvation():
    run = O.Request(0, 0.0, 1.0, remaining=1.0)
    old = O.Request(1, -1000.0, 1.0)
    tl = O.hrrs_schedule(0.0, O.Request(0, 0.0, 1.0), run, [old], 5.0, 5.0)
    assert tl[0][0] is old


def test_product_scheduler_matches_oracle():
    rng = random.Random(1)
    for _ in range(200):
        n = rng.randrange(1, 8)
        specs = [(rng.randrange(3), rng.uniform(0, 20), rng.uniform(0.1, 6)) for _ in range(n)]
        now = 25.0
        tl_, to_ = rng.uniform(0, 3), rng.uniform(0, 3)
        has_run = rng.random() < 0.7
        o = [O.Request(j, a, e) for j, a, e in specs]
        p = [Req(j, a, e) for j, a, e in specs]
        orun = prun = None
        if has_run:
            orun, prun = O.Request(0, 1.0, 4.0, remaining=2.0), Req(0, 1.0, 4.0, remaining=2.0)
        ot = O.hrrs_schedule(now, o[0], orun, o[1:], tl_, to_)
        pt = schedule(now, p[0], prun, p[1:], Setup(to_, tl_))
        assert [(r.job, r.arrival, round(s, 9), round(e, 9)) for r, s, e in ot] == \
               [(r.job, r.arrival, round(s, 9), round(e, 9)) for r, s, e in pt]
        assert all(priority(pr, now, prun, Setup(to_, tl_)) ==
                   pytest.approx(O.hrrs_score(orr, now, orun, tl_, to_)) for pr, orr in zip(p, o))


def test_duplex_gap_is_max():
    assert Setup(2.0, 3.0, duplex=True).gap == 3.0
    assert Setup(2.0, 3.0).gap == 5.0
