"""HRRS runtime ordering fed by the measured switch cost (NEXT-4).

PAPER.md §4.4, Alg. 1 (:417-457) and Eq. 3-4 (:468-480): each pending request
i gets priority P_i = 1 + W_i / (E_i + 1_switch(i, curr) * C_setup) and the
timeline is laid out by descending priority with a setup gap wherever the
resident job changes.  C_setup = T_offload + T_load is not a guess here: it is
what this library's transition path measures (``Setup.from_stats``), and with
the duplex switch (NEXT-1) the gap is max(T_offload, T_load) instead.

Host logic only (scheduling decisions, no state bytes).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple


@dataclass
class Setup:
    t_offload: float
    t_load: float
    duplex: bool = False

    @property
    def gap(self) -> float:
        """Timeline gap of one context switch (Eq. 3's C_setup; overlapped when duplex)."""
        return max(self.t_offload, self.t_load) if self.duplex else self.t_offload + self.t_load

    @staticmethod
    def from_stats(stats: Dict[str, dict], n_offloads: int, n_onloads: int, duplex: bool = False) -> "Setup":
        """Per-switch T_offload / T_load (seconds) from StateManager.stats()."""
        off = stats["d2h"]["ms"] / max(1, n_offloads) / 1e3
        on = stats["h2d"]["ms"] / max(1, n_onloads) / 1e3
        return Setup(off, on, duplex)


@dataclass
class Req:
    job: int
    arrival: float
    exec_time: float
    remaining: float = 0.0
    name: str = field(default="")


def priority(r: Req, now: float, running: Optional[Req], setup: Setup) -> float:
    """Eq. 4 (with the running request using its remaining time, Alg. 1 line 4)."""
    wait = now - r.arrival
    if running is not None and r is running:
        s = r.remaining
    else:
        switch = running is None or r.job != running.job
        s = r.exec_time + (setup.t_offload + setup.t_load if switch else 0.0)
    return (wait + s) / s


def schedule(now: float, new: Req, running: Optional[Req], scheduled: Sequence[Req],
             setup: Setup) -> List[Tuple[Req, float, float]]:
    """Alg. 1 timeline: [(request, start, end)] by descending priority; a
    switch gap (Setup.gap, or T_load alone from an empty group) precedes every
    change of resident job."""
    omega = [new] + ([running] if running is not None else []) + list(scheduled)
    pri = [priority(r, now, running, setup) for r in omega]
    order = sorted(range(len(omega)), key=lambda i: -pri[i])
    cursor, resident = now, (running.job if running is not None else None)
    plan = []
    for i in order:
        r = omega[i]
        if r.job != resident:
            cursor += setup.gap if resident is not None else setup.t_load
            resident = r.job
        dur = r.remaining if (running is not None and r is running) else r.exec_time
        plan.append((r, cursor, cursor + dur))
        cursor += dur
    return plan
