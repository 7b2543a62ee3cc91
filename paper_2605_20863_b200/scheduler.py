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
    # optional per-job model: switch cost from the state bytes of the two jobs
    # and the host-link rates the library measured (bytes / second)
    job_bytes: Optional[Dict[int, int]] = None
    bw_out: float = 0.0
    bw_in: float = 0.0

    @property
    def gap(self) -> float:
        """Timeline gap of one context switch (Eq. 3's C_setup; overlapped when duplex)."""
        return max(self.t_offload, self.t_load) if self.duplex else self.t_offload + self.t_load

    def switch_cost(self, prev: Optional[int], nxt: int) -> float:
        """C_setup of switching the group from job `prev` (None = empty) to `nxt`."""
        if self.job_bytes is None:
            return self.gap if prev is not None else self.t_load
        t_off = self.job_bytes[prev] / self.bw_out if prev is not None else 0.0
        t_on = self.job_bytes[nxt] / self.bw_in
        return max(t_off, t_on) if self.duplex else t_off + t_on

    @staticmethod
    def from_stats(stats: Dict[str, dict], n_offloads: int, n_onloads: int, duplex: bool = False,
                   job_bytes: Optional[Dict[int, int]] = None) -> "Setup":
        """T_offload / T_load per switch (seconds) from StateManager.stats(); with
        job_bytes, a per-job model from the measured D2H / H2D rates."""
        off = stats["d2h"]["ms"] / max(1, n_offloads) / 1e3
        on = stats["h2d"]["ms"] / max(1, n_onloads) / 1e3
        bw_out = stats["d2h"]["bytes"] / max(1e-9, stats["d2h"]["ms"] * 1e-3)
        bw_in = stats["h2d"]["bytes"] / max(1e-9, stats["h2d"]["ms"] * 1e-3)
        return Setup(off, on, duplex, job_bytes, bw_out, bw_in)


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
        if not switch:
            s = r.exec_time
        elif setup.job_bytes is None:
            s = r.exec_time + setup.t_offload + setup.t_load        # Eq. 3 as written
        else:
            s = r.exec_time + setup.switch_cost(running.job if running is not None else None, r.job)
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
            cursor += setup.switch_cost(resident, r.job)
            resident = r.job
        dur = r.remaining if (running is not None and r is running) else r.exec_time
        plan.append((r, cursor, cursor + dur))
        cursor += dur
    return plan
