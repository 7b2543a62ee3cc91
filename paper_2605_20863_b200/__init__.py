"""B200-native state-transition path of PlexRL (arXiv 2605.20863).

Suspend/resume (gather-pack -> pinned host -> restore) and train->rollout
weight sync (fp32 master -> bf16 RNE -> TP/EP reshard over NVLink) as
hand-written sm_100a kernels behind the C ABI of ``include/plex.h``
(``libplex.so``).  Importing this package loads the library and fails if it
is missing: there is no CPU fallback.
"""
from . import _lib  # noqa: F401  (loads libplex.so or raises ImportError)
from ._lib import PlexError  # noqa: F401
from .state import (Group, Job, Plan, Slab, StateManager, cast_rne, checksum, synth_fill,  # noqa: F401
                    synth_mutate, transition_decide)

__all__ = ["Group", "Job", "Plan", "Slab", "StateManager", "PlexError", "synth_fill", "synth_mutate",
           "checksum", "cast_rne", "transition_decide"]
