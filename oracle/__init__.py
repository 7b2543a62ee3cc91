"""CPU oracle (TEST INFRASTRUCTURE): see oracle/plex_oracle.py header.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package.  The product never does.
"""
from .plex_oracle import *  # noqa: F401,F403
