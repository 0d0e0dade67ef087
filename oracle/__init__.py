"""CPU oracle for the EF21M + ARC-Top-K step (test infrastructure only).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product package ``paper_2510_26709_b200`` never imports it.
"""
from .oracle import *  # noqa: F401,F403
