"""CPU oracle for the GSCL hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  The product package
(``paper_1207_1746_b200``) never imports it, and it imports nothing from the
product package.  See ``oracle/gscl_oracle.cpp`` for what each entry point
computes and which PAPER.md passage it follows.
"""
from .oracle import *  # noqa: F401,F403
