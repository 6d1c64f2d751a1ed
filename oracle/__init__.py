"""CPU oracle for the restarted-PDHG LP iteration (TEST INFRASTRUCTURE ONLY).

Only ``tests/``, ``__graft_entry__.smoke()`` and the ``cpu_baseline`` /
``--impl reference`` legs of ``bench.py`` may import this package.  The product
(``paper_2412_09734_b200``) never imports it.  See ``oracle/mpax_oracle.c`` for
the contract and citations.
"""
from .oracle import *  # noqa: F401,F403
from . import spo  # noqa: F401,E402
