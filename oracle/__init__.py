"""TEST INFRASTRUCTURE ONLY -- the CPU oracle for the Founsure 1.0 encode hot path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
may import this package.  The product (paper_1702_07409_b200/) never does.
"""
from .oracle import *  # noqa: F401,F403
