"""CPU oracle for the bootstrapped-gate hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  The engine under
paper_2306_11006_b200/ never does, and has no CPU fallback.
"""
from .oracle import *  # noqa: F401,F403
