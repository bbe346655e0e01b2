"""MGPBD oracle — TEST INFRASTRUCTURE ONLY.

ctypes wrapper around the plain serial fp64 C oracle (oracle.c).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import this
package; the product path (paper_2505_13390_b200) never does.
"""
from .oracle import *  # noqa: F401,F403
