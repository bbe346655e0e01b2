"""B200-native (sm_100a) hot path of MGPBD (arXiv 2505.13390): UA-AMG-preconditioned CG on the XPBD
dual system, behind the C-ABI of include/mgpbd.h (libmgpbd.so).  This package holds the ctypes
binding (mgpbd.py), the in-tree build (build.py), the seeded input generators (scenes.py) and the
CUDA sources (csrc/)."""
from . import scenes  # noqa: F401
from .mgpbd import (Config, Context, MgpbdError, Stats, config_default, lib)  # noqa: F401
