"""B200-native IT-MPPI (arXiv 1707.02342) hot path.

The product is ``lib/libmppi_gpu.so`` (C ABI: ``include/mppi_gpu.h``) built
from ``csrc/`` for sm_100a; this package is its host-side mirror of the
reference controller API (see :mod:`.api`).
"""
from .api import *  # noqa: F401,F403
from .api import initial_states, make_config  # noqa: F401
