"""B200-native ARKV decode hot path (arXiv 2603.08727): CUDA kernels for sm_100a
behind the C ABI in include/arkv.h, with a thin ctypes binding (arkv.py)."""
from .arkv import (ArkvCache, ArkvConfig, ArkvError, arkv_cache_bytes, arkv_oq_score,  # noqa: F401
                   arkv_schedule, arkv_version, make_config, lib)
